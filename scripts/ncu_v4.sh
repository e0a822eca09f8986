#!/usr/bin/env bash
# ncu --set full capture of the v4 solver on a config-4 subset (one launch).
#   bash scripts/ncu_v4.sh <precision> <problems> <out-name>
set -u
cd "$(dirname "$0")/.."
prec=${1:-mixed}; n=${2:-2048}; name=${3:-v4_$prec}
cat > /tmp/ncu_v4_run.py <<PY
import sys, os
sys.path[:0] = ["$PWD", "$PWD/src"]
import torch
from paper_2506_05558_b200 import solver
from paper_2506_05558_b200.synth import make_batch
b = make_batch($n, n_cams=8, K=2000, seed=0, workers=os.cpu_count())
db = solver.to_device(solver.pack_synth(b))
prm = solver.LmParams(max_iters=200, precision="$prec", kernel="${KERNEL:-v4}")
sol = solver.solve(db, prm); torch.cuda.synchronize()
sol = solver.solve(db, prm, sol); torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-solve_v4} -s 1 -c 1 \
    -o gpurun_out/$name -f python /tmp/ncu_v4_run.py > gpurun_out/$name.log 2>&1
python scripts/ncu_summary.py gpurun_out/$name.ncu-rep > gpurun_out/$name.txt 2>&1
