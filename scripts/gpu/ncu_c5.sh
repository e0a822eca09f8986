cat > /tmp/ncu_c5_run.py <<PY
import sys, os
sys.path[:0] = ["$PWD", "$PWD/src"]
import torch
from paper_2506_05558_b200 import solver
from paper_2506_05558_b200.synth import make_batch, CONFIGS
c = CONFIGS[5]
b = make_batch(1, n_cams=32, K=200000, seed=0, outlier_frac=0.2)
db = solver.to_device(solver.pack_synth(b))
prm = solver.LmParams(max_iters=int(os.environ.get("ITERS", "10")), loss="cauchy", precision="${PREC:-f64}")
sol = solver.solve(db, prm); torch.cuda.synchronize()
sol = solver.solve(db, prm, sol); torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:solve_grid -s 1 -c 1 \
    -o gpurun_out/ncu_c5_${PREC:-f64} -f python /tmp/ncu_c5_run.py > gpurun_out/ncu_c5.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_c5_${PREC:-f64}.ncu-rep > gpurun_out/ncu_c5_${PREC:-f64}.txt 2>&1
cat gpurun_out/ncu_c5_${PREC:-f64}.txt | head -70
