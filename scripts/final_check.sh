#!/usr/bin/env bash
# End-of-round check on one B200: GPU tests, smoke(), the reference smoke script
# against the drop-in package, and the round evidence (bench lines, launch list,
# ncu captures, per-config throughput, pose-LM bench).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
timeout 300 python oracle/_ref/smoke_miniba.py > gpurun_out/fin_ref_smoke.log 2>&1
bash scripts/round_evidence.sh
bash scripts/configs_quick.sh > gpurun_out/ev_configs.jsonl 2>&1
python scripts/bench_pose.py > gpurun_out/ev_pose.jsonl 2>&1
python scripts/bench_pose.py --batch 256 --m 4 --iters 5 >> gpurun_out/ev_pose.jsonl 2>&1
cat gpurun_out/fin_pytest.log; tail -2 gpurun_out/fin_smoke.log; tail -2 gpurun_out/fin_ref_smoke.log
