set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python scripts/parity_sweep.py --config 4 --problems 512 --precision mixed > gpurun_out/sweep_mixed.json 2>&1
python -m pytest tests/test_gpu_parity.py -q -x -k "mixed_precision_against_golden" 2>&1 | tail -15
python bench.py --precision mixed --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_mixed.json 2>&1
cat gpurun_out/sweep_mixed.json; cut -c1-600 gpurun_out/bench_mixed.json
