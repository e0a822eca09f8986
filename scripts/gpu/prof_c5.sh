python -m pytest tests/test_gpu_acceptance.py -q -x -k jacobians 2>&1 | tail -3
python scripts/phase_prof.py --config 5 --problems 1 --precision f64 > gpurun_out/phase_c5_f64.json 2>&1; cat gpurun_out/phase_c5_f64.json
python bench.py --config 5 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-700
