# v4 linearisation cache: parity (cluster kernel paths) + config 4 / 3 throughput
python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch_api.py tests/test_gpu_acceptance.py -q -x 2>&1 | tail -2
for p in f64 mixed; do python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --precision $p 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c4', '$p', round(d['value']), d['roofline']['frac'])"; done
python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c3 f64', round(d['value']))"
python scripts/parity_sweep.py --config 4 --problems 512 --precision f64 > gpurun_out/parity_c4_f64.json 2>&1; tail -c 400 gpurun_out/parity_c4_f64.json
