python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch_api.py -q -x 2>&1 | tail -2
for p in f64 mixed; do python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --precision $p 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c3', '$p', d['value'], d['roofline']['plan'])"; done
for p in f64 mixed; do python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --precision $p 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c4', '$p', d['value'], d['roofline']['plan'])"; done
