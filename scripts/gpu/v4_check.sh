python -m pytest tests/test_gpu_parity.py -q -x -k "v4 or golden or batched or hetero or clusters or config3" 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('f64', d['value'], d['solver']['mean_lm_iters'])"
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --precision mixed 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('mixed', d['value'], d['solver']['mean_lm_iters'])"
python scripts/phase_prof.py --config 4 --problems 8192 --precision f64 > gpurun_out/phase_c4.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/phase_c4.json'));print(d['ms'], {k:round(v['cycles_per_problem_iter']) for k,v in d['phases'].items() if v['frac']>0.001})"
