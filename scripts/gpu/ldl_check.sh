# blocked LDL^T in the grid / CTA kernels: parity + config-5 timing + phase split
python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch_api.py -q -x 2>&1 | tail -3
python bench.py --config 5 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-300
python scripts/phase_prof.py --config 5 --problems 1 --precision f64 > gpurun_out/phase_c5_f64.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/phase_c5_f64.json'));print(d['ms'], {k:round(v['frac'],3) for k,v in d['phases'].items() if v['frac']>0})"
