# config-5 evidence: bench lines (f64, mixed), phase split, ncu capture, parity tests
python -m pytest tests/test_gpu_parity.py -q -x -k "config5 or grid or cauchy or cta" 2>&1 | tail -2
python bench.py --config 5 --steps 5 --warmup 3 --no-e2e > gpurun_out/r2_bench_c5.log 2>&1; tail -1 gpurun_out/r2_bench_c5.log > gpurun_out/r2_bench_c5.json
python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --precision mixed > gpurun_out/r2_bench_c5_mixed.log 2>&1; tail -1 gpurun_out/r2_bench_c5_mixed.log > gpurun_out/r2_bench_c5_mixed.json
python scripts/phase_prof.py --config 5 --problems 1 --precision f64 > gpurun_out/phase_c5_f64.json 2>&1
ITERS=10 bash scripts/gpu/ncu_c5.sh > /dev/null 2>&1
python -c "
import json
for f in ['gpurun_out/r2_bench_c5.json','gpurun_out/r2_bench_c5_mixed.json']:
    d=json.load(open(f)); print(f, d['value'], d['ms_per_step'], d['clocks'], d.get('cpu_baseline',{}).get('value'))
d=json.load(open('gpurun_out/phase_c5_f64.json')); print(d['ms'], {k:round(v['frac'],3) for k,v in d['phases'].items() if v['frac']>0})"
head -30 gpurun_out/ncu_c5_f64.txt
