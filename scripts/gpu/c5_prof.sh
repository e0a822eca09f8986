python scripts/phase_prof.py --config 5 --problems 1 --precision f64 > gpurun_out/phase_c5_f64.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/phase_c5_f64.json'));print(d['ms'], {k:round(v['frac'],3) for k,v in d['phases'].items() if v['frac']>0})"
