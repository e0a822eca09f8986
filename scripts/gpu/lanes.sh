python scripts/phase_prof.py --config 5 --problems 1 --precision f64 > gpurun_out/phase_c5_l.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/phase_c5_l.json'));p=list(d['phases'].values());print('c5', d['ms'], 'pair lanes', p[13]['cycles_per_problem_iter']/max(p[14]['cycles_per_problem_iter'],1))"
python scripts/phase_prof.py --config 4 --problems 8192 --precision f64 > gpurun_out/phase_c4_l.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/phase_c4_l.json'));p=list(d['phases'].values());print('c4', d['ms'], 'cam lanes', p[11]['cycles_per_problem_iter']/max(p[12]['cycles_per_problem_iter'],1), 'pair lanes', p[13]['cycles_per_problem_iter']/max(p[14]['cycles_per_problem_iter'],1), {k:round(v['frac'],3) for k,v in d['phases'].items() if v['frac']>0.001})"
