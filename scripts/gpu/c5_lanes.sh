python scripts/phase_prof.py --config 5 --problems 1 --precision f64 > gpurun_out/phase_c5_l.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/phase_c5_l.json'));p=d['phases'];print(d['ms'], 'active lanes sum', p['setup_perm|n_cam_chunks']['cycles_per_problem_iter'], 'pair iters (tid0)', p['setup_pairs|n_pair_chunks']['cycles_per_problem_iter'])"
