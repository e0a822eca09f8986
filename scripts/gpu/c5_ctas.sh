for n in 148; do
MBA_GRID_CTAS=$n python scripts/phase_prof.py --config 5 --problems 1 --precision f64 > gpurun_out/phase_c5_$n.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/phase_c5_$n.json'));p=d['phases'];print($n, d['ms'], 'cam/chunk', p['setup_stage_validate|cam_chunks_cyc']['cycles_per_problem_iter']/max(p['setup_perm|n_cam_chunks']['cycles_per_problem_iter'],1), 'pair/chunk', p['setup_slots_X|pair_chunks_cyc']['cycles_per_problem_iter']/max(p['setup_pairs|n_pair_chunks']['cycles_per_problem_iter'],1))"
done
