# full round-2 evidence: GPU tests, smoke, bench lines, ncu, (f)-row measurements
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r2_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; tail -1 gpurun_out/r2_smoke.txt
bash scripts/gpu/final_evidence.sh > /dev/null 2>&1
python scripts/bench_bootstrap.py --reps 5 2>&1 | tail -1 > gpurun_out/r2_bench_bootstrap.json
bash scripts/gpu/f_rows.sh > /dev/null 2>&1
rm -f gpurun_out/*.ncu-rep
for f in default mixed ref c1 c2 c3 c5 c3_mixed; do echo "== $f"; tail -1 gpurun_out/r2_bench_$f.log | cut -c1-250; done
