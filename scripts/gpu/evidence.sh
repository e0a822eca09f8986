# round evidence: sanitizers, parity sweeps
set -x
for tool in memcheck racecheck synccheck; do
  echo "## $tool" >> gpurun_out/sanitizers.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 5 python scripts/sanitize_run.py 2>&1 | tail -3 >> gpurun_out/sanitizers.txt
done
python scripts/parity_sweep.py --config 4 --problems 512 --precision f64 > gpurun_out/parity_c4_f64.json 2>&1
python scripts/parity_sweep.py --config 4 --problems 512 --precision mixed > gpurun_out/parity_c4_mixed.json 2>&1
python scripts/parity_sweep.py --config 3 --problems 16 --precision f64 > gpurun_out/parity_c3_f64.json 2>&1
python scripts/parity_sweep.py --config 3 --problems 16 --precision mixed > gpurun_out/parity_c3_mixed.json 2>&1
cat gpurun_out/sanitizers.txt gpurun_out/parity_*.json
