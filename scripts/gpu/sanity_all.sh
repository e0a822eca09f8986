# full GPU suite + compute-sanitizer over every kernel family
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
rm -f gpurun_out/sanitizers.txt
for tool in memcheck racecheck synccheck; do
  echo "## $tool" >> gpurun_out/sanitizers.txt
  timeout 1200 compute-sanitizer --tool $tool --print-limit 5 python scripts/sanitize_run.py 2>&1 | tail -3 >> gpurun_out/sanitizers.txt
done
cat gpurun_out/sanitizers.txt
