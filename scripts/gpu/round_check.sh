# acceptance + bootstrap tests, then the default bench line
python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_stages.py -q -x 2>&1 | tail -15
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 3000 gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
