set -x
lscpu | grep -E "Model name|^CPU\(s\)|Flags" | cut -c1-300
nproc; python -c "import os;print(len(os.sched_getaffinity(0)))"
python scripts/gpu/hosttime.py 2>&1 || true
python -m pytest tests/test_gpu_batch_api.py tests/test_host_pack.py -x -q 2>&1 | tail -15
python scripts/bench_e2e_api.py --problems 65536 --steps 3 > gpurun_out/e2e_api.json 2>&1; tail -3 gpurun_out/e2e_api.json
