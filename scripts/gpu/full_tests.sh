python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; tail -40 gpurun_out/pytest_gpu.txt
