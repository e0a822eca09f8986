for r in 1 2 4 8; do echo "R=$r"; MBA_V4_R=$r python scripts/bench_bootstrap.py --reps 5 2>&1 | tail -1 | cut -c1-400; done
for r in 1 2 4 8 16; do echo "cfg1 R=$r"; MBA_V4_R=$r python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['roofline']['plan'])"; done
