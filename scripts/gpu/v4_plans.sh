# config-4 f64 throughput under alternative cluster / occupancy plans
for env in "" "MBA_V4_R=2 MBA_V4_PERSM=2" "MBA_V4_R=2 MBA_V4_PERSM=1" "MBA_V4_R=4 MBA_V4_PERSM=2"; do
  echo "== $env"
  env $env MBA_DEBUG=1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/plan_err.txt | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['roofline'].get('plan'))"
  grep "plan:" gpurun_out/plan_err.txt | head -2
done
