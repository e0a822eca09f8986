#!/usr/bin/env bash
# config 3 (1,024 x K=20k) device throughput per cluster size R (MBA_V4_R)
set -u
cd "$(dirname "$0")/.."
N=${N:-512}
for prec in f64 mixed; do
  for R in ${RS:-auto 8 9 10 12 16}; do
    env_r=""; [ "$R" != auto ] && env_r="MBA_V4_R=$R"
    out=$(env $env_r MBA_DEBUG=1 timeout 300 python bench.py --config 3 --precision $prec --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --problems $N 2>/tmp/c3err | tail -1)
    echo "prec=$prec R=$R $(grep -m1 'active clusters' /tmp/c3err) :: $(python -c 'import json,sys; d=json.loads(sys.argv[1]); print(round(d["value"]), "problems/s", round(d["ms_per_step"],2), "ms", d["roofline"].get("plan"))' "$out" 2>&1 | tail -1)"
  done
done
