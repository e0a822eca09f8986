#!/usr/bin/env bash
# Bench every BASELINE config (1-5) in both precisions; one JSON line each.
#   bash scripts/bench_all.sh > gpurun_out/bench_all.jsonl
set -u
cd "$(dirname "$0")/.."
for cfg in 1 2 3 4 5; do
  for prec in f64 mixed; do
    steps=3; warm=3
    [ "$cfg" = 4 ] && steps=3
    python bench.py --config "$cfg" --precision "$prec" --steps "$steps" --warmup "$warm" \
      $( [ "$prec" = mixed ] && echo --no-cpu-baseline ) 2>/dev/null | tail -1
  done
done
