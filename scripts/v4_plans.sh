#!/usr/bin/env bash
# v4 launch-plan sweep on a config-4 subset (cluster size R, CTAs per SM, threads per CTA)
set -u
cd "$(dirname "$0")/.."
N=${1:-16384}
run() { env "$@" MBA_DEBUG=1 bash scripts/kernel_sweep.sh v4 "$PREC" "$N" 2>&1 | tail -1 | sed "s/^/$* /"; }
for PREC in mixed f64; do
  run MBA_V4_X=default
  run MBA_V4_PERSM=1
  run MBA_V4_PERSM=2 MBA_V4_NT=128
  run MBA_V4_PERSM=2 MBA_V4_R=4
  run MBA_V4_PERSM=1 MBA_V4_R=2
done
