#!/usr/bin/env bash
# threads-per-CTA sweep of the v4 kernel (one problem per SM) on a config-4 subset
set -u
cd "$(dirname "$0")/.."
N=${1:-16384}
for PREC in mixed f64; do
  for NT in 256 384 512; do
    env MBA_V4_NT=$NT MBA_V4_PERSM=1 MBA_V4_R=1 bash scripts/kernel_sweep.sh v4 "$PREC" "$N" 2>&1 | tail -1 | sed "s/^/NT=$NT /"
  done
done
