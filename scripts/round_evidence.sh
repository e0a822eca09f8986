#!/usr/bin/env bash
# Round evidence on one B200: bench lines (f64 default + mixed + reference arm),
# ncu launch list of the default bench, ncu --set full of the solve kernel.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/ev_bench_f64.log 2>&1
python bench.py --precision mixed --no-cpu-baseline > gpurun_out/ev_bench_mixed.log 2>&1
python bench.py --impl reference > gpurun_out/ev_bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
    --problems 16384 > gpurun_out/ev_launches_bench.log 2>&1
KERNEL=auto bash scripts/ncu_v4.sh f64 2048 ev_ncu_f64
KERNEL=auto bash scripts/ncu_v4.sh mixed 2048 ev_ncu_mixed
rm -f gpurun_out/ev_ncu_mixed.ncu-rep   # keep the pull under 64 MiB (summary is in ev_ncu_mixed.txt)
tail -1 gpurun_out/ev_bench_f64.log | cut -c1-300
tail -1 gpurun_out/ev_bench_mixed.log | cut -c1-200
tail -1 gpurun_out/ev_bench_ref.log | cut -c1-200
