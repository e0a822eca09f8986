# Round-2 evidence on one B200: bench lines (default f64, mixed, configs 1/2/3/5,
# reference arm), ncu launch list of the default bench command, ncu --set full
# of the cluster kernel (f64 + mixed) and of the config-5 grid kernel.
set -u
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_default.log 2>&1
python bench.py --steps 10 --warmup 3 --precision mixed --no-cpu-baseline > gpurun_out/r2_bench_mixed.log 2>&1
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1
for c in 1 2 3 5; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2_bench_c$c.log 2>&1; done
python bench.py --config 3 --steps 5 --warmup 3 --precision mixed --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_c3_mixed.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
    --problems 16384 > gpurun_out/r2_launches_bench.log 2>&1
KERNEL=auto bash scripts/ncu_v4.sh f64 2048 r2_ncu_v4_f64
KERNEL=auto bash scripts/ncu_v4.sh mixed 2048 r2_ncu_v4_mixed
rm -f gpurun_out/r2_ncu_v4_mixed.ncu-rep gpurun_out/r2_ncu_v4_f64.ncu-rep
ITERS=10 bash scripts/gpu/ncu_c5.sh > /dev/null 2>&1
cp gpurun_out/ncu_c5_f64.txt gpurun_out/r2_ncu_grid_c5_f64.txt; rm -f gpurun_out/ncu_c5_f64.ncu-rep
for f in default mixed ref c1 c2 c3 c5 c3_mixed; do echo "== $f"; tail -1 gpurun_out/r2_bench_$f.log | cut -c1-400; done
