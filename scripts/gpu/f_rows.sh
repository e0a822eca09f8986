# throughput + roofline at sizes larger than L2, ncu captures
python scripts/bench_pose.py --batch 65536 --m 256 --iters 5 > gpurun_out/f_pose.json 2>&1; tail -1 gpurun_out/f_pose.json | cut -c1-1500
python scripts/bench_triangulate.py --tracks 4000000 > gpurun_out/f_tri.json 2>&1; tail -1 gpurun_out/f_tri.json | cut -c1-1500
python scripts/bench_match.py > gpurun_out/f_match.json 2>&1; tail -1 gpurun_out/f_match.json | cut -c1-800
for k in pose tri; do
  if [ $k = pose ]; then cmd="scripts/bench_pose.py --batch 65536 --m 256 --iters 5 --steps 1 --cpu-problems 8"; re=pose_lm; fi
  if [ $k = tri ]; then cmd="scripts/bench_triangulate.py --tracks 4000000 --steps 1 --cpu-tracks 10"; re=triangulate; fi
  ncu --set full --clock-control none --import-source on -k regex:$re -s 3 -c 1 -o gpurun_out/ncu_f_$k -f python $cmd > gpurun_out/ncu_f_$k.log 2>&1
  python scripts/ncu_summary.py gpurun_out/ncu_f_$k.ncu-rep > gpurun_out/ncu_f_$k.txt 2>&1; head -22 gpurun_out/ncu_f_$k.txt
done
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 1 -c 1 -o gpurun_out/ncu_f_match -f python scripts/bench_match.py > gpurun_out/ncu_f_match.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_f_match.ncu-rep > gpurun_out/ncu_f_match.txt 2>&1; head -22 gpurun_out/ncu_f_match.txt
