# config-5 solve time vs the grid kernel's cost-pass unroll (MBA_GRID_COST_U)
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
C=paper_2506_05558_b200/csrc
rm -rf /tmp/objs; mkdir -p /tmp/objs
(for s in mba_stages mba_pose mba_tri mba_match mba_pack mba_bootstrap; do
   /usr/local/cuda/bin/nvcc $F -c $C/$s.cu -o /tmp/objs/$s.o & done;
 /usr/local/cuda/bin/nvcc $F -c $C/mba_v4.cu -o /tmp/objs/mba_v4_f64.o &
 /usr/local/cuda/bin/nvcc $F -DMBA_V4_F32 -c $C/mba_v4.cu -o /tmp/objs/mba_v4_f32.o & wait)
for u in 4 1 2 8 4; do
  /usr/local/cuda/bin/nvcc $F -DMBA_GRID_COST_U=$u -c $C/mba_solve.cu -o /tmp/mba_solve.o
  /usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o /tmp/libminiba_u.so /tmp/mba_solve.o /tmp/objs/*.o -lcudart
  MBA_LIB=/tmp/libminiba_u.so python bench.py --config 5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('U=$u', round(d['ms_per_step'],3))"
done
