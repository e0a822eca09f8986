# config-4 mixed throughput vs the cost-pass unroll factors of the fp32 translation unit
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
C=paper_2506_05558_b200/csrc
rm -rf /tmp/objs; mkdir -p /tmp/objs
(for s in mba_solve mba_stages mba_pose mba_tri mba_match mba_pack mba_bootstrap; do
   /usr/local/cuda/bin/nvcc $F -c $C/$s.cu -o /tmp/objs/$s.o & done;
 /usr/local/cuda/bin/nvcc $F -c $C/mba_v4.cu -o /tmp/objs/mba_v4_f64.o & wait)
for cu in "4 2" "1 1" "2 1" "4 2" "1 1"; do
  set -- $cu
  /usr/local/cuda/bin/nvcc $F -DMBA_V4_F32 -DMBA_COST_U=$1 -DMBA_COST4_U=$2 -c $C/mba_v4.cu -o /tmp/mba_v4_f32.o
  /usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o /tmp/libminiba_u.so /tmp/mba_v4_f32.o /tmp/objs/*.o -lcudart
  MBA_LIB=/tmp/libminiba_u.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --precision mixed 2>&1 | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('mixed U=$1 U4=$2', round(d['value']))"
done
