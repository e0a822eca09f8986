// FP64 FMA throughput / latency calibration on one SM: NT threads, NC
// independent chains per thread, clock64 around the loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 dfma_rate.cu -o dfma_rate
#include <cstdio>
template <int NC>
__global__ void k(double a, double b, int n, long long* cyc, double* out) {
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = threadIdx.x + c;
  __syncthreads();
  long long t = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = fma(acc[c], a, b);
  __syncthreads();
  t = clock64() - t;
  double s = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t;
}
int main() {
  long long* dc; double* o;
  cudaMalloc(&dc, 8); cudaMalloc(&o, 8 << 20);
  const int n = 4096;
  for (int nt : {32, 128, 256, 512, 1024}) {
    auto run = [&](auto kern, int NC) {
      kern<<<1, nt>>>(1.0000001, 1e-9, n, dc, o);
      kern<<<1, nt>>>(1.0000001, 1e-9, n, dc, o);
      long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      const double fma_per_clk = (double)nt * NC * n / c;
      printf("threads %4d chains %2d: %.1f FMA/clk/SM  (%.2f cycles per dependent DFMA)\n", nt, NC, fma_per_clk,
             (double)c / n);
    };
    run(k<1>, 1); run(k<4>, 4); run(k<16>, 16);
  }
  return 0;
}
