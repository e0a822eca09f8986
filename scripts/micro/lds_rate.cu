// Shared-memory load throughput per SM for broadcast (all lanes same address)
// and linear (lane-contiguous) patterns at 32/64/128-bit width, 8 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 lds_rate.cu -o lds_rate
#include <cstdio>
template <int W, bool BC>
__global__ void k(int n, long long* cyc, float* out) {
  __shared__ __align__(16) float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float acc = 0;
  long long t = clock64();
  for (int it = 0; it < n; ++it) {
    const int base = (it * 64) & 4095;
    const int off = BC ? base : base + lane * (W / 4);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int o = off + u * 256;
      if constexpr (W == 4) acc += s[o];
      else if constexpr (W == 8) { float2 v = *reinterpret_cast<float2*>(s + o); acc += v.x + v.y; }
      else { float4 v = *reinterpret_cast<float4*>(s + o); acc += v.x + v.y + v.z + v.w; }
    }
  }
  __syncthreads();
  t = clock64() - t;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t;
}
int main() {
  long long* dc; float* o;
  cudaMalloc(&dc, 8); cudaMalloc(&o, 1 << 20);
  const int n = 2048;
  auto run = [&](auto kern, const char* name) {
    kern<<<1, 256>>>(n, dc, o);
    kern<<<1, 256>>>(n, dc, o);
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("%-22s %.2f cycles per warp-LDS (SM-wide, 8 warps)\n", name, (double)c / (n * 8.0 * 8));
  };
  run(k<4, true>, "LDS.32 broadcast");
  run(k<8, true>, "LDS.64 broadcast");
  run(k<16, true>, "LDS.128 broadcast");
  run(k<4, false>, "LDS.32 linear");
  run(k<8, false>, "LDS.64 linear");
  run(k<16, false>, "LDS.128 linear");
  return 0;
}
