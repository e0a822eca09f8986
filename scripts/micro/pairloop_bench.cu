// Micro-benchmark: the grid kernel's pair-job loop (two 18-double Y rows per
// co-observation pair from global memory, 36 FP64 accumulators per lane) on
// config-5-sized data, with and without a large dynamic shared-memory
// allocation (which shrinks the L1 data cache to a few KB).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void pair_loop(const double* __restrict__ Y, const int2* __restrict__ pairs, int n_pairs, int chunk,
                          double* out, long long* ns, int smem_touch) {
  extern __shared__ double sm[];
  if (smem_touch && threadIdx.x == 0) sm[0] = 0;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  double acc[36];
  for (int i = 0; i < 36; ++i) acc[i] = 0;
  const int n_chunks = (n_pairs + chunk - 1) / chunk;
  for (int c = gw; c < n_chunks; c += nw) {
    const int q1 = min(n_pairs, (c + 1) * chunk);
    for (int q = c * chunk + lane; q < q1; q += 32) {
      const int2 pr = pairs[q];
      double yi[18], yj[18];
      const double2* a = reinterpret_cast<const double2*>(Y + (size_t)pr.x * 20);
      const double2* b = reinterpret_cast<const double2*>(Y + (size_t)pr.y * 20);
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        double2 u = a[i], v = b[i];
        yi[2 * i] = u.x; yi[2 * i + 1] = u.y; yj[2 * i] = v.x; yj[2 * i + 1] = v.y;
      }
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int cc = 0; cc < 6; ++cc)
          acc[r * 6 + cc] += yi[r * 3] * yj[cc * 3] + yi[r * 3 + 1] * yj[cc * 3 + 1] + yi[r * 3 + 2] * yj[cc * 3 + 2];
    }
  }
  long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  double s = 0;
  for (int i = 0; i < 36; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (lane == 0) ns[gw] = t1 - t0;
}

int main() {
  const int K = 200000, n_pairs = 550000, chunk = 512;
  std::vector<double> hY((size_t)K * 20);
  for (size_t i = 0; i < hY.size(); ++i) hY[i] = (double)(i % 97) * 1e-3;
  std::vector<int2> hp(n_pairs);
  srand(1);
  for (int q = 0; q < n_pairs; ++q) hp[q] = make_int2(rand() % K, rand() % K);
  double *Y, *out;
  int2* p;
  long long* ns;
  cudaMalloc(&Y, hY.size() * 8);
  cudaMalloc(&p, n_pairs * 8);
  cudaMalloc(&out, 148 * 256 * 8);
  cudaMalloc(&ns, 148 * 8 * 8);
  cudaMemcpy(Y, hY.data(), hY.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(p, hp.data(), n_pairs * 8, cudaMemcpyHostToDevice);
  for (int big : {0, 1}) {
    int smem = big ? 220 * 1024 : 0;
    cudaFuncSetAttribute(pair_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      pair_loop<<<148, 256, smem>>>(Y, p, n_pairs, chunk, out, ns, big);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<long long> h(148 * 8);
      cudaMemcpy(h.data(), ns, h.size() * 8, cudaMemcpyDeviceToHost);
      long long mx = 0, sm_ = 0;
      for (auto v : h) { mx = v > mx ? v : mx; sm_ += v; }
      printf("smem=%dKB kernel %.3f ms; per-warp max %.1f us mean %.1f us (%s)\n", smem / 1024, ms, mx / 1e3,
             sm_ / 1e3 / h.size(), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
