// mba_pack.cu -- device-side packing of raw observation arrays into the
// solver's point-major 16-byte records (sm_100a).
//
// The reference's producers emit observations track-major
// (miniba.py:762-770, bootstrap) or camera-major (smoke_miniba.py:50-55), and
// BaProblem (miniba.py:65-83) carries them as separate cam_idx / pt_idx / uv
// arrays. mba_solve consumes {float u, float v, int32 cam, int32 pt} records
// sorted point-major within each problem (plus an optional float2 low-order
// uv stream). This kernel builds them on the device from the uploaded raw
// arrays (int32 indices, uv rounded to float32 and -- only when some value is
// not fp32-representable -- its low-order float32 residual), one CTA per
// problem:
//
//  * one coalesced pass validates the indices (out of range -> the records are
//    written as given and mba_solve reports the problem malformed) and checks
//    whether the problem is already point-major -- the common case, then a
//    straight conversion pass;
//  * otherwise a stable counting sort: per-point counts (shared-memory
//    atomics, or global for very large problems), a block-wide exclusive scan,
//    then placement in input order by warp 0 with __match_any_sync ranks, so
//    observations of one point keep their input order (numpy's stable argsort,
//    which the fp64 reductions' order is defined by).
//
// Algorithmic bytes per observation: 16 read (int32 cam, int32 pt, 2 x f32
// uv) + 16 written (+ 8 + 8 with the low-order stream); HBM-bound.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/miniba.h"

namespace mba {
namespace pack {

constexpr int kThreads = 256;
constexpr int kSmemCounts = 8192;   // points whose counts fit in shared memory (32 KB)

__device__ __forceinline__ MbaObs make_rec(float2 uv, int c, int p) {
  MbaObs r;
  r.u = uv.x;
  r.v = uv.y;
  r.cam = c;
  r.pt = p;
  return r;
}

__global__ void __launch_bounds__(kThreads) pack_kernel(int n_problems, const int64_t* __restrict__ obs_off,
                                                        const int64_t* __restrict__ pt_off,
                                                        const int64_t* __restrict__ cam_off,
                                                        const int32_t* __restrict__ cam,
                                                        const int32_t* __restrict__ pt,
                                                        const float2* __restrict__ uv,
                                                        const float2* __restrict__ uv_lo, MbaObs* __restrict__ out,
                                                        float2* __restrict__ out_lo, int32_t* __restrict__ gcount) {
  __shared__ int s_cnt[kSmemCounts];
  __shared__ int s_wsum[kThreads / 32];
  const int b = blockIdx.x;
  if (b >= n_problems) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t k0 = obs_off[b];
  const int K = (int)(obs_off[b + 1] - k0);
  const int P = (int)(pt_off[b + 1] - pt_off[b]);
  const int n = (int)(cam_off[b + 1] - cam_off[b]);
  int bad = 0, uns = 0;
  for (int k = tid; k < K; k += kThreads) {
    const int c = __ldg(cam + k0 + k), p = __ldg(pt + k0 + k);
    bad |= c < 0 || c >= n || p < 0 || p >= P;
    if (k > 0) uns |= __ldg(pt + k0 + k - 1) > p;
  }
  bad = __syncthreads_or(bad);
  uns = __syncthreads_or(uns);
  const bool lo = out_lo != nullptr && uv_lo != nullptr;
  if (bad || !uns) {   // as given: already point-major (or malformed: mba_solve flags it)
    for (int k = tid; k < K; k += kThreads) {
      out[k0 + k] = make_rec(__ldg(uv + k0 + k), __ldg(cam + k0 + k), __ldg(pt + k0 + k));
      if (lo) out_lo[k0 + k] = __ldg(uv_lo + k0 + k);
    }
    return;
  }
  // stable counting sort by point
  int* cnt = P <= kSmemCounts ? s_cnt : gcount + pt_off[b];
  for (int p = tid; p < P; p += kThreads) cnt[p] = 0;
  __syncthreads();
  for (int k = tid; k < K; k += kThreads) atomicAdd(cnt + __ldg(pt + k0 + k), 1);
  __syncthreads();
  // exclusive scan of cnt[0..P) in tiles of kThreads
  int carry = 0;
  for (int base = 0; base < P; base += kThreads) {
    const int p = base + tid;
    const int v = p < P ? cnt[p] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[wid] = x;
    __syncthreads();
    int pre = carry, tot = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      if (w < wid) pre += s_wsum[w];
      tot += s_wsum[w];
    }
    if (p < P) cnt[p] = pre + x - v;
    carry += tot;
    __syncthreads();
  }
  // placement in input order (warp 0): ranks among equal points by match_any
  if (wid == 0) {
    const unsigned lt = (1u << lane) - 1u;
    for (int base = 0; base < K; base += 32) {
      const int k = base + lane;
      const bool act = k < K;
      const unsigned m = __ballot_sync(0xffffffffu, act);
      int p = -1 - lane;   // distinct keys for inactive lanes
      float2 q = make_float2(0.f, 0.f), ql = make_float2(0.f, 0.f);
      int c = 0;
      if (act) {
        p = __ldg(pt + k0 + k);
        c = __ldg(cam + k0 + k);
        q = __ldg(uv + k0 + k);
        if (lo) ql = __ldg(uv_lo + k0 + k);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, p) & m;
      const int dst = act ? cnt[p] + __popc(peers & lt) : 0;
      __syncwarp();
      if (act && (peers & lt) == 0) cnt[p] += __popc(peers);
      __syncwarp();
      if (act) {
        out[k0 + dst] = make_rec(q, c, p);
        if (lo) out_lo[k0 + dst] = ql;
      }
    }
  }
}

}  // namespace pack
}  // namespace mba

extern "C" {

size_t mba_pack_obs_workspace_bytes(int64_t total_points) { return (size_t)(total_points > 0 ? total_points : 1) * 4; }

int32_t mba_pack_obs(int32_t n_problems, const int64_t* obs_off, const int64_t* pt_off, const int64_t* cam_off,
                     const int32_t* cam, const int32_t* pt, const float* uv, const float* uv_lo, MbaObs* out,
                     float* out_lo, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_problems < 0 || (n_problems > 0 && (!obs_off || !pt_off || !cam_off || !out))) return MBA_ERR_INVALID;
  if (n_problems == 0) return MBA_OK;
  (void)workspace_bytes;   // >= 4 x total points (mba_pack_obs_workspace_bytes); used for P > 8192 only
  mba::pack::pack_kernel<<<n_problems, mba::pack::kThreads, 0, (cudaStream_t)stream>>>(
      n_problems, obs_off, pt_off, cam_off, cam, pt, reinterpret_cast<const float2*>(uv),
      reinterpret_cast<const float2*>(uv_lo), out, reinterpret_cast<float2*>(out_lo), (int32_t*)workspace);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Trace compaction: the per-problem LM traces mba_solve writes are max_iters
// wide (costs max_iters + 1), but only the first n_iters entries of each row
// are meaningful (config 4: 11.6 of 200). Packing them back to back before the
// read-back cuts the device-to-host traffic of a batch by ~95 %.

namespace mba {
namespace pack {

// off[b] = sum_{b' < b} n_iters[b'] (one CTA)
__global__ void __launch_bounds__(1024) trace_scan_kernel(int n, const int32_t* __restrict__ n_iters,
                                                          int64_t* __restrict__ off) {
  __shared__ long long warp_tot[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base <= n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const long long v = i < n ? n_iters[i] : 0;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    long long pre = carry, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < wid) pre += warp_tot[w];
      tot += warp_tot[w];
    }
    if (i <= n) off[i] = pre + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// one warp per problem: row b's first n entries to off[b] (costs: n + 1 to off[b] + b)
__global__ void trace_copy_kernel(int n, int max_iters, const int32_t* __restrict__ n_iters,
                                  const int64_t* __restrict__ off, const double* __restrict__ costs,
                                  const double* __restrict__ lambdas, const uint8_t* __restrict__ accepted,
                                  const uint8_t* __restrict__ evals, double* __restrict__ c_out,
                                  double* __restrict__ l_out, uint8_t* __restrict__ a_out,
                                  uint8_t* __restrict__ e_out) {
  const int b = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= n) return;
  const int it = n_iters[b];
  const int w = max_iters > 0 ? max_iters : 1;
  const int64_t o = off[b];
  for (int i = lane; i <= it; i += 32) c_out[o + b + i] = costs[(int64_t)b * (max_iters + 1) + i];
  for (int i = lane; i < it; i += 32) {
    l_out[o + i] = lambdas[(int64_t)b * w + i];
    a_out[o + i] = accepted[(int64_t)b * w + i];
    e_out[o + i] = evals[(int64_t)b * w + i];
  }
}

}  // namespace pack
}  // namespace mba

extern "C" int32_t mba_compact_traces(int32_t n_problems, int32_t max_iters, const int32_t* n_iters,
                                      const double* costs, const double* lambdas, const uint8_t* accepted,
                                      const uint8_t* evals, int64_t* trace_off, double* costs_out,
                                      double* lambdas_out, uint8_t* accepted_out, uint8_t* evals_out,
                                      void* stream) {
  if (n_problems < 0 || max_iters < 0) return MBA_ERR_INVALID;
  if (n_problems == 0) return MBA_OK;
  cudaStream_t st = (cudaStream_t)stream;
  mba::pack::trace_scan_kernel<<<1, 1024, 0, st>>>(n_problems, n_iters, trace_off);
  const int threads = 256;
  const int blocks = (int)(((int64_t)n_problems * 32 + threads - 1) / threads);
  mba::pack::trace_copy_kernel<<<blocks, threads, 0, st>>>(n_problems, max_iters, n_iters, trace_off, costs,
                                                           lambdas, accepted, evals, costs_out, lambdas_out,
                                                           accepted_out, evals_out);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}
