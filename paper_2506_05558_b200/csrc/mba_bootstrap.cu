// mba_bootstrap.cu -- the bootstrap schedule around lm_solve as one device
// sequence (reference gsrecon/miniba.py:782-805, run_schedule):
//
//     solve (first half of the iterations)              mba_solve
//  -> residual norms of the half-converged state,       filter_kernel
//     median + factor * MAD keep mask (miniba.py:57-62),
//     points need >= 2 surviving observations
//  -> exclusive scan of the surviving counts            scan_kernel
//  -> stable compaction of the observation records      compact_kernel
//  -> solve (second half, from the first half's state)  mba_solve
//  -> gauge: unit mean pairwise camera distance          gauge_kernel
//
// Batched over independent problems (bootstrap windows / initialisations),
// with no host round trip: the second solve's descriptor points at the
// device-side compacted offsets and uses the first solve's maxima as bounds.
//
// Exactness: the filter decides, per observation, e <= med + factor * MAD on
// float64 values computed in the reference's operation order without FMA
// contraction (residuals, miniba.py:85-98; np.linalg.norm; np.median as the
// mean of the two middle order statistics), so the kept set is the
// reference's. Order statistics are found by an 8-pass radix select on the
// (monotone) bit patterns of the non-negative values. The gauge scale uses
// numpy's pairwise summation order for the mean of the pairwise distances.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/miniba.h"

namespace mba {
namespace boot {

constexpr int kThreads = 256;

// p = R X + t and the residual, reference order, no FMA contraction
__device__ __forceinline__ double resid_norm(const double* __restrict__ R, const double* __restrict__ t,
                                             const double* __restrict__ X, double f, double cx, double cy,
                                             double u, double v) {
  double p[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    // einsum("kij,kj->ki"): ((R_i0 X_0 + R_i1 X_1) + R_i2 X_2), then + t_i
    double s = __dmul_rn(R[3 * i], X[0]);
    s = __dadd_rn(s, __dmul_rn(R[3 * i + 1], X[1]));
    s = __dadd_rn(s, __dmul_rn(R[3 * i + 2], X[2]));
    p[i] = __dadd_rn(s, t[i]);
  }
  double r0, r1;
  if (!(p[2] > 1e-12)) {
    r0 = r1 = 1e6;
  } else {
    // focal * p / z + cx - uv
    r0 = __dadd_rn(__dadd_rn(__ddiv_rn(__dmul_rn(f, p[0]), p[2]), cx), -u);
    r1 = __dadd_rn(__dadd_rn(__ddiv_rn(__dmul_rn(f, p[1]), p[2]), cy), -v);
  }
  return __dsqrt_rn(__dadd_rn(__dmul_rn(r0, r0), __dmul_rn(r1, r1)));
}

// k-th smallest (0-based) of n non-negative doubles key(i), block-wide
template <typename KeyF>
__device__ double radix_select(int n, int k, KeyF key, int* hist) {
  unsigned long long prefix = 0ull, mask = 0ull;
  for (int pass = 7; pass >= 0; --pass) {
    const int sh = 8 * pass;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(key(i));
      if ((b & mask) == prefix) atomicAdd(hist + ((b >> sh) & 255ull), 1);
    }
    __syncthreads();
    __shared__ int s_bucket, s_below;
    if (threadIdx.x == 0) {
      int acc = 0, bk = 255;
      for (int d = 0; d < 256; ++d) {
        if (acc + hist[d] > k) {
          bk = d;
          break;
        }
        acc += hist[d];
      }
      s_bucket = bk;
      s_below = acc;
    }
    __syncthreads();
    prefix |= (unsigned long long)s_bucket << sh;
    mask |= 255ull << sh;
    k -= s_below;
    __syncthreads();
  }
  return __longlong_as_double((long long)prefix);
}

template <typename KeyF>
__device__ double median_of(int n, KeyF key, int* hist) {
  if (n & 1) return radix_select(n, (n - 1) / 2, key, hist);
  const double a = radix_select(n, n / 2 - 1, key, hist);
  const double b = radix_select(n, n / 2, key, hist);
  return __ddiv_rn(__dadd_rn(a, b), 2.0);
}

struct FilterArgs {
  int n_problems;
  const int64_t* cam_off;
  const int64_t* pt_off;
  const int64_t* obs_off;
  const MbaObs* obs;
  const float* obs_lo;
  const double* cx;
  const double* cy;
  const double* R;       // state after the first solve
  const double* t;
  const double* focal;
  const double* points;
  double factor;
  double* e;             // [total obs] scratch
  int32_t* count;        // [total points] scratch
  uint8_t* keep;         // [total obs]
  int64_t* n_kept;       // [n_problems]
  uint8_t* pt_alive;     // [total points]
};

__global__ void __launch_bounds__(kThreads) filter_kernel(FilterArgs A) {
  __shared__ int hist[256];
  const int b = blockIdx.x;
  if (b >= A.n_problems) return;
  const int64_t ob = A.obs_off[b], cb = A.cam_off[b], pb = A.pt_off[b];
  const int K = (int)(A.obs_off[b + 1] - ob);
  const int P = (int)(A.pt_off[b + 1] - pb);
  const double f = A.focal[b], cx = A.cx[b], cy = A.cy[b];
  double* e = A.e + ob;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const MbaObs o = A.obs[ob + k];
    double u = (double)o.u, v = (double)o.v;
    if (A.obs_lo) {
      u += (double)A.obs_lo[2 * (ob + k)];
      v += (double)A.obs_lo[2 * (ob + k) + 1];
    }
    e[k] = resid_norm(A.R + 9 * (cb + o.cam), A.t + 3 * (cb + o.cam), A.points + 3 * (pb + o.pt), f, cx, cy, u, v);
  }
  for (int p = threadIdx.x; p < P; p += blockDim.x) A.count[pb + p] = 0;
  __syncthreads();
  // robust_filter (miniba.py:57-62): e <= median + factor * median(|e - median|)
  const double med = median_of(K, [&](int i) { return e[i]; }, hist);
  const double mad = median_of(K, [&](int i) { return fabs(__dadd_rn(e[i], -med)); }, hist);
  const double thr = __dadd_rn(med, __dmul_rn(A.factor, mad));
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const bool kk = e[k] <= thr;
    A.keep[ob + k] = kk;
    if (kk) atomicAdd(A.count + pb + A.obs[ob + k].pt, 1);
  }
  __syncthreads();
  // a point needs >= 2 surviving observations to stay constrained
  int kept = 0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const bool kk = A.keep[ob + k] && A.count[pb + A.obs[ob + k].pt] >= 2;
    A.keep[ob + k] = kk;
    kept += kk;
  }
  for (int p = threadIdx.x; p < P; p += blockDim.x) A.pt_alive[pb + p] = A.count[pb + p] >= 2;
  // block total of the survivors (fixed order: warp sums, then warps in order)
  __shared__ int s_wk[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kept += __shfl_xor_sync(0xffffffffu, kept, o);
  if ((threadIdx.x & 31) == 0) s_wk[threadIdx.x >> 5] = kept;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < kThreads / 32; ++w) tot += s_wk[w];
    A.n_kept[b] = tot;
  }
}

// obs_off2 = exclusive scan of n_kept (one block)
__global__ void __launch_bounds__(1024) scan_kernel(int n, const int64_t* __restrict__ n_kept,
                                                    int64_t* __restrict__ off) {
  __shared__ long long warp_tot[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base <= n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const long long v = i < n ? n_kept[i] : 0;
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

// stable compaction of the kept records (order preserved: still point-major)
__global__ void __launch_bounds__(kThreads) compact_kernel(int n_problems, const int64_t* __restrict__ obs_off,
                                                           const int64_t* __restrict__ obs_off2,
                                                           const uint8_t* __restrict__ keep,
                                                           const MbaObs* __restrict__ obs,
                                                           const float2* __restrict__ lo, MbaObs* __restrict__ obs2,
                                                           float2* __restrict__ lo2) {
  __shared__ int warp_tot[kThreads / 32];
  const int b = blockIdx.x;
  if (b >= n_problems) return;
  const int64_t ob = obs_off[b], o2 = obs_off2[b];
  const int K = (int)(obs_off[b + 1] - ob);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int carry = 0;
  for (int base = 0; base < K; base += kThreads) {
    const int k = base + threadIdx.x;
    const int f = k < K ? keep[ob + k] : 0;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) warp_tot[wid] = __popc(m);
    __syncthreads();
    int pre = carry, tot = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      if (w < wid) pre += warp_tot[w];
      tot += warp_tot[w];
    }
    if (f) {
      const int dst = pre + __popc(m & ((1u << lane) - 1u));
      obs2[o2 + dst] = obs[ob + k];
      if (lo) lo2[o2 + dst] = lo[ob + k];
    }
    carry += tot;
    __syncthreads();
  }
}

// gauge: t, points *= 1 / mean pairwise camera-centre distance (miniba.py:797-804)
__global__ void gauge_kernel(int n_problems, const int64_t* __restrict__ cam_off, const int64_t* __restrict__ pt_off,
                             double* __restrict__ R, double* __restrict__ t, double* __restrict__ X,
                             double* __restrict__ scale_out) {
  const int b = blockIdx.x;
  if (b >= n_problems) return;
  const int64_t cb = cam_off[b], pb = pt_off[b];
  const int n = (int)(cam_off[b + 1] - cb);
  const int P = (int)(pt_off[b + 1] - pb);
  __shared__ double s_inv;
  __shared__ int s_apply;
  if (threadIdx.x == 0) {
    // centres: einsum("nji,nj->ni", R, -t)
    double c[64][3];
    const int nn = n < 64 ? n : 64;   // bootstrap windows are cfg.n_init (8) frames
    for (int i = 0; i < nn; ++i)
      for (int a = 0; a < 3; ++a) {
        const double* Ri = R + 9 * (cb + i);
        const double* ti = t + 3 * (cb + i);
        double s = __dmul_rn(Ri[a], -ti[0]);
        s = __dadd_rn(s, __dmul_rn(Ri[3 + a], -ti[1]));
        c[i][a] = __dadd_rn(s, __dmul_rn(Ri[6 + a], -ti[2]));
      }
    // np.mean of the pairwise distances with numpy's summation order
    // (pairwise_sum: fewer than 8 values summed in order; up to 128 values
    // eight interleaved partial sums combined as ((r0+r1)+(r2+r3))+((r4+r5)+
    // (r6+r7)), then the remaining values added one by one); up to 16 cameras
    // (120 pairs) exactly, beyond that in plain order
    constexpr int kMaxPairs = 120;
    double dist[kMaxPairs];
    int m = 0;
    double seq = 0.0;
    const int npairs = nn * (nn - 1) / 2;
    for (int i = 0; i < nn; ++i)
      for (int j = i + 1; j < nn; ++j, ++m) {
        const double d0 = __dadd_rn(c[i][0], -c[j][0]), d1 = __dadd_rn(c[i][1], -c[j][1]),
                     d2 = __dadd_rn(c[i][2], -c[j][2]);
        const double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
        if (m < kMaxPairs) dist[m] = d;
        seq = __dadd_rn(seq, d);
      }
    double sum = seq;
    if (npairs >= 8 && npairs <= kMaxPairs) {
      double r[8];
      for (int q = 0; q < 8; ++q) r[q] = dist[q];
      int i = 8;
      for (; i < npairs - npairs % 8; i += 8)
        for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], dist[i + q]);
      sum = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      for (; i < npairs; ++i) sum = __dadd_rn(sum, dist[i]);
    }
    const double mean_d = npairs > 0 ? __ddiv_rn(sum, (double)npairs) : 0.0;
    s_apply = mean_d > 1e-12;
    s_inv = s_apply ? __ddiv_rn(1.0, mean_d) : 1.0;
    if (scale_out) scale_out[b] = mean_d;
  }
  __syncthreads();
  if (!s_apply) return;
  const double inv = s_inv;
  for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) t[3 * cb + i] = __dmul_rn(t[3 * cb + i], inv);
  for (int i = threadIdx.x; i < 3 * P; i += blockDim.x) X[3 * pb + i] = __dmul_rn(X[3 * pb + i], inv);
}

}  // namespace boot
}  // namespace mba

extern "C" {

size_t mba_bootstrap_workspace_bytes(const MbaBatchDesc* d, const MbaLmConfig* cfg1) {
  (void)cfg1;
  // e (8 B per observation), keep (1 B), counts (4 B per point): sized from the
  // descriptor maxima, which bound every problem
  const size_t K = (size_t)d->max_obs * (size_t)d->n_problems, P = (size_t)d->max_points * (size_t)d->n_problems;
  const size_t al = [](size_t x) { return (x + 255) & ~(size_t)255; }(8 * K) + ((K + 255) & ~(size_t)255) +
                    ((4 * P + 255) & ~(size_t)255);
  return al + mba_workspace_bytes(d, cfg1) + 1024;
}

int32_t mba_bootstrap_schedule(const MbaBatchDesc* d, const MbaLmConfig* cfg1, const MbaLmConfig* cfg2,
                               double mad_factor, const MbaOutputs* out1, const MbaOutputs* out2,
                               MbaObs* obs2, float* obs_lo2, int64_t* obs_off2, int64_t* n_kept,
                               uint8_t* pt_alive, double* gauge_scale, void* ws, size_t ws_bytes,
                               void* stream) {
  if (!d || !cfg1 || !cfg2 || !out1 || !out2 || !obs2 || !obs_off2 || !n_kept || !pt_alive || !ws)
    return MBA_ERR_INVALID;
  if (d->n_problems == 0) return MBA_OK;
  if (out2->R_in != out1->R_out || out2->t_in != out1->t_out || out2->focal_in != out1->focal_out ||
      out2->points_in != out1->points_out)
    return MBA_ERR_INVALID;   // the second half continues from the first half's state
  cudaStream_t st = (cudaStream_t)stream;
  const size_t need = mba_bootstrap_workspace_bytes(d, cfg1);
  if (ws_bytes < need) return MBA_ERR_INVALID;
  const size_t K = (size_t)d->max_obs * (size_t)d->n_problems, P = (size_t)d->max_points * (size_t)d->n_problems;
  unsigned char* w = (unsigned char*)ws;
  double* e = (double*)w;
  w += (8 * K + 255) & ~(size_t)255;
  uint8_t* keep = (uint8_t*)w;
  w += (K + 255) & ~(size_t)255;
  int32_t* count = (int32_t*)w;
  w += (4 * P + 255) & ~(size_t)255;
  const size_t solve_ws = ws_bytes - (size_t)(w - (unsigned char*)ws);
  int32_t rc = mba_solve(d, cfg1, out1, w, solve_ws, stream);
  if (rc != MBA_OK) return rc;
  mba::boot::FilterArgs A;
  A.n_problems = d->n_problems;
  A.cam_off = d->cam_off;
  A.pt_off = d->pt_off;
  A.obs_off = d->obs_off;
  A.obs = d->obs;
  A.obs_lo = d->obs_lo;
  A.cx = d->cx;
  A.cy = d->cy;
  A.R = out1->R_out;
  A.t = out1->t_out;
  A.focal = out1->focal_out;
  A.points = out1->points_out;
  A.factor = mad_factor;
  A.e = e;
  A.count = count;
  A.keep = keep;
  A.n_kept = n_kept;
  A.pt_alive = pt_alive;
  mba::boot::filter_kernel<<<d->n_problems, mba::boot::kThreads, 0, st>>>(A);
  mba::boot::scan_kernel<<<1, 1024, 0, st>>>(d->n_problems, n_kept, obs_off2);
  mba::boot::compact_kernel<<<d->n_problems, mba::boot::kThreads, 0, st>>>(
      d->n_problems, d->obs_off, obs_off2, keep, d->obs, reinterpret_cast<const float2*>(d->obs_lo), obs2,
      reinterpret_cast<float2*>(obs_lo2));
  if (cudaGetLastError() != cudaSuccess) return MBA_ERR_CUDA;
  MbaBatchDesc d2 = *d;
  d2.obs = obs2;
  d2.obs_off = obs_off2;
  d2.obs_lo = d->obs_lo ? obs_lo2 : nullptr;
  // a problem whose filter removed every observation is reported by n_kept
  // (the host raises BootstrapFailure); the solver sees it as empty and
  // returns it unchanged
  rc = mba_solve(&d2, cfg2, out2, w, solve_ws, stream);
  if (rc != MBA_OK) return rc;
  mba::boot::gauge_kernel<<<d->n_problems, 256, 0, st>>>(d->n_problems, d->cam_off, d->pt_off, out2->R_out,
                                                        out2->t_out, out2->points_out, gauge_scale);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}

}  // extern "C"
