// mba_stages.cu -- float64 stage kernels behind the reference's internal API
// (the functions smoke_miniba.py calls directly). Verification path: simple,
// deterministic, no atomics; the hot path is mba_solve.cu.
//
//   mba_residuals  BaProblem.residuals      miniba.py:85-98
//   mba_robust     huber_cost/huber_weights miniba.py:46-54 (+ Cauchy)
//   mba_blocks     _build_blocks            miniba.py:101-132
//   mba_assemble   _assemble                miniba.py:135-177
//   mba_solve_step solve_step               miniba.py:180-220
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "mba_common.cuh"

namespace mba {

__global__ void residuals_kernel(int64_t K, const double* __restrict__ R, const double* __restrict__ t,
                                 double f, double cx, double cy, const double* __restrict__ X,
                                 const int64_t* __restrict__ cam, const int64_t* __restrict__ pt,
                                 const double* __restrict__ uv, double* r, double* pc, uint8_t* bad) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cam[k], j = pt[k];
    const double Xp[3] = {X[3 * j], X[3 * j + 1], X[3 * j + 2]};
    Proj p = project_residual(R + 9 * c, t + 3 * c, Xp, f, cx, cy, uv[2 * k], uv[2 * k + 1]);
    r[2 * k] = p.ru;
    r[2 * k + 1] = p.rv;
    pc[3 * k] = p.pc[0];
    pc[3 * k + 1] = p.pc[1];
    pc[3 * k + 2] = p.pc[2];
    bad[k] = p.behind;
  }
}

__global__ void robust_kernel(int64_t n, const double* __restrict__ e, double delta, int loss,
                              double* w, double* cost) {
  // one block: weights elementwise, cost by a deterministic block reduction
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = fabs(e[i]);
    if (w) w[i] = robust_w(a, delta, loss);
    acc += robust_rho(a, delta, loss);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0 && cost) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    cost[0] = s;
  }
}

__global__ void blocks_kernel(int64_t K, const double* __restrict__ R, const double* __restrict__ t,
                              double f, const int64_t* __restrict__ cam, const double* __restrict__ pc,
                              const uint8_t* __restrict__ bad, double* A, double* F, double* B) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cam[k];
    Proj p;
    for (int i = 0; i < 3; ++i) {
      p.pc[i] = pc[3 * k + i];
      p.v[i] = p.pc[i] - t[3 * c + i];
    }
    p.behind = bad[k] != 0;
    // _build_blocks clamps z but only zeroes rows flagged bad (miniba.py:106,114,131)
    double a[12], fb[2], bm[6];
    if (p.behind) {
      jac_blocks<double>(p, R + 9 * c, f, a, fb, bm);
    } else {
      Proj q = p;
      q.pc[2] = p.pc[2] > kZMin ? p.pc[2] : kZMin;
      jac_blocks<double>(q, R + 9 * c, f, a, fb, bm);
    }
    for (int i = 0; i < 12; ++i) A[12 * k + i] = a[i];
    F[2 * k] = fb[0];
    F[2 * k + 1] = fb[1];
    for (int i = 0; i < 6; ++i) B[6 * k + i] = bm[i];
  }
}

// V, g_p, Wf: one thread per point over its observations (pt_order/pt_ptr)
__global__ void assemble_points_kernel(int64_t P, int32_t C, const int32_t* __restrict__ slot,
                                       int32_t has_f, const int64_t* __restrict__ cam,
                                       const double* __restrict__ w, const double* __restrict__ r,
                                       const double* __restrict__ A, const double* __restrict__ F,
                                       const double* __restrict__ B, const int64_t* __restrict__ order,
                                       const int64_t* __restrict__ ptr, double* V, double* g_p,
                                       double* Wf) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P; j += (int64_t)gridDim.x * blockDim.x) {
    double v[9] = {0}, g[3] = {0};
    double* W = Wf + j * C * 3;
    for (int64_t q = ptr[j]; q < ptr[j + 1]; ++q) {
      const int64_t k = order[q];
      const double wk = w[k];
      const double* b = B + 6 * k;
      const double wb[6] = {wk * b[0], wk * b[1], wk * b[2], wk * b[3], wk * b[4], wk * b[5]};
      for (int a = 0; a < 3; ++a) {
        for (int c = 0; c < 3; ++c) v[a * 3 + c] += b[a] * wb[c] + b[3 + a] * wb[3 + c];
        g[a] += wb[a] * r[2 * k] + wb[3 + a] * r[2 * k + 1];
      }
      const int s = slot[cam[k]];
      if (s >= 0) {
        const double* ak = A + 12 * k;
        for (int rr = 0; rr < 6; ++rr) {
          const double wa0 = wk * ak[rr], wa1 = wk * ak[6 + rr];
          for (int c = 0; c < 3; ++c) W[(6 * s + rr) * 3 + c] += wa0 * b[c] + wa1 * b[3 + c];
        }
      }
      if (has_f) {
        const double wf0 = wk * F[2 * k], wf1 = wk * F[2 * k + 1];
        for (int c = 0; c < 3; ++c) W[(C - 1) * 3 + c] += wf0 * b[c] + wf1 * b[3 + c];
      }
    }
    for (int i = 0; i < 9; ++i) V[9 * j + i] = v[i];
    for (int i = 0; i < 3; ++i) g_p[3 * j + i] = g[i];
  }
}

// U, g_c: one block per free camera (+ one block for the focal terms)
__global__ void assemble_cams_kernel(int32_t nf, int32_t C, const int32_t* __restrict__ cam_of_slot,
                                     int32_t has_f, int64_t K, const double* __restrict__ w,
                                     const double* __restrict__ r, const double* __restrict__ A,
                                     const double* __restrict__ F, const int64_t* __restrict__ order,
                                     const int64_t* __restrict__ ptr, double* U, double* g_c) {
  __shared__ double red[8][48];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double acc[48];
  for (int i = 0; i < 48; ++i) acc[i] = 0.0;
  const int s = blockIdx.x;
  if (s < nf) {
    const int c = cam_of_slot[s];
    for (int64_t q = ptr[c] + threadIdx.x; q < ptr[c + 1]; q += blockDim.x) {
      const int64_t k = order[q];
      const double wk = w[k];
      const double* a = A + 12 * k;
      for (int i = 0; i < 6; ++i) {
        const double wa0 = wk * a[i], wa1 = wk * a[6 + i];
        for (int j = 0; j < 6; ++j) acc[i * 6 + j] += wa0 * a[j] + wa1 * a[6 + j];
        acc[36 + i] += wa0 * r[2 * k] + wa1 * r[2 * k + 1];
        acc[42 + i] += wa0 * F[2 * k] + wa1 * F[2 * k + 1];
      }
    }
  } else {
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
      const double wk = w[k], f0 = F[2 * k], f1 = F[2 * k + 1];
      acc[0] += wk * (f0 * f0 + f1 * f1);
      acc[1] += wk * (f0 * r[2 * k] + f1 * r[2 * k + 1]);
    }
  }
  for (int i = 0; i < 48; ++i) {
    double v = warp_sum(acc[i]);
    if (lane == 0) red[wid][i] = v;
  }
  __syncthreads();
  if (threadIdx.x < 48) {
    double v = 0.0;
    for (int ww = 0; ww < nw; ++ww) v += red[ww][threadIdx.x];
    red[0][threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (s < nf) {
    for (int i = 0; i < 6; ++i) {
      for (int j = 0; j < 6; ++j) U[(6 * s + i) * C + 6 * s + j] = red[0][i * 6 + j];
      g_c[6 * s + i] = red[0][36 + i];
      if (has_f) {
        U[(6 * s + i) * C + C - 1] = red[0][42 + i];
        U[(C - 1) * C + 6 * s + i] = red[0][42 + i];
      }
    }
  } else if (has_f) {
    U[(C - 1) * C + C - 1] = red[0][0];
    g_c[C - 1] = red[0][1];
  }
}

// ---- solve_step ------------------------------------------------------------

// Vinv (3x3 via adjugate, as np.linalg.inv) and T = Wf Vinv: one thread per point
__global__ void schur_prep_kernel(int32_t C, int64_t P, const double* __restrict__ V,
                                  const double* __restrict__ Wf, double lam, double* Vinv,
                                  double* Tm) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P; j += (int64_t)gridDim.x * blockDim.x) {
    double m[9];
    for (int i = 0; i < 9; ++i) m[i] = V[9 * j + i];
    for (int d = 0; d < 3; ++d) m[4 * d] += lam * fmax(V[9 * j + 4 * d], kDiagFloor);
    const double c00 = m[4] * m[8] - m[5] * m[7], c01 = m[5] * m[6] - m[3] * m[8],
                 c02 = m[3] * m[7] - m[4] * m[6];
    const double det = m[0] * c00 + m[1] * c01 + m[2] * c02;
    const double id = 1.0 / det;
    double inv[9] = {c00 * id, (m[2] * m[7] - m[1] * m[8]) * id, (m[1] * m[5] - m[2] * m[4]) * id,
                     c01 * id, (m[0] * m[8] - m[2] * m[6]) * id, (m[2] * m[3] - m[0] * m[5]) * id,
                     c02 * id, (m[1] * m[6] - m[0] * m[7]) * id, (m[0] * m[4] - m[1] * m[3]) * id};
    for (int i = 0; i < 9; ++i) Vinv[9 * j + i] = inv[i];
    for (int a = 0; a < C; ++a) {
      const double* w = Wf + (j * C + a) * 3;
      for (int e = 0; e < 3; ++e)
        Tm[(j * C + a) * 3 + e] = w[0] * inv[e] + w[1] * inv[3 + e] + w[2] * inv[6 + e];
    }
  }
}

// S = Ud - sum_p T_p Wf_p^T ; rhs = -g_c + sum_p T_p g_p. One thread per (a, b) entry.
__global__ void schur_reduce_kernel(int32_t C, int64_t P, const double* __restrict__ U,
                                    const double* __restrict__ g_c, const double* __restrict__ g_p,
                                    const double* __restrict__ Wf, const double* __restrict__ Tm,
                                    double lam, double* S, double* rhs) {
  const int64_t n = (int64_t)C * (C + 1);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(idx / (C + 1)), b = (int)(idx % (C + 1));
    double acc = 0.0;
    if (b < C) {
      for (int64_t j = 0; j < P; ++j) {
        const double* t = Tm + (j * C + a) * 3;
        const double* w = Wf + (j * C + b) * 3;
        acc += t[0] * w[0] + t[1] * w[1] + t[2] * w[2];
      }
      double u = U[a * C + b];
      if (a == b) u += lam * fmax(U[a * C + a], kDiagFloor);
      S[a * C + b] = u - acc;
    } else {
      for (int64_t j = 0; j < P; ++j) {
        const double* t = Tm + (j * C + a) * 3;
        acc += t[0] * g_p[3 * j] + t[1] * g_p[3 * j + 1] + t[2] * g_p[3 * j + 2];
      }
      rhs[a] = -g_c[a] + acc;
    }
  }
}

// In-place dense Cholesky (lower) + solve of an n x n SPD system in global
// memory by one CTA. status[0] = 1 on a non-positive pivot.
__global__ void dense_cholesky_solve_kernel(int64_t n, double* H, double* b, int* status) {
  __shared__ int fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) fail = 0;
  __syncthreads();
  for (int64_t k = 0; k < n; ++k) {
    if (tid == 0) {
      const double d = H[k * n + k];
      if (!(d > 0.0) || !isfinite(d)) fail = 1;
      else H[k * n + k] = sqrt(d);
    }
    __syncthreads();
    if (fail) break;
    const double dk = H[k * n + k];
    for (int64_t i = k + 1 + tid; i < n; i += nt) H[i * n + k] /= dk;
    __syncthreads();
    const int64_t m = n - k - 1;
    for (int64_t q = tid; q < m * m; q += nt) {
      const int64_t i = k + 1 + q / m, j = k + 1 + q % m;
      if (j <= i) H[i * n + j] -= H[i * n + k] * H[j * n + k];
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) status[0] = 1;
    return;
  }
  for (int64_t k = 0; k < n; ++k) {
    if (tid == 0) b[k] /= H[k * n + k];
    __syncthreads();
    for (int64_t i = k + 1 + tid; i < n; i += nt) b[i] -= H[i * n + k] * b[k];
    __syncthreads();
  }
  for (int64_t k = n - 1; k >= 0; --k) {
    if (tid == 0) b[k] /= H[k * n + k];
    __syncthreads();
    for (int64_t i = tid; i < k; i += nt) b[i] -= H[k * n + i] * b[k];
    __syncthreads();
  }
  if (tid == 0) status[0] = 0;
}

// dp = Vinv (-g_p - Wf^T dc)
__global__ void backsub_kernel(int32_t C, int64_t P, const double* __restrict__ Vinv,
                               const double* __restrict__ g_p, const double* __restrict__ Wf,
                               const double* __restrict__ dc, double* dp) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P; j += (int64_t)gridDim.x * blockDim.x) {
    double u[3] = {-g_p[3 * j], -g_p[3 * j + 1], -g_p[3 * j + 2]};
    for (int a = 0; a < C; ++a) {
      const double* w = Wf + (j * C + a) * 3;
      for (int d = 0; d < 3; ++d) u[d] -= w[d] * dc[a];
    }
    const double* m = Vinv + 9 * j;
    for (int d = 0; d < 3; ++d) dp[3 * j + d] = m[3 * d] * u[0] + m[3 * d + 1] * u[1] + m[3 * d + 2] * u[2];
  }
}

// full H for the dense verification path (miniba.py:195-205)
__global__ void dense_build_kernel(int32_t C, int64_t P, const double* __restrict__ U,
                                   const double* __restrict__ g_c, const double* __restrict__ V,
                                   const double* __restrict__ g_p, const double* __restrict__ Wf,
                                   double lam, double* H, double* g) {
  const int64_t n = C + 3 * P;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n, j = idx % n;
    double v = 0.0;
    if (i < C && j < C) {
      v = U[i * C + j];
      if (i == j) v += lam * fmax(U[i * C + i], kDiagFloor);
    } else if (i < C) {
      const int64_t p = (j - C) / 3, e = (j - C) % 3;
      v = Wf[(p * C + i) * 3 + e];
    } else if (j < C) {
      const int64_t p = (i - C) / 3, e = (i - C) % 3;
      v = Wf[(p * C + j) * 3 + e];
    } else {
      const int64_t p = (i - C) / 3, q = (j - C) / 3;
      if (p == q) {
        const int64_t a = (i - C) % 3, e = (j - C) % 3;
        v = V[9 * p + 3 * a + e];
        if (a == e) v += lam * fmax(V[9 * p + 4 * a], kDiagFloor);
      }
    }
    H[idx] = v;
    if (j == 0) g[i] = -(i < C ? g_c[i] : g_p[i - C]);
  }
}

static inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 65535) g = 65535;
  return (int)g;
}

}  // namespace mba

using namespace mba;

extern "C" {

int32_t mba_residuals(int64_t K, const double* R, const double* t, double focal, double cx, double cy,
                      const double* points, const int64_t* cam_idx, const int64_t* pt_idx,
                      const double* uv, double* r, double* p_cam, uint8_t* bad, void* stream) {
  if (K <= 0) return MBA_OK;
  residuals_kernel<<<grid_for(K), 256, 0, (cudaStream_t)stream>>>(K, R, t, focal, cx, cy, points,
                                                                  cam_idx, pt_idx, uv, r, p_cam, bad);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}

int32_t mba_robust(int64_t n, const double* e, double delta, int32_t loss, double* w, double* cost,
                   void* stream) {
  robust_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(n, e, delta, loss, w, cost);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}

int32_t mba_blocks(int64_t K, const double* R, const double* t, double focal, const int64_t* cam_idx,
                   const double* p_cam, const uint8_t* bad, double* A, double* F, double* B,
                   void* stream) {
  if (K <= 0) return MBA_OK;
  blocks_kernel<<<grid_for(K), 256, 0, (cudaStream_t)stream>>>(K, R, t, focal, cam_idx, p_cam, bad,
                                                               A, F, B);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}

int32_t mba_assemble(int64_t K, int32_t n_cams, int32_t n_free, int64_t P, const int32_t* slot,
                     const int32_t* cam_of_slot, int32_t optimize_focal, int32_t optimize_points,
                     const int64_t* cam_idx, const double* w, const double* r, const double* A,
                     const double* F, const double* B, const int64_t* pt_order, const int64_t* pt_ptr,
                     const int64_t* cam_order, const int64_t* cam_ptr, double* U, double* g_c,
                     double* V, double* g_p, double* Wf, void* stream) {
  (void)n_cams;
  cudaStream_t st = (cudaStream_t)stream;
  const int32_t C = 6 * n_free + (optimize_focal ? 1 : 0);
  cudaMemsetAsync(U, 0, sizeof(double) * C * C, st);
  cudaMemsetAsync(g_c, 0, sizeof(double) * C, st);
  cudaMemsetAsync(V, 0, sizeof(double) * 9 * P, st);
  cudaMemsetAsync(g_p, 0, sizeof(double) * 3 * P, st);
  cudaMemsetAsync(Wf, 0, sizeof(double) * 3 * C * P, st);
  if (optimize_points && P > 0)
    assemble_points_kernel<<<grid_for(P), 128, 0, st>>>(P, C, slot, optimize_focal, cam_idx, w, r, A,
                                                         F, B, pt_order, pt_ptr, V, g_p, Wf);
  assemble_cams_kernel<<<n_free + 1, 256, 0, st>>>(n_free, C, cam_of_slot, optimize_focal, K, w, r, A,
                                                   F, cam_order, cam_ptr, U, g_c);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}

size_t mba_solve_step_scratch_bytes(int32_t C, int64_t P, int32_t method) {
  if (method == 1) {
    const int64_t n = C + 3 * P;
    return sizeof(double) * (size_t)(n * n + n) + 256;
  }
  return sizeof(double) * (size_t)(9 * P + 3 * C * P + C * C + C) + 256;
}

int32_t mba_solve_step(int32_t C, int64_t P, const double* U, const double* g_c, const double* V,
                       const double* g_p, const double* Wf, double lam, int32_t method, double* dc,
                       double* dp, void* scratch, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int* status = reinterpret_cast<int*>(scratch);
  double* base = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(scratch) + 256);
  int h_status = 0;
  if (method == 1) {
    const int64_t n = C + 3 * P;
    double* H = base;
    double* g = base + n * n;
    dense_build_kernel<<<grid_for(n * n), 256, 0, st>>>(C, P, U, g_c, V, g_p, Wf, lam, H, g);
    dense_cholesky_solve_kernel<<<1, 1024, 0, st>>>(n, H, g, status);
    cudaMemcpyAsync(&h_status, status, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return MBA_ERR_CUDA;
    if (h_status) return MBA_ERR_NOT_PD;
    cudaMemcpyAsync(dc, g, sizeof(double) * C, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(dp, g + C, sizeof(double) * 3 * P, cudaMemcpyDeviceToDevice, st);
    return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
  }
  if (method != 0) return MBA_ERR_INVALID;
  double* Vinv = base;
  double* Tm = Vinv + 9 * P;
  double* S = Tm + 3 * C * P;
  double* rhs = S + C * C;
  if (P > 0) schur_prep_kernel<<<grid_for(P, 128), 128, 0, st>>>(C, P, V, Wf, lam, Vinv, Tm);
  schur_reduce_kernel<<<grid_for((int64_t)C * (C + 1)), 256, 0, st>>>(C, P, U, g_c, g_p, Wf, Tm, lam, S, rhs);
  dense_cholesky_solve_kernel<<<1, 1024, 0, st>>>(C, S, rhs, status);
  cudaMemcpyAsync(&h_status, status, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return MBA_ERR_CUDA;
  if (h_status) return MBA_ERR_NOT_PD;
  cudaMemcpyAsync(dc, rhs, sizeof(double) * C, cudaMemcpyDeviceToDevice, st);
  if (P > 0) backsub_kernel<<<grid_for(P), 256, 0, st>>>(C, P, Vinv, g_p, Wf, rhs, dp);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}

}  // extern "C"
