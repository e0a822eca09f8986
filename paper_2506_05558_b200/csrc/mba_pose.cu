// mba_pose.cu -- batched pose-only LM (K6) and RANSAC hypothesis scoring.
//
// Replaces pose_lm (miniba.py:334-389) and the scoring block of
// estimate_pose_ransac (miniba.py:418-431). One warp owns one pose problem
// (a RANSAC hypothesis or the single refine_pose problem): lanes stride over
// the correspondences, the 6x6 normal equations are reduced with fixed-order
// warp butterflies (deterministic), and every lane then solves the damped
// system redundantly in registers. All `iters` iterations run in one launch.
//
// Semantics kept from the reference: Huber IRLS weights times the in-front
// mask (349), Marquardt damping lam*max(diag,1e-12) (371), a single trial per
// iteration with no backtracking (377-386), per-problem lambda (385-386),
// _exp_so3_batch without the small-angle branch (303-316).
// Deviation (documented): the reference's LinAlgError fallback adds 1e-6 to
// the diagonal of EVERY batch member (372-376); here it applies per problem.
// It cannot trigger for lam > 0 because the damped diagonal is strictly
// positive and H is PSD.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "mba_common.cuh"

namespace mba {

__device__ __forceinline__ void exp_so3_batch_form(const double w[3], double R[9]) {
  double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  th = fmax(th, 1e-30);
  const double kx = w[0] / th, ky = w[1] / th, kz = w[2] / th;
  const double K[9] = {0.0, -kz, ky, kz, 0.0, -kx, -ky, kx, 0.0};
  const double a = sin(th), b = 1.0 - cos(th);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double kk = K[i * 3] * K[j] + K[i * 3 + 1] * K[3 + j] + K[i * 3 + 2] * K[6 + j];
      R[i * 3 + j] = (i == j ? 1.0 : 0.0) + a * K[i * 3 + j] + b * kk;
    }
}

__device__ __forceinline__ double pose_cost(const double* R, const double* t, const double* X,
                                            const double* uv, int m, double f, double cx, double cy,
                                            double delta, int lane) {
  double c = 0.0;
  for (int i = lane; i < m; i += 32) {
    const double Xp[3] = {X[3 * i], X[3 * i + 1], X[3 * i + 2]};
    Proj p = project_residual(R, t, Xp, f, cx, cy, uv[2 * i], uv[2 * i + 1]);
    c += robust_rho(hypot(p.ru, p.rv), delta, MBA_LOSS_HUBER);
  }
  return warp_sum(c);
}

// Cholesky solve of a 6x6 SPD system; false if not PD. Fully unrolled (no
// early exit inside the loops) so L, y and x stay in registers.
__device__ __forceinline__ bool chol6_solve(const double H[36], const double g[6], double x[6]) {
  double L[36];
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 36; ++i) L[i] = 0.0;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    double d = H[j * 6 + j];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= L[j * 6 + k] * L[j * 6 + k];
    ok = ok && d > 0.0;
    const double ljj = sqrt(d > 0.0 ? d : 1.0);
    L[j * 6 + j] = ljj;
#pragma unroll
    for (int i = j + 1; i < 6; ++i) {
      double s = H[i * 6 + j];
#pragma unroll
      for (int k = 0; k < j; ++k) s -= L[i * 6 + k] * L[j * 6 + k];
      L[i * 6 + j] = s / ljj;
    }
  }
  double y[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double s = -g[i];
#pragma unroll
    for (int k = 0; k < i; ++k) s -= L[i * 6 + k] * y[k];
    y[i] = s / L[i * 6 + i];
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double s = y[i];
#pragma unroll
    for (int k = i + 1; k < 6; ++k) s -= L[k * 6 + i] * x[k];
    x[i] = s / L[i * 6 + i];
  }
  return ok;
}

__global__ void __launch_bounds__(128) pose_lm_kernel(
    int nb, int m, const double* __restrict__ Xb, const double* __restrict__ uvb, double f, double cx,
    double cy, int iters, double lam0, double nu, double delta, double* Rb, double* tb, double* costb,
    int m_all, const double* __restrict__ X_all, const double* __restrict__ uv_all, double thr,
    int* inliers, double* sse) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nb) return;
  const double* X = Xb + (size_t)b * m * 3;
  const double* uv = uvb + (size_t)b * m * 2;
  double R[9], t[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = Rb[9 * b + i];
#pragma unroll
  for (int i = 0; i < 3; ++i) t[i] = tb[3 * b + i];
  double lam = lam0;
  double cost = pose_cost(R, t, X, uv, m, f, cx, cy, delta, lane);
  for (int itr = 0; itr < iters; ++itr) {
    double acc[27];
#pragma unroll
    for (int i = 0; i < 27; ++i) acc[i] = 0.0;
    for (int i = lane; i < m; i += 32) {
      const double Xp[3] = {X[3 * i], X[3 * i + 1], X[3 * i + 2]};
      Proj p = project_residual(R, t, Xp, f, cx, cy, uv[2 * i], uv[2 * i + 1]);
      if (p.behind) continue;  // weight 0 (miniba.py:349)
      const double w = robust_w(hypot(p.ru, p.rv), delta, MBA_LOSS_HUBER);
      double A[12], Fb[2], Bm[6];
      jac_blocks<double>(p, R, f, A, Fb, Bm);
      int idx = 0;
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double wa0 = w * A[r], wa1 = w * A[6 + r];
#pragma unroll
        for (int c = 0; c <= r; ++c) acc[idx++] += A[c] * wa0 + A[6 + c] * wa1;
        acc[21 + r] += wa0 * p.ru + wa1 * p.rv;
      }
    }
#pragma unroll
    for (int i = 0; i < 27; ++i) acc[i] = warp_sum(acc[i]);
    double H[36], g[6], dx[6];
    int idx = 0;
#pragma unroll
    for (int r = 0; r < 6; ++r) {
#pragma unroll
      for (int c = 0; c <= r; ++c, ++idx) H[r * 6 + c] = H[c * 6 + r] = acc[idx];
      g[r] = acc[21 + r];
    }
#pragma unroll
    for (int d = 0; d < 6; ++d) H[d * 6 + d] += lam * fmax(H[d * 6 + d], kDiagFloor);
    if (!chol6_solve(H, g, dx)) {
#pragma unroll
      for (int d = 0; d < 6; ++d) H[d * 6 + d] += 1e-6;
      if (!chol6_solve(H, g, dx))
#pragma unroll
        for (int d = 0; d < 6; ++d) dx[d] = 0.0;
    }
    double E[9], Rt[9], tt[3];
    exp_so3_batch_form(dx, E);
    matmul33(E, R, Rt);
#pragma unroll
    for (int i = 0; i < 3; ++i) tt[i] = t[i] + dx[3 + i];
    const double ct = pose_cost(Rt, tt, X, uv, m, f, cx, cy, delta, lane);
    if (ct < cost) {
#pragma unroll
      for (int i = 0; i < 9; ++i) R[i] = Rt[i];
#pragma unroll
      for (int i = 0; i < 3; ++i) t[i] = tt[i];
      cost = ct;
      lam = fmax(lam / nu, 1e-15);
    } else {
      lam = fmin(lam * nu, kLambdaMax);
    }
  }
  if (lane == 0) {
    for (int i = 0; i < 9; ++i) Rb[9 * b + i] = R[i];
    for (int i = 0; i < 3; ++i) tb[3 * b + i] = t[i];
    costb[b] = cost;
  }
  if (X_all != nullptr) {
    int cnt = 0;
    double s = 0.0;
    for (int i = lane; i < m_all; i += 32) {
      const double Xp[3] = {X_all[3 * i], X_all[3 * i + 1], X_all[3 * i + 2]};
      Proj p = project_residual(R, t, Xp, f, cx, cy, uv_all[2 * i], uv_all[2 * i + 1]);
      if (p.behind) continue;  // err = inf, never an inlier (miniba.py:425)
      const double e = hypot(p.ru, p.rv);
      if (e < thr) {
        ++cnt;
        s += e * e;
      }
    }
    cnt = warp_sum(cnt);
    s = warp_sum(s);
    if (lane == 0) {
      inliers[b] = cnt;
      sse[b] = s;
    }
  }
}

}  // namespace mba

extern "C" int32_t mba_pose_lm(int32_t nb, int32_t m, const double* X, const double* uv, double focal,
                               double cx, double cy, int32_t iters, double lambda_init, double nu,
                               double delta, double* R, double* t, double* cost, int32_t m_all,
                               const double* X_all, const double* uv_all, double inlier_px,
                               int32_t* inliers, double* inlier_sse, void* stream) {
  if (nb <= 0) return MBA_OK;
  if (m <= 0) return MBA_ERR_INVALID;
  // 4 warps (problems) per CTA: at ~158 registers per thread three CTAs fit
  // an SM (12 warps in flight) where one 8-warp CTA did
  const int warps = 4;
  const int grid = (nb + warps - 1) / warps;
  mba::pose_lm_kernel<<<grid, warps * 32, 0, (cudaStream_t)stream>>>(
      nb, m, X, uv, focal, cx, cy, iters, lambda_init, nu, delta, R, t, cost, m_all, X_all, uv_all,
      inlier_px, inliers, inlier_sse);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}
