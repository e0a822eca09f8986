// mba_common.cuh -- device helpers shared by the mini-BA kernels (sm_100a).
//
// Geometry and loss conventions follow the reference exactly:
//   projection / behind-camera rule   miniba.py:85-98
//   Huber cost and IRLS weight        miniba.py:46-54 (+ Cauchy extension)
//   Jacobian blocks (left perturbation R <- exp(w) R)  miniba.py:101-132
//   Rodrigues with small-angle series scene.py:126-135
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/miniba.h"

namespace mba {

constexpr double kLambdaMax = 1e10;    // miniba.py:23
constexpr double kDiagFloor = 1e-12;   // miniba.py:24
constexpr int kBacktrackTries = 5;     // miniba.py:25
constexpr double kZMin = 1e-12;        // miniba.py:91,96
constexpr double kBadResidual = 1e6;   // miniba.py:97

__device__ __forceinline__ double robust_rho(double e, double delta, int loss) {
  if (loss == MBA_LOSS_CAUCHY) {
    double q = e / delta;
    return 0.5 * delta * delta * log1p(q * q);
  }
  return e <= delta ? 0.5 * e * e : delta * (e - 0.5 * delta);
}

__device__ __forceinline__ double robust_w(double e, double delta, int loss) {
  if (loss == MBA_LOSS_CAUCHY) {
    double q = e / delta;
    return 1.0 / (1.0 + q * q);
  }
  return e <= delta ? 1.0 : delta / fmax(e, 1e-300);
}

// Rodrigues: axis-angle -> row-major 3x3 (scene.py:126-135).
__device__ __forceinline__ void exp_so3(const double w[3], double R[9]) {
  double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double K[9];
  double a, b;
  if (th < 1e-12) {
    K[0] = 0.0;   K[1] = -w[2]; K[2] = w[1];
    K[3] = w[2];  K[4] = 0.0;   K[5] = -w[0];
    K[6] = -w[1]; K[7] = w[0];  K[8] = 0.0;
    a = 1.0;
    b = 0.5;
  } else {
    double kx = w[0] / th, ky = w[1] / th, kz = w[2] / th;
    K[0] = 0.0; K[1] = -kz; K[2] = ky;
    K[3] = kz;  K[4] = 0.0; K[5] = -kx;
    K[6] = -ky; K[7] = kx;  K[8] = 0.0;
    a = sin(th);
    b = 1.0 - cos(th);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double kk = K[i * 3 + 0] * K[0 * 3 + j] + K[i * 3 + 1] * K[1 * 3 + j] + K[i * 3 + 2] * K[2 * 3 + j];
      R[i * 3 + j] = (i == j ? 1.0 : 0.0) + a * K[i * 3 + j] + b * kk;
    }
}

__device__ __forceinline__ void matmul33(const double A[9], const double B[9], double C[9]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      C[i * 3 + j] = A[i * 3 + 0] * B[0 * 3 + j] + A[i * 3 + 1] * B[1 * 3 + j] + A[i * 3 + 2] * B[2 * 3 + j];
}

// Camera-frame point and pixel residual in float64 (miniba.py:85-98).
struct Proj {
  double v[3];    // R X
  double pc[3];   // R X + t
  double ru, rv;  // residual
  bool behind;
};

__device__ __forceinline__ Proj project_residual(const double* __restrict__ R,
                                                 const double* __restrict__ t, const double X[3],
                                                 double f, double cx, double cy, double u,
                                                 double vv) {
  Proj o;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    o.pc[i] = R[i * 3 + 0] * X[0] + R[i * 3 + 1] * X[1] + R[i * 3 + 2] * X[2] + t[i];
    o.v[i] = o.pc[i] - t[i];  // R X recovered as p_cam - t, as miniba.py:117 does
  }
  o.behind = !(o.pc[2] > kZMin);
  double z = o.behind ? kZMin : o.pc[2];
  if (o.behind) {
    o.ru = kBadResidual;
    o.rv = kBadResidual;
  } else {
    o.ru = f * o.pc[0] / z + cx - u;
    o.rv = f * o.pc[1] / z + cy - vv;
  }
  return o;
}

// Same as project_residual with one reciprocal instead of two divisions
// (results differ from the reference's (f x)/z by at most 1 ulp).
__device__ __forceinline__ Proj project_residual_fast(const double* __restrict__ R,
                                                      const double* __restrict__ t,
                                                      const double X[3], double f, double cx,
                                                      double cy, double u, double vv) {
  Proj o;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    o.pc[i] = R[i * 3 + 0] * X[0] + R[i * 3 + 1] * X[1] + R[i * 3 + 2] * X[2] + t[i];
    o.v[i] = o.pc[i] - t[i];
  }
  o.behind = !(o.pc[2] > kZMin);
  const double iz = 1.0 / (o.behind ? kZMin : o.pc[2]);
  o.ru = o.behind ? kBadResidual : f * o.pc[0] * iz + cx - u;
  o.rv = o.behind ? kBadResidual : f * o.pc[1] * iz + cy - vv;
  return o;
}

// Jacobian blocks (miniba.py:101-132) in arithmetic type T.
// A: 2x6 [rot | trans], Fb: 2 (focal), Bm: 2x3 (point).
template <typename T>
__device__ __forceinline__ void jac_blocks(const Proj& p, const double* __restrict__ R, double f,
                                           T A[12], T Fb[2], T Bm[6]) {
  if (p.behind) {
#pragma unroll
    for (int i = 0; i < 12; ++i) A[i] = T(0);
    Fb[0] = Fb[1] = T(0);
#pragma unroll
    for (int i = 0; i < 6; ++i) Bm[i] = T(0);
    return;
  }
  double iz = 1.0 / p.pc[2];
  T fz = T(f * iz);
  T j02 = T(-f * p.pc[0] * iz * iz);
  T j12 = T(-f * p.pc[1] * iz * iz);
  T v0 = T(p.v[0]), v1 = T(p.v[1]), v2 = T(p.v[2]);
  // -Jp [v]x with Jp = [[fz,0,j02],[0,fz,j12]], [v]x = [[0,-v2,v1],[v2,0,-v0],[-v1,v0,0]]
  A[0] = -(j02 * (-v1));
  A[1] = -(fz * (-v2) + j02 * v0);
  A[2] = -(fz * v1);
  A[6] = -(fz * v2 + j12 * (-v1));
  A[7] = -(j12 * v0);
  A[8] = -(fz * (-v0));
  A[3] = fz;   A[4] = T(0);  A[5] = j02;
  A[9] = T(0); A[10] = fz;   A[11] = j12;
  Fb[0] = T(p.pc[0] * iz);
  Fb[1] = T(p.pc[1] * iz);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    Bm[j] = fz * T(R[0 * 3 + j]) + j02 * T(R[2 * 3 + j]);
    Bm[3 + j] = fz * T(R[1 * 3 + j]) + j12 * T(R[2 * 3 + j]);
  }
}

// ---- reductions -----------------------------------------------------------

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction of N values per thread; result returned to
// every thread. `scratch` holds (blockDim/32) * N elements.
template <typename T, int N>
__device__ __forceinline__ void block_sum(T (&v)[N], T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < N; ++i) scratch[wid * N + i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T s = T(0);
    for (int w = 0; w < nw; ++w) s += scratch[w * N + i];
    v[i] = s;
  }
  __syncthreads();
}

__host__ __device__ __forceinline__ int64_t tri_idx(int64_t i, int64_t j) {  // packed lower, j <= i
  return i * (i + 1) / 2 + j;
}

template <typename T, int N, int C, int H>
__device__ __forceinline__ void rs_stage(T (&v)[N], int o, bool up) {
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const T lo = v[i];
    T hi = T(0);
    if (H + i < C) hi = v[(H + i) < N ? (H + i) : 0];
    const T send = up ? lo : hi;
    const T keep = up ? hi : lo;
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
  }
}

// Transposed warp reduction of N per-lane values: 5 halving butterfly stages
// (sum(ceil(N/2^s)) shuffles instead of 5N); the total of value i is written to
// out[i] by exactly one lane. Fixed order -> bit-reproducible.
template <typename T, int N, typename F>
__device__ __forceinline__ void warp_reduce_apply(T (&v)[N], int lane, F&& put) {
  constexpr int h0 = (N + 1) / 2, h1 = (h0 + 1) / 2, h2 = (h1 + 1) / 2, h3 = (h2 + 1) / 2,
                h4 = (h3 + 1) / 2;
  rs_stage<T, N, N, h0>(v, 16, lane & 16);
  rs_stage<T, N, h0, h1>(v, 8, lane & 8);
  rs_stage<T, N, h1, h2>(v, 4, lane & 4);
  rs_stage<T, N, h2, h3>(v, 2, lane & 2);
  rs_stage<T, N, h3, h4>(v, 1, lane & 1);
  const int b0 = lane & 1, b1 = (lane >> 1) & 1, b2 = (lane >> 2) & 1, b3 = (lane >> 3) & 1,
            b4 = (lane >> 4) & 1;
#pragma unroll
  for (int j = 0; j < h4; ++j) {
    int i = j + b0 * h4;
    if (i >= h3) continue;
    i += b1 * h3;
    if (i >= h2) continue;
    i += b2 * h2;
    if (i >= h1) continue;
    i += b3 * h1;
    if (i >= h0) continue;
    i += b4 * h0;
    if (i >= N) continue;
    put(i, v[j]);
  }
}
template <typename T, int N>
__device__ __forceinline__ void warp_reduce_to(T (&v)[N], T* out, int lane) {
  warp_reduce_apply(v, lane, [out](int i, T x) { out[i] = x; });
}


}  // namespace mba
