// mba_tri.cu -- batched triangulation: triangulate,
// miniba.py:458-530, for many tracks at once, one thread per track.
//
// Per track: rays of every view (camera centre -R^T t, direction
// R^T K^-1 (u, v, 1) normalised), the view pair with the widest angle (first in
// (i, j) order on ties, as the reference's strict comparison), the midpoint of
// the closest points of those two rays, then `gn_steps` Gauss-Newton steps on
// the reprojection error with H = J^T J + 1e-12 I (3x3 solve), and the mean
// reprojection error check. Failures are status codes (the reference raises
// TriangulationFailure with the matching message).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "mba_common.cuh"

namespace mba {

enum { TRI_OK = 0, TRI_FEW = 1, TRI_BASELINE = 2, TRI_PARALLEL = 3, TRI_BEHIND = 4, TRI_REPROJ = 5, TRI_BAD_CAM = 6 };

__device__ __forceinline__ void ray_dir(const double* __restrict__ R, double u, double v, double f, double cx,
                                        double cy, double d[3]) {
  const double x = (u - cx) / f, y = (v - cy) / f;
#pragma unroll
  for (int a = 0; a < 3; ++a) d[a] = R[0 * 3 + a] * x + R[1 * 3 + a] * y + R[2 * 3 + a];
  const double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
#pragma unroll
  for (int a = 0; a < 3; ++a) d[a] /= nrm;
}

__device__ __forceinline__ void centre(const double* __restrict__ R, const double* __restrict__ t, double o[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) o[a] = -(R[0 * 3 + a] * t[0] + R[1 * 3 + a] * t[1] + R[2 * 3 + a] * t[2]);
}

__global__ void __launch_bounds__(128) triangulate_kernel(
    int n_tracks, const int64_t* __restrict__ off, const int32_t* __restrict__ cam,
    const double* __restrict__ uv, int n_cams, const double* __restrict__ Rall, const double* __restrict__ tall, double f,
    double cx, double cy, double max_reproj, double min_angle_deg, int gn_steps, double* __restrict__ X_out,
    int32_t* __restrict__ status, double* __restrict__ err_out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_tracks) return;
  const int64_t o0 = off[k];
  const int n = (int)(off[k + 1] - o0);
  auto fail = [&](int code) {
    status[k] = code;
    X_out[3 * k] = X_out[3 * k + 1] = X_out[3 * k + 2] = nan("");
    if (err_out) err_out[k] = nan("");
  };
  if (n < 2) {
    fail(TRI_FEW);
    return;
  }
  for (int i = 0; i < n; ++i)   // a camera index outside [0, n_cams) never reads R / t
    if (cam[o0 + i] < 0 || cam[o0 + i] >= n_cams) {
      fail(TRI_BAD_CAM);
      return;
    }
  // widest-angle pair (degrees(arccos(clip(|d_i . d_j|))), strict > in (i, j) order)
  double best = -1.0;
  int bi = 0, bj = 1;
  for (int i = 0; i < n; ++i) {
    double di[3];
    ray_dir(Rall + 9 * cam[o0 + i], uv[2 * (o0 + i)], uv[2 * (o0 + i) + 1], f, cx, cy, di);
    for (int j = i + 1; j < n; ++j) {
      double dj[3];
      ray_dir(Rall + 9 * cam[o0 + j], uv[2 * (o0 + j)], uv[2 * (o0 + j) + 1], f, cx, cy, dj);
      double cs = fabs(di[0] * dj[0] + di[1] * dj[1] + di[2] * dj[2]);
      cs = fmin(fmax(cs, -1.0), 1.0);
      const double ang = acos(cs) * (180.0 / M_PI);
      if (ang > best) {
        best = ang;
        bi = i;
        bj = j;
      }
    }
  }
  if (best <= min_angle_deg) {
    fail(TRI_BASELINE);
    return;
  }
  double d1[3], d2[3], c1[3], c2[3];
  const int ci = cam[o0 + bi], cj = cam[o0 + bj];
  ray_dir(Rall + 9 * ci, uv[2 * (o0 + bi)], uv[2 * (o0 + bi) + 1], f, cx, cy, d1);
  ray_dir(Rall + 9 * cj, uv[2 * (o0 + bj)], uv[2 * (o0 + bj) + 1], f, cx, cy, d2);
  centre(Rall + 9 * ci, tall + 3 * ci, c1);
  centre(Rall + 9 * cj, tall + 3 * cj, c2);
  const double a = d1[0] * d1[0] + d1[1] * d1[1] + d1[2] * d1[2];
  const double b = d1[0] * d2[0] + d1[1] * d2[1] + d1[2] * d2[2];
  const double c = d2[0] * d2[0] + d2[1] * d2[1] + d2[2] * d2[2];
  const double w[3] = {c2[0] - c1[0], c2[1] - c1[1], c2[2] - c1[2]};
  const double den = a * c - b * b;
  if (den < 1e-18) {
    fail(TRI_PARALLEL);
    return;
  }
  const double d1w = d1[0] * w[0] + d1[1] * w[1] + d1[2] * w[2];
  const double d2w = d2[0] * w[0] + d2[1] * w[1] + d2[2] * w[2];
  const double s = (c * d1w - b * d2w) / den;
  const double u = (b * d1w - a * d2w) / den;
  double X[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) X[q] = 0.5 * (c1[q] + s * d1[q] + c2[q] + u * d2[q]);

  for (int step = 0; step < gn_steps; ++step) {
    double H[6] = {0, 0, 0, 0, 0, 0};   // 00 10 11 20 21 22
    double g[3] = {0, 0, 0};
    for (int v = 0; v < n; ++v) {
      const double* R = Rall + 9 * cam[o0 + v];
      const double* t = tall + 3 * cam[o0 + v];
      double pc[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) pc[q] = R[3 * q] * X[0] + R[3 * q + 1] * X[1] + R[3 * q + 2] * X[2] + t[q];
      if (pc[2] <= 1e-12) {
        fail(TRI_BEHIND);
        return;
      }
      const double z = pc[2];
      const double fz = f / z, j02 = -f * pc[0] / (z * z), j12 = -f * pc[1] / (z * z);
      double J0[3], J1[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        J0[q] = fz * R[q] + j02 * R[6 + q];
        J1[q] = fz * R[3 + q] + j12 * R[6 + q];
      }
      const double r0 = f * pc[0] / z + cx - uv[2 * (o0 + v)];
      const double r1 = f * pc[1] / z + cy - uv[2 * (o0 + v) + 1];
      H[0] += J0[0] * J0[0] + J1[0] * J1[0];
      H[1] += J0[1] * J0[0] + J1[1] * J1[0];
      H[2] += J0[1] * J0[1] + J1[1] * J1[1];
      H[3] += J0[2] * J0[0] + J1[2] * J1[0];
      H[4] += J0[2] * J0[1] + J1[2] * J1[1];
      H[5] += J0[2] * J0[2] + J1[2] * J1[2];
#pragma unroll
      for (int q = 0; q < 3; ++q) g[q] += J0[q] * r0 + J1[q] * r1;
    }
    H[0] += 1e-12;
    H[2] += 1e-12;
    H[5] += 1e-12;
    // 3x3 symmetric solve H x = g by Cholesky
    const double L00 = sqrt(H[0]);
    const double L10 = H[1] / L00, L20 = H[3] / L00;
    const double L11 = sqrt(H[2] - L10 * L10);
    const double L21 = (H[4] - L20 * L10) / L11;
    const double L22 = sqrt(H[5] - L20 * L20 - L21 * L21);
    const double y0 = g[0] / L00, y1 = (g[1] - L10 * y0) / L11, y2 = (g[2] - L20 * y0 - L21 * y1) / L22;
    const double x2 = y2 / L22, x1 = (y1 - L21 * x2) / L11, x0 = (y0 - L10 * x1 - L20 * x2) / L00;
    X[0] -= x0;
    X[1] -= x1;
    X[2] -= x2;
  }
  double esum = 0.0;
  for (int v = 0; v < n; ++v) {
    const double* R = Rall + 9 * cam[o0 + v];
    const double* t = tall + 3 * cam[o0 + v];
    double pc[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) pc[q] = R[3 * q] * X[0] + R[3 * q + 1] * X[1] + R[3 * q + 2] * X[2] + t[q];
    if (pc[2] <= 1e-12) {
      fail(TRI_BEHIND);
      return;
    }
    const double e0 = f * pc[0] / pc[2] + cx - uv[2 * (o0 + v)];
    const double e1 = f * pc[1] / pc[2] + cy - uv[2 * (o0 + v) + 1];
    esum += sqrt(e0 * e0 + e1 * e1);
  }
  const double mean = esum / n;
  if (mean > max_reproj) {
    fail(TRI_REPROJ);
    return;
  }
  status[k] = TRI_OK;
  X_out[3 * k] = X[0];
  X_out[3 * k + 1] = X[1];
  X_out[3 * k + 2] = X[2];
  if (err_out) err_out[k] = mean;
}

}  // namespace mba

extern "C" int32_t mba_triangulate(int32_t n_tracks, const int64_t* obs_off, const int32_t* cam,
                                   const double* uv, int32_t n_cams, const double* R, const double* t,
                                   double focal, double cx, double cy, double max_reproj_px,
                                   double min_angle_deg, int32_t gn_steps, double* X, int32_t* status,
                                   double* mean_err, void* stream) {
  if (n_tracks < 0 || n_cams < 0 || gn_steps < 0 || !(focal != 0.0)) return MBA_ERR_INVALID;
  if (n_tracks == 0) return MBA_OK;
  if (!obs_off || !cam || !uv || !R || !t || !X || !status) return MBA_ERR_INVALID;
  const int threads = 128;
  const int blocks = (n_tracks + threads - 1) / threads;
  mba::triangulate_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(
      n_tracks, obs_off, cam, uv, n_cams, R, t, focal, cx, cy, max_reproj_px, min_angle_deg, gn_steps, X, status,
      mean_err);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}
