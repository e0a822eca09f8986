// mba_ldl.cuh -- blocked LDL^T of the packed augmented reduced camera system
// in shared memory, for one CTA (solve_step's Schur solve, miniba.py:207-217).
//
// Storage: column-major packed lower triangle of the (C+1) x C augmented
// matrix [S; rhs^T]: column j holds rows j..C at acol(j) (row C = rhs_j).
// On return S[k][k] = d_k, S[i][k] = L_ik d_k, invd[k] = 1/d_k and the rhs row
// holds the forward-substituted y (so D L^T x = y remains).
//
// Right-looking, panels of kLdlPanel = 8 columns, two barriers per panel:
//   rows      one thread per row i >= k+8 solves its 8 panel entries against
//             the factorised diagonal block (W_ip = A_ip - sum_q<p W_iq L_pq),
//             writes them back and stages L_ip = W_ip / d_p in `lst`;
//   trailing  the rank-8 update of rows/columns >= k+8 in warp tiles of 32
//             rows x 16 columns: a lane owns one row (its 8 W values in
//             registers, the 16 S entries of a column block coalesced across
//             the warp), the 16 L values per panel column are broadcast
//             16-byte loads from `lst`; interior tiles run unpredicated.
//             Warp 0 takes tile 0 -- which holds the next panel's diagonal
//             block -- and factorises that block straight from its
//             accumulators (lookahead) while warps 1..NW-1 take the other
//             tiles, so the pivot chain (one reciprocal per column) is off the
//             critical path while trailing work remains.
// Measured (scripts/micro/ldl_blocked_bench.cu, C = 187, one CTA of 256
// threads, f64): 152k cycles vs 268k for the rank-2 unblocked scheme; the
// trailing update is bound by the broadcast L loads in the shared-memory pipe.
#pragma once

#include <cuda_runtime.h>

namespace mba {

constexpr int kLdlPanel = 8;

__host__ __device__ __forceinline__ constexpr int ldl_lstr(int C) { return ((C + 1 + 15) / 16) * 16 + 32; }

// Factorise the (w x w, w <= 8) diagonal block held by lanes 0..w-1 of one warp
// (lane r: a[c] = A[r][c] for c <= r). On return a[c] holds W_rc (c < r) and
// d_r (c == r); s_ltop[r * 8 + c] = L_rc, invd[k + r] = 1 / d_r. Returns
// nonzero (on every lane) when a pivot is not positive and finite.
template <typename T>
__device__ __forceinline__ int ldl_block_factor(T a[kLdlPanel], int w, int lane, int k, T* s_ltop, T* invd) {
  int bad = 0;
#pragma unroll
  for (int p = 0; p < kLdlPanel; ++p) {
    if (p < w) {
      const T d = __shfl_sync(0xffffffffu, a[p], p);
      T wc[kLdlPanel];
#pragma unroll
      for (int c = p + 1; c < kLdlPanel; ++c) wc[c] = __shfl_sync(0xffffffffu, a[p], c);
      bad |= !(d > T(0)) || !isfinite((double)d);
      const T inv = T(1) / d;
      const T l = a[p] * inv;
#pragma unroll
      for (int c = p + 1; c < kLdlPanel; ++c)
        if (c <= lane) a[c] = a[c] - l * wc[c];
      if (lane > p && lane < w) s_ltop[lane * kLdlPanel + p] = l;
      if (lane == p) invd[k + p] = inv;
    }
  }
  return bad;
}

// S(i, j0 + c) relative to S(i, j0): columns shrink by one entry each
__device__ __forceinline__ int ldl_col_step(int c, int j0, int C) { return c * C - (c * j0 + c * (c - 1) / 2); }

// The factorisation. All NT threads of the CTA call it; `lst` holds
// kLdlPanel * ldl_lstr(C) values of T. Returns true when a pivot failed.
template <typename T, int NT>
__device__ bool ldl_blocked(T* S, int C, T* invd, T* lst, T* s_ltop, int* s_bad) {
  constexpr int PW = kLdlPanel, NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int LSTR = ldl_lstr(C);
  if (wid == 0) {   // prologue: diagonal block of panel 0
    const int w = C < PW ? C : PW;
    T a[PW];
#pragma unroll
    for (int c = 0; c < PW; ++c) a[c] = (lane < w && c <= lane) ? S[acol(c, C) + lane - c] : T(0);
    const int bad = ldl_block_factor(a, w, lane, 0, s_ltop, invd);
#pragma unroll
    for (int c = 0; c < PW; ++c)
      if (lane < w && c <= lane) S[acol(c, C) + lane - c] = a[c];
    if (lane == 0) *s_bad = bad;
  }
  __syncthreads();
  for (int k = 0; k < C; k += PW) {
    if (*s_bad) return true;
    const int w = C - k < PW ? C - k : PW;
    const int j0s = k + w;
    const int bk = acol(k, C) - k;   // S(i, k) = S[bk + i]; column k+p+1 starts C-(k+p) later
    // ---- panel rows j0s..C ----
    for (int i = j0s + tid; i <= C; i += NT) {
      T x[PW];
      int b = bk + i;
#pragma unroll
      for (int p = 0; p < PW; ++p)
        if (p < w) {
          x[p] = S[b];
          b += C - (k + p);
        }
#pragma unroll
      for (int p = 1; p < PW; ++p)
#pragma unroll
        for (int q = 0; q < p; ++q)
          if (p < w) x[p] = x[p] - x[q] * s_ltop[p * PW + q];
      b = bk + i;
#pragma unroll
      for (int p = 0; p < PW; ++p)
        if (p < w) {
          S[b] = x[p];
          lst[p * LSTR + i] = x[p] * invd[k + p];
          b += C - (k + p);
        }
    }
    __syncthreads();
    // ---- trailing update: rows j0s..C, columns j0s..C-1 (j <= i); here w == PW ----
    const int m = C + 1 - j0s;
    if (m >= 2) {
      const int nrb = (m + 31) >> 5, ncb = (m - 1 + 15) >> 4;
      int ntile = 0;
      for (int rb = 0; rb < nrb; ++rb) ntile += min(ncb, 2 * rb + 2);
      for (int tl = (wid == 0 ? 0 : wid); tl < ntile; tl += (wid == 0 ? ntile : NW - 1)) {
        int rb = 0, tt = tl;
        for (;;) {
          const int nc = min(ncb, 2 * rb + 2);
          if (tt < nc) break;
          tt -= nc;
          ++rb;
        }
        const int ib = j0s + 32 * rb, j0 = j0s + 16 * tt, i = ib + lane;
        const bool interior = ib >= j0 + 16 && ib + 31 <= C && j0 + 16 <= C;
        T wv[PW];
        {
          int b = bk + (i <= C ? i : C);
#pragma unroll
          for (int p = 0; p < PW; ++p) {
            wv[p] = S[b];
            b += C - (k + p);
          }
        }
        const int a0 = acol(j0, C) - j0 + i;
        T acc[16];
        if (interior) {
#pragma unroll
          for (int c = 0; c < 16; ++c) acc[c] = S[a0 + ldl_col_step(c, j0, C)];
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int j = j0 + c;
            acc[c] = (i <= C && j <= i && j < C) ? S[a0 + ldl_col_step(c, j0, C)] : T(0);
          }
        }
#pragma unroll
        for (int p = 0; p < PW; ++p) {
          const T* lp = lst + p * LSTR + j0;
          if constexpr (sizeof(T) == 8) {
#pragma unroll
            for (int c = 0; c < 16; c += 2) {
              const double2 v = *reinterpret_cast<const double2*>(lp + c);
              acc[c] = acc[c] - wv[p] * (T)v.x;
              acc[c + 1] = acc[c + 1] - wv[p] * (T)v.y;
            }
          } else {
#pragma unroll
            for (int c = 0; c < 16; c += 4) {
              const float4 v = *reinterpret_cast<const float4*>(lp + c);
              acc[c] = acc[c] - wv[p] * (T)v.x;
              acc[c + 1] = acc[c + 1] - wv[p] * (T)v.y;
              acc[c + 2] = acc[c + 2] - wv[p] * (T)v.z;
              acc[c + 3] = acc[c + 3] - wv[p] * (T)v.w;
            }
          }
        }
        if (interior) {
#pragma unroll
          for (int c = 0; c < 16; ++c) S[a0 + ldl_col_step(c, j0, C)] = acc[c];
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int j = j0 + c;
            if (i <= C && j <= i && j < C) S[a0 + ldl_col_step(c, j0, C)] = acc[c];
          }
        }
        if (tl == 0) {   // lookahead: the next panel's diagonal block is in lanes 0..7, acc[0..7]
          const int w2 = C - j0s < PW ? C - j0s : PW;
          T a[PW];
#pragma unroll
          for (int c = 0; c < PW; ++c) a[c] = (lane < w2 && c <= lane) ? acc[c] : T(0);
          const int bad = ldl_block_factor(a, w2, lane, j0s, s_ltop, invd);
#pragma unroll
          for (int c = 0; c < PW; ++c)
            if (lane < w2 && c <= lane) S[a0 + ldl_col_step(c, j0, C)] = a[c];
          if (lane == 0) *s_bad = bad;
        }
      }
    }
    __syncthreads();
  }
  return false;
}

// Back substitution D L^T x = y on the factorised system, blocked like the
// factorisation (panels of 8 from the bottom): warp 0 solves the panel's 8 x 8
// unit triangle (x_p = u_p / d_p, u_q -= L_pq d_q x_p), then every thread
// j < k folds the panel's x into its u_j with 8 contiguous loads from column j
// (u_j -= sum_p S(k+p, j) x_{k+p}). `u` is scratch for C values of T; the
// result goes to x_out (double). Two barriers per 8 columns; the column-
// oriented single-warp scheme it replaces spent ~730 cycles per column.
template <typename T, int NT>
__device__ void ldl_backsub(const T* S, int C, const T* invd, T* u, double* x_out) {
  constexpr int PW = kLdlPanel;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int j = tid; j < C; j += NT) u[j] = S[acol(j, C) + C - j];
  __syncthreads();
  for (int k = ((C - 1) / PW) * PW; k >= 0; k -= PW) {
    const int w = C - k < PW ? C - k : PW;
    if (wid == 0) {
      T up = lane < w ? u[k + lane] : T(0);
      const T il = lane < w ? invd[k + lane] : T(0);
      const int bl = acol(k + lane, C) - (k + lane) + k;   // S(k + p, k + lane) = S[bl + p]
#pragma unroll
      for (int p = PW - 1; p >= 0; --p) {
        if (p < w) {
          const T xp = __shfl_sync(0xffffffffu, up * il, p);
          if (lane == p) up = xp;
          if (lane < p) up = up - S[bl + p] * xp;
        }
      }
      if (lane < w) u[k + lane] = up;
    }
    __syncthreads();
    if (k == 0) break;
    T xs[PW];
#pragma unroll
    for (int p = 0; p < PW; ++p) xs[p] = p < w ? u[k + p] : T(0);
    for (int j = tid; j < k; j += NT) {
      const T* col = S + acol(j, C) - j + k;
      T acc = u[j];
#pragma unroll
      for (int p = 0; p < PW; ++p)
        if (p < w) acc = acc - col[p] * xs[p];
      u[j] = acc;
    }
    __syncthreads();
  }
  for (int j = tid; j < C; j += NT) x_out[j] = (double)u[j];
}

}  // namespace mba
