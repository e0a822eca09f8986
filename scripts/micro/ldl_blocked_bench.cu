// Microbenchmark: blocked LDL^T of the packed augmented reduced camera system
// (C = 187: config 5's 31 free cameras + focal) in shared memory, one CTA of
// 256 threads, clock64 per sub-phase (diagonal block / panel rows / trailing
// update). Variants of the trailing update:
//   V0  lane = one row, 16 columns per warp tile (L broadcast from staging)
//   V1  lane = 4 rows x 4 columns (W and L staged, two 16-B loads per column)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ldl_blocked_bench.cu -o ldl_blocked_bench
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

__host__ __device__ __forceinline__ int acol(int j, int C) { return j * (C + 1) - (j * (j - 1)) / 2; }

constexpr int NT = 256, NW = NT / 32, PW = 8;

template <typename T, int V>
__global__ void __launch_bounds__(NT, 1) bench(const T* __restrict__ Ain, int C, int reps, long long* cyc, T* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int CA = C * (C + 3) / 2;
  const int LSTR = ((C + 1 + 15) / 16) * 16 + 32;
  T* S = (T*)smem;
  T* invd = S + ((CA + 15) / 16) * 16;
  T* lst = invd + 256;
  T* wst = lst + PW * LSTR;
  __shared__ T s_ltop[PW * PW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  long long c1 = 0, c2 = 0, c3 = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = tid; i < CA; i += NT) S[i] = Ain[i];
    __syncthreads();
    long long t = clock64();
    for (int k = 0; k < C; k += PW) {
      const int w = C - k < PW ? C - k : PW;
      if (wid == 0) {
        const int rr = lane;
        T a[PW];
#pragma unroll
        for (int c = 0; c < PW; ++c) a[c] = (rr < w && c <= rr) ? S[acol(k + c, C) + rr - c] : T(0);
#pragma unroll
        for (int p = 0; p < PW; ++p) {
          if (p < w) {
            const T d = __shfl_sync(0xffffffffu, a[p], p);
            const T inv = T(1) / d;
            const T l = a[p] * inv;
#pragma unroll
            for (int c = p + 1; c < PW; ++c) {
              const T lc = __shfl_sync(0xffffffffu, l, c);
              if (rr > p && c <= rr) a[c] = a[c] - a[p] * lc;
            }
            if (rr > p && rr < w) s_ltop[rr * PW + p] = l;
            if (rr == p) invd[k + p] = inv;
          }
        }
#pragma unroll
        for (int c = 0; c < PW; ++c)
          if (rr < w && c <= rr) S[acol(k + c, C) + rr - c] = a[c];
      }
      __syncthreads();
      if (tid == 0) { long long n = clock64(); c1 += n - t; t = n; }
      const int j0s = k + w;
      for (int i = j0s + tid; i <= C; i += NT) {
        T x[PW];
#pragma unroll
        for (int p = 0; p < PW; ++p)
          if (p < w) x[p] = S[acol(k + p, C) + i - (k + p)];
#pragma unroll
        for (int p = 1; p < PW; ++p)
#pragma unroll
          for (int q = 0; q < p; ++q)
            if (p < w) x[p] = x[p] - x[q] * s_ltop[p * PW + q];
#pragma unroll
        for (int p = 0; p < PW; ++p)
          if (p < w) {
            S[acol(k + p, C) + i - (k + p)] = x[p];
            lst[p * LSTR + i] = x[p] * invd[k + p];
            if (V == 1 || V == 4) wst[p * LSTR + i] = x[p];
          }
      }
      __syncthreads();
      if (tid == 0) { long long n = clock64(); c2 += n - t; t = n; }
      const int m = C + 1 - j0s;
      if (m >= 2) {
        const int nrb = (m + 31) >> 5, ncb = (m - 1 + 15) >> 4;
        int ntile = 0;
        for (int rb = 0; rb < nrb; ++rb) ntile += min(ncb, 2 * rb + 2);
        for (int tl = wid; tl < ntile; tl += NW) {
          int rb = 0, tt = tl;
          for (;;) {
            const int nc = min(ncb, 2 * rb + 2);
            if (tt < nc) break;
            tt -= nc;
            ++rb;
          }
          if constexpr (V != 1) {
            const int i = j0s + 32 * rb + lane, j0 = j0s + 16 * tt;
            const bool row_ok = i <= C;
            const int a0 = acol(j0, C) + i - j0;
            T acc[16];
            {
              int a = a0;
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                const int j = j0 + c;
                acc[c] = (row_ok && j <= i && j < C) ? S[a] : T(0);
                a += C - j;
              }
            }
            for (int p = 0; p < w; ++p) {
              const T wi = row_ok ? S[acol(k + p, C) + i - (k + p)] : T(0);
              const T* lp = lst + p * LSTR + j0;
#pragma unroll
              for (int c = 0; c < 16; c += 2) {
                if constexpr (V == 2) {
                  acc[c] = acc[c] - wi * lp[c];
                  acc[c + 1] = acc[c + 1] - wi * lp[c + 1];
                } else if constexpr (V == 3) {   // calibration: no L loads
                  acc[c] = acc[c] - wi * acc[15 - c];
                  acc[c + 1] = acc[c + 1] - wi * acc[14 - c];
                } else {
                  const double2 v = *reinterpret_cast<const double2*>(lp + c);
                  acc[c] = acc[c] - wi * v.x;
                  acc[c + 1] = acc[c + 1] - wi * v.y;
                }
              }
            }
            {
              int a = a0;
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                const int j = j0 + c;
                if (row_ok && j <= i && j < C) S[a] = acc[c];
                a += C - j;
              }
            }
          } else {
            // lane (ry = lane & 7, cx = lane >> 3): rows i0..i0+3, columns c0..c0+3
            const int ry = lane & 7, cx = lane >> 3;
            const int i0 = j0s + 32 * rb + 4 * ry, c0 = j0s + 16 * tt + 4 * cx;
            T acc[4][4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int j = c0 + jj;
              const int a = acol(j, C) - j;
#pragma unroll
              for (int ii = 0; ii < 4; ++ii) {
                const int i = i0 + ii;
                acc[ii][jj] = (i <= C && j <= i && j < C) ? S[a + i] : T(0);
              }
            }
#pragma unroll 2
            for (int p = 0; p < w; ++p) {
              const double2 wa = *reinterpret_cast<const double2*>(wst + p * LSTR + i0);
              const double2 wb = *reinterpret_cast<const double2*>(wst + p * LSTR + i0 + 2);
              const double2 la = *reinterpret_cast<const double2*>(lst + p * LSTR + c0);
              const double2 lb = *reinterpret_cast<const double2*>(lst + p * LSTR + c0 + 2);
              const T wv[4] = {wa.x, wa.y, wb.x, wb.y}, lv[4] = {la.x, la.y, lb.x, lb.y};
#pragma unroll
              for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = acc[ii][jj] - wv[ii] * lv[jj];
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int j = c0 + jj;
              const int a = acol(j, C) - j;
#pragma unroll
              for (int ii = 0; ii < 4; ++ii) {
                const int i = i0 + ii;
                if (i <= C && j <= i && j < C) S[a + i] = acc[ii][jj];
              }
            }
          }
        }
      }
      __syncthreads();
      if (tid == 0) { long long n = clock64(); c3 += n - t; t = n; }
    }
  }
  if (tid == 0) {
    cyc[0] = c1 / reps;
    cyc[1] = c2 / reps;
    cyc[2] = c3 / reps;
  }
  for (int i = tid; i < CA; i += NT) out[i] = S[i];
  for (int i = tid; i < C; i += NT) out[CA + i] = invd[i];
}

// V5: lookahead blocked LDL^T. Per panel: row solves (all threads), barrier,
// trailing update (full unroll over the 8 panel columns, W in registers,
// unpredicated interior tiles) during which warp 0 takes tile 0 and then
// factorises the NEXT panel's diagonal block straight from its accumulators,
// barrier. Two barriers per 8 columns, the block factorisation off the
// critical path.
template <int BF, typename T>
__device__ __forceinline__ int block_factor(T a[PW], int w, int lane, int k, T* s_ltop, T* invd) {
  int bad = 0;
  if constexpr (BF == 2) {   // gather the block to lane 0, factorise serially in registers
    T b[PW][PW];
#pragma unroll
    for (int r = 0; r < PW; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) b[r][c] = __shfl_sync(0xffffffffu, a[c], r);
    if (lane == 0) {
#pragma unroll
      for (int p = 0; p < PW; ++p) {
        if (p < w) {
          const T d = b[p][p];
          bad |= !(d > T(0)) || !isfinite((double)d);
          const T inv = __drcp_rn(d);
          invd[k + p] = inv;
          T l[PW];
#pragma unroll
          for (int r = p + 1; r < PW; ++r) {
            l[r] = b[r][p] * inv;
            if (r < w) s_ltop[r * PW + p] = l[r];
          }
#pragma unroll
          for (int r = p + 1; r < PW; ++r)
#pragma unroll
            for (int c = p + 1; c <= r; ++c) b[r][c] = b[r][c] - l[r] * b[c][p];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < PW; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) {
        const T v = __shfl_sync(0xffffffffu, b[r][c], 0);
        if (lane == r) a[c] = v;
      }
    return __shfl_sync(0xffffffffu, bad, 0);
  }
#pragma unroll
  for (int p = 0; p < PW; ++p) {
    if (p < w) {
      const T d = __shfl_sync(0xffffffffu, a[p], p);
      T wc[PW];
#pragma unroll
      for (int c = p + 1; c < PW; ++c) wc[c] = __shfl_sync(0xffffffffu, a[p], c);
      bad |= !(d > T(0)) || !isfinite((double)d);
      T inv;
      if constexpr (BF == 3) {
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"((double)d));
        double e = fma(-(double)d, r, 1.0);
        r = fma(r, e, r);
        e = fma(-(double)d, r, 1.0);
        inv = (T)fma(r, e, r);
      } else {
        inv = BF == 1 ? __drcp_rn(d) : T(1) / d;
      }
      const T l = a[p] * inv;
#pragma unroll
      for (int c = p + 1; c < PW; ++c)
        if (c <= lane) a[c] = a[c] - l * wc[c];
      if (lane > p && lane < w) s_ltop[lane * PW + p] = l;
      if (lane == p) invd[k + p] = inv;
    }
  }
  return bad;
}

template <typename T, int BF, int RPL = 1>
__global__ void __launch_bounds__(NT, 1) bench5(const T* __restrict__ Ain, int C, int reps, long long* cyc, T* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int CA = C * (C + 3) / 2;
  const int LSTR = ((C + 1 + 15) / 16) * 16 + 32;
  T* S = (T*)smem;
  T* invd = S + ((CA + 15) / 16) * 16;
  T* lst = invd + 256;
  __shared__ T s_ltop[PW * PW];
  __shared__ int s_bad;
  __shared__ long long s_busy[NW + 1];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid <= NW) s_busy[tid] = 0;
  long long c1 = 0, c2 = 0, c3 = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = tid; i < CA; i += NT) S[i] = Ain[i];
    __syncthreads();
    long long t = clock64();
    if (wid == 0) {   // prologue: diagonal block of panel 0
      const int w = C < PW ? C : PW;
      T a[PW];
#pragma unroll
      for (int c = 0; c < PW; ++c) a[c] = (lane < w && c <= lane) ? S[acol(c, C) + lane - c] : T(0);
      const int bad = block_factor<BF>(a, w, lane, 0, s_ltop, invd);
#pragma unroll
      for (int c = 0; c < PW; ++c)
        if (lane < w && c <= lane) S[acol(c, C) + lane - c] = a[c];
      if (lane == 0) s_bad = bad;
    }
    __syncthreads();
    if (tid == 0) { long long n = clock64(); c1 += n - t; t = n; }
    for (int k = 0; k < C; k += PW) {
      if (s_bad) break;
      const int w = C - k < PW ? C - k : PW;
      const int j0s = k + w;
      // panel rows
      for (int i = j0s + tid; i <= C; i += NT) {
        T x[PW];
        int b = acol(k, C) - k + i;
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
        b = acol(k, C) - k + i;
#pragma unroll
        for (int p = 0; p < PW; ++p)
          if (p < w) {
            S[b] = x[p];
            lst[p * LSTR + i] = x[p] * invd[k + p];
            b += C - (k + p);
          }
      }
      __syncthreads();
      if (tid == 0) { long long n = clock64(); c2 += n - t; t = n; }
      const int m = C + 1 - j0s;
      if (m >= 2) {   // here w == PW
        constexpr int RB = 32 * RPL;   // rows per warp tile
        const int nrb = (m + RB - 1) / RB, ncb = (m - 1 + 15) >> 4;
        int ntile = 0;
        for (int rb = 0; rb < nrb; ++rb) ntile += min(ncb, (RB / 16) * rb + RB / 16);
        // warp 0: tile 0 (+ next diagonal block); warps 1..NW-1: tiles 1..
        long long tb0 = clock64();
        for (int tl = (wid == 0 ? 0 : wid); tl < ntile; tl += (wid == 0 ? ntile : NW - 1)) {
          int rb = 0, tt = tl;
          for (;;) {
            const int nc = min(ncb, (RB / 16) * rb + RB / 16);
            if (tt < nc) break;
            tt -= nc;
            ++rb;
          }
          const int ib = j0s + RB * rb, j0 = j0s + 16 * tt;
          const bool interior = ib >= j0 + 16 && ib + RB - 1 <= C && j0 + 16 <= C;
          T wv[RPL][PW];
          T acc[RPL][16];
          int a0[RPL];
#pragma unroll
          for (int h = 0; h < RPL; ++h) {
            const int i = ib + 32 * h + lane;
            int b = acol(k, C) - k + (i <= C ? i : C);
#pragma unroll
            for (int p = 0; p < PW; ++p) {
              wv[h][p] = S[b];
              b += C - (k + p);
            }
            a0[h] = acol(j0, C) - j0 + i;
            if (interior) {
#pragma unroll
              for (int c = 0; c < 16; ++c) acc[h][c] = S[a0[h] + c * C - (c * j0 + c * (c - 1) / 2)];
            } else {
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                const int j = j0 + c;
                acc[h][c] = (i <= C && j <= i && j < C) ? S[a0[h] + c * C - (c * j0 + c * (c - 1) / 2)] : T(0);
              }
            }
          }
#pragma unroll
          for (int p = 0; p < PW; ++p) {
            const double2* lp = reinterpret_cast<const double2*>(lst + p * LSTR + j0);
#pragma unroll
            for (int c = 0; c < 16; c += 2) {
              const double2 v = lp[c / 2];
#pragma unroll
              for (int h = 0; h < RPL; ++h) {
                acc[h][c] = acc[h][c] - wv[h][p] * v.x;
                acc[h][c + 1] = acc[h][c + 1] - wv[h][p] * v.y;
              }
            }
          }
#pragma unroll
          for (int h = 0; h < RPL; ++h) {
            const int i = ib + 32 * h + lane;
            if (interior) {
#pragma unroll
              for (int c = 0; c < 16; ++c) S[a0[h] + c * C - (c * j0 + c * (c - 1) / 2)] = acc[h][c];
            } else {
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                const int j = j0 + c;
                if (i <= C && j <= i && j < C) S[a0[h] + c * C - (c * j0 + c * (c - 1) / 2)] = acc[h][c];
              }
            }
          }
          if (tl == 0 && j0s < C) {   // factorise the next panel's diagonal block from acc
            long long tq = clock64();
            const int w2 = C - j0s < PW ? C - j0s : PW;
            T a[PW];
#pragma unroll
            for (int c = 0; c < PW; ++c) a[c] = (lane < w2 && c <= lane) ? acc[0][c] : T(0);
            const int bad = block_factor<BF>(a, w2, lane, j0s, s_ltop, invd);
#pragma unroll
            for (int c = 0; c < PW; ++c)
              if (lane < w2 && c <= lane) S[a0[0] + c * C - (c * j0 + c * (c - 1) / 2)] = a[c];
            if (lane == 0) s_bad = bad;
            if (lane == 0) s_busy[NW] += clock64() - tq;
          }
        }
        if (lane == 0) s_busy[wid] += clock64() - tb0;
      }
      __syncthreads();
      if (tid == 0) { long long n = clock64(); c3 += n - t; t = n; }
    }
  }
  if (tid == 0) {
    cyc[0] = c1 / reps;
    cyc[1] = c2 / reps;
    cyc[2] = c3 / reps;
    for (int q = 0; q <= NW; ++q) cyc[3 + q] = s_busy[q] / reps;
  }
  for (int i = tid; i < CA; i += NT) out[i] = S[i];
  for (int i = tid; i < C; i += NT) out[CA + i] = invd[i];
}

int main(int argc, char** argv) {
  const int C = argc > 1 ? atoi(argv[1]) : 187, CA = C * (C + 3) / 2;
  // SPD system: A = B B^T + C I, augmented with a rhs row
  std::vector<double> full((size_t)C * C), B((size_t)C * C), rhs(C);
  srand(1);
  for (auto& v : B) v = (double)rand() / RAND_MAX - 0.5;
  for (int i = 0; i < C; ++i)
    for (int j = 0; j < C; ++j) {
      double s = 0;
      for (int q = 0; q < C; ++q) s += B[i * C + q] * B[j * C + q];
      full[i * C + j] = s + (i == j ? C : 0);
    }
  for (auto& v : rhs) v = (double)rand() / RAND_MAX - 0.5;
  std::vector<double> A(CA);
  for (int j = 0; j < C; ++j) {
    for (int i = j; i < C; ++i) A[acol(j, C) + i - j] = full[i * C + j];
    A[acol(j, C) + C - j] = rhs[j];
  }
  // CPU solve for reference: Cholesky
  std::vector<double> Lc(full);
  for (int j = 0; j < C; ++j) {
    double d = Lc[j * C + j];
    for (int q = 0; q < j; ++q) d -= Lc[j * C + q] * Lc[j * C + q];
    d = std::sqrt(d);
    Lc[j * C + j] = d;
    for (int i = j + 1; i < C; ++i) {
      double s = Lc[i * C + j];
      for (int q = 0; q < j; ++q) s -= Lc[i * C + q] * Lc[j * C + q];
      Lc[i * C + j] = s / d;
    }
  }
  std::vector<double> y(C), x(C);
  for (int i = 0; i < C; ++i) {
    double s = rhs[i];
    for (int q = 0; q < i; ++q) s -= Lc[i * C + q] * y[q];
    y[i] = s / Lc[i * C + i];
  }
  for (int i = C - 1; i >= 0; --i) {
    double s = y[i];
    for (int q = i + 1; q < C; ++q) s -= Lc[q * C + i] * x[q];
    x[i] = s / Lc[i * C + i];
  }
  double *dA, *dO;
  long long* dc;
  cudaMalloc(&dA, CA * 8);
  cudaMalloc(&dO, (CA + C) * 8);
  cudaMalloc(&dc, 256);
  cudaMemcpy(dA, A.data(), CA * 8, cudaMemcpyHostToDevice);
  const int LSTR = ((C + 1 + 15) / 16) * 16 + 32;
  const size_t sm = (size_t)8 * (((CA + 15) / 16) * 16 + 256 + 2 * PW * (((C + 1 + 15) / 16) * 16 + 32));
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<1, NT, sm>>>(dA, C, 20, dc, dO);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    long long c[12] = {};
    cudaMemcpy(c, dc, 96, cudaMemcpyDeviceToHost);
    std::vector<double> o(CA + C);
    cudaMemcpy(o.data(), dO, (CA + C) * 8, cudaMemcpyDeviceToHost);
    // back substitution D L^T x = y (column oriented, as in the kernels)
    std::vector<double> u(C);
    for (int j = 0; j < C; ++j) u[j] = o[acol(j, C) + C - j];
    for (int k = C - 1; k >= 0; --k) {
      const double xk = u[k] * o[CA + k];
      u[k] = xk;
      for (int j = 0; j < k; ++j) u[j] -= o[acol(j, C) + k - j] * xk;
    }
    double err = 0, nx = 0;
    for (int i = 0; i < C; ++i) { err = fmax(err, fabs(u[i] - x[i])); nx = fmax(nx, fabs(x[i])); }
    printf("%s: block %lld rows %lld trailing %lld total %lld cycles; max|x - x_ref| / max|x| = %.3g\n", name, c[0],
           c[1], c[2], c[0] + c[1] + c[2], err / nx);
    if (c[3]) printf("   trailing busy per warp: %lld %lld %lld %lld %lld %lld %lld %lld; warp-0 block factor %lld\n", c[3], c[4], c[5], c[6], c[7], c[8], c[9], c[10], c[11]);
  };
  run(bench<double, 0>, "V0 lane=row x16");
  run(bench<double, 1>, "V1 4x4 per lane");
  run(bench<double, 2>, "V2 lane=row, scalar L loads");
  run(bench5<double, 0>, "V5 lookahead, unrolled, interior fast path");
  run(bench5<double, 0, 2>, "V6 = V5 with 2 rows per lane");
  run(bench5<double, 3>, "V5 + MUFU-seeded Newton reciprocal");
  run(bench<double, 3>, "V3 calibration (no L loads, wrong result)");
  return 0;
}
