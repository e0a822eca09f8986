// Microbenchmark: LDL^T of the packed augmented reduced system (C = 43) in
// shared memory, one CTA of 256 threads, clock64 per factorisation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ldl_bench.cu -o ldl_bench
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

__host__ __device__ __forceinline__ int acol(int j, int C) { return j * (C + 1) - (j * (j - 1)) / 2; }

constexpr int NT = 256;
constexpr int MAXCA = 49 * 52 / 2;

template <typename T, int V>
__global__ void bench(const T* __restrict__ Ain, int C, int reps, long long* cyc, T* out) {
  __shared__ T S[MAXCA], S0[MAXCA], invd[64];
  __shared__ unsigned short tab[MAXCA];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int CA = C * (C + 3) / 2;
  for (int i = tid; i < CA; i += NT) S0[i] = Ain[i];
  for (int j = tid; j < C; j += NT) {
    const int a0 = acol(j, C);
    for (int i = j; i <= C; ++i) tab[a0 + i - j] = (unsigned short)((i << 8) | j);
  }
  __syncthreads();
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = tid; i < CA; i += NT) S[i] = S0[i];
    __syncthreads();
    long long t0 = clock64();
    if constexpr (V == 0) {   // all threads, 1 barrier per column, unrolled x4
      for (int k = 0; k < C; ++k) {
        const T* colk = S + acol(k, C) - k;
        const int e0 = acol(k + 1, C);
        const T d = colk[k];
        for (int eb = e0 + tid; eb < CA; eb += 4 * NT) {
          unsigned ij[4]; T ci[4], cj[4], sv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) ij[u] = eb + u * NT < CA ? tab[eb + u * NT] : 0u;
#pragma unroll
          for (int u = 0; u < 4; ++u) { ci[u] = colk[ij[u] >> 8]; cj[u] = colk[ij[u] & 255u]; sv[u] = eb + u * NT < CA ? S[eb + u * NT] : T(0); }
          const T inv = T(1) / d;
#pragma unroll
          for (int u = 0; u < 4; ++u) if (eb + u * NT < CA) S[eb + u * NT] = sv[u] - ci[u] * cj[u] * inv;
        }
        if (tid == 0) invd[k] = T(1) / d;
        __syncthreads();
      }
    } else if constexpr (V == 1) {  // one warp, syncwarp per column, unrolled x4
      if (wid == 0) {
        for (int k = 0; k < C; ++k) {
          const T* colk = S + acol(k, C) - k;
          const int e0 = acol(k + 1, C);
          const T d = colk[k];
          const T inv = T(1) / d;
          for (int eb = e0 + lane; eb < CA; eb += 4 * 32) {
            unsigned ij[4]; T ci[4], cj[4], sv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) ij[u] = eb + u * 32 < CA ? tab[eb + u * 32] : 0u;
#pragma unroll
            for (int u = 0; u < 4; ++u) { ci[u] = colk[ij[u] >> 8]; cj[u] = colk[ij[u] & 255u]; sv[u] = eb + u * 32 < CA ? S[eb + u * 32] : T(0); }
#pragma unroll
            for (int u = 0; u < 4; ++u) if (eb + u * 32 < CA) S[eb + u * 32] = sv[u] - ci[u] * cj[u] * inv;
          }
          if (lane == 0) invd[k] = inv;
          __syncwarp();
        }
      }
      __syncthreads();
    } else if constexpr (V == 2) {  // one warp, lane = row (rows l, l+32), smem, loop over columns j
      if (wid == 0) {
        const int i0 = lane, i1 = lane + 32;
        for (int k = 0; k < C; ++k) {
          const T* colk = S + acol(k, C) - k;
          const T d = colk[k];
          const T inv = T(1) / d;
          const T l0 = (i0 > k && i0 <= C) ? colk[i0] * inv : T(0);
          const T l1 = (i1 > k && i1 <= C) ? colk[i1] * inv : T(0);
          const int jmax = (i1 <= C ? i1 : (i0 <= C ? i0 : -1));
          // row i updates entries j in (k, min(i, C-1)]
#pragma unroll 4
          for (int j = k + 1; j < C; ++j) {
            const T cjk = colk[j];
            T* colj = S + acol(j, C) - j;
            if (i0 >= j && i0 <= C) colj[i0] -= l0 * cjk;
            if (i1 >= j && i1 <= C) colj[i1] -= l1 * cjk;
          }
          if (lane == 0) invd[k] = inv;
          __syncwarp();
          (void)jmax;
        }
      }
      __syncthreads();
    } else if constexpr (V == 3) {  // all threads, 2 columns per barrier (rank-2 step)
      int k = 0;
      for (; k + 1 < C; k += 2) {
        const T* colk = S + acol(k, C) - k;
        T* colk1 = S + acol(k + 1, C) - (k + 1);
        const T d0 = colk[k];
        const T i0 = T(1) / d0;
        const T l10 = colk[k + 1] * i0;                  // L_{k+1,k}
        const T d1 = colk1[k + 1] - l10 * colk[k + 1];
        const T i1 = T(1) / d1;
        const int e0 = acol(k + 2, C);
        for (int eb = e0 + tid; eb < CA; eb += 2 * NT) {
          unsigned ij[2]; T a[2], b[2], c[2], dd[2], sv[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) ij[u] = eb + u * NT < CA ? tab[eb + u * NT] : 0u;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int i = ij[u] >> 8, j = ij[u] & 255u;
            a[u] = colk[i]; b[u] = colk[j]; c[u] = colk1[i]; dd[u] = colk1[j];
            sv[u] = eb + u * NT < CA ? S[eb + u * NT] : T(0);
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const T ci1 = c[u] - a[u] * l10, cj1 = dd[u] - b[u] * l10;   // column k+1 after step k
            if (eb + u * NT < CA) S[eb + u * NT] = sv[u] - a[u] * b[u] * i0 - ci1 * cj1 * i1;
          }
        }
        __syncthreads();
        // finalise column k+1 (rows k+1..C) -- disjoint from the trailing region
        for (int i = k + 1 + tid; i <= C; i += NT) colk1[i] = (i == k + 1) ? d1 : colk1[i] - colk[i] * l10;
        if (tid == 0) { invd[k] = i0; invd[k + 1] = i1; }
        __syncthreads();
      }
      for (; k < C; ++k) {
        const T* colk = S + acol(k, C) - k;
        const T d = colk[k];
        for (int e = acol(k + 1, C) + tid; e < CA; e += NT) { const unsigned ij = tab[e]; S[e] -= colk[ij >> 8] * colk[ij & 255u] / d; }
        if (tid == 0) invd[k] = T(1) / d;
        __syncthreads();
      }
    } else if constexpr (V == 4) {  // barrier only
      for (int k = 0; k < C; ++k) __syncthreads();
    } else if constexpr (V == 5) {  // LDS -> STS chain + barrier
      for (int k = 0; k < C; ++k) {
        const T d = S[acol(k, C)];
        if (tid < CA) S[(tid + k) % CA] = d + T(1);
        __syncthreads();
      }
    } else if constexpr (V == 6) {  // register-owned entries (5 per thread), publish column k+1
      constexpr int E = 5;
      T v[E]; int ii[E], jj[E], ee[E];
#pragma unroll
      for (int u = 0; u < E; ++u) {
        ee[u] = tid + u * NT;
        const unsigned ij = ee[u] < CA ? tab[ee[u]] : 0u;
        ii[u] = ij >> 8; jj[u] = ij & 255u;
        v[u] = ee[u] < CA ? S[ee[u]] : T(0);
      }
      for (int k = 0; k < C; ++k) {
        const T* colk = S + acol(k, C) - k;
        const T d = colk[k];
        const T inv = T(1) / d;
#pragma unroll
        for (int u = 0; u < E; ++u) {
          if (ee[u] < CA && jj[u] > k) {
            v[u] -= colk[ii[u]] * colk[jj[u]] * inv;
            if (jj[u] == k + 1) S[ee[u]] = v[u];   // publish the next pivot column
          }
        }
        if (tid == 0) invd[k] = inv;
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < E; ++u) if (ee[u] < CA) S[ee[u]] = v[u];
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) cyc[0] = tot / reps;
  for (int i = tid; i < CA; i += NT) out[i] = S[i];
}


// register-resident single-warp LDL^T: lane owns rows l and l+32 (row C = rhs),
// pivot column broadcast by shuffles; CM = compile-time bound on C
template <typename T, int CM>
__device__ __forceinline__ void ldl_regs(T* S, T* invd, int C, int lane) {
  T a[32], b[CM];
  const int i0 = lane, i1 = lane + 32;
#pragma unroll
  for (int j = 0; j < 32; ++j) a[j] = (j <= i0 && i0 <= C && j < C) ? S[acol(j, C) + i0 - j] : T(0);
#pragma unroll
  for (int j = 0; j < CM; ++j) b[j] = (i1 <= C && j <= i1 && j < C) ? S[acol(j, C) + i1 - j] : T(0);
#pragma unroll
  for (int k = 0; k < CM; ++k) {
    if (k >= C) break;
    const T dk = __shfl_sync(0xffffffffu, k < 32 ? a[k < 32 ? k : 0] : b[k], k & 31);
    const T inv = T(1) / dk;
    if (lane == 0) invd[k] = inv;
    const T l0 = (k < 32 && i0 > k) ? a[k < 32 ? k : 0] * inv : T(0);
    const T l1 = (i1 > k) ? b[k] * inv : T(0);
#pragma unroll
    for (int j = k + 1; j < CM; ++j) {
      if (j >= C) break;
      const T cjk = __shfl_sync(0xffffffffu, j < 32 ? a[k < 32 ? k : 0] : b[k], j & 31);
      if (j < 32 && i0 >= j) a[j < 32 ? j : 0] -= l0 * cjk;
      b[j] -= l1 * cjk;
    }
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) if (j <= i0 && i0 <= C && j < C) S[acol(j, C) + i0 - j] = a[j];
#pragma unroll
  for (int j = 0; j < CM; ++j) if (i1 <= C && j <= i1 && j < C) S[acol(j, C) + i1 - j] = b[j];
}

template <typename T, int CM>
__global__ void bench_regs(const T* __restrict__ Ain, int C, int reps, long long* cyc, T* out) {
  __shared__ T S[MAXCA], S0[MAXCA], invd[64];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int CA = C * (C + 3) / 2;
  for (int i = tid; i < CA; i += NT) S0[i] = Ain[i];
  __syncthreads();
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = tid; i < CA; i += NT) S[i] = S0[i];
    __syncthreads();
    long long t0 = clock64();
    if (wid == 0) ldl_regs<T, CM>(S, invd, C, lane);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) cyc[0] = tot / reps;
  for (int i = tid; i < CA; i += NT) out[i] = S[i];
}


__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ float frcp(float x) { return __frcp_rn(x); }

// rank-2 steps, fast reciprocals, register-held (i,j) per thread entry
template <typename T>
__global__ void bench_r2f(const T* __restrict__ Ain, int C, int reps, long long* cyc, T* out) {
  __shared__ T S[MAXCA], S0[MAXCA], invd[64];
  __shared__ unsigned short tab[MAXCA];
  const int tid = threadIdx.x;
  const int CA = C * (C + 3) / 2;
  for (int i = tid; i < CA; i += NT) S0[i] = Ain[i];
  for (int j = tid; j < C; j += NT) {
    const int a0 = acol(j, C);
    for (int i = j; i <= C; ++i) tab[a0 + i - j] = (unsigned short)((i << 8) | j);
  }
  __syncthreads();
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = tid; i < CA; i += NT) S[i] = S0[i];
    __syncthreads();
    long long t0 = clock64();
    constexpr int E = 5;
    int ii[E], jj[E];
#pragma unroll
    for (int u = 0; u < E; ++u) {
      const int e = tid + u * NT;
      const unsigned ij = e < CA ? tab[e] : 0u;
      ii[u] = e < CA ? (int)(ij >> 8) : 0;
      jj[u] = e < CA ? (int)(ij & 255u) : -1;
    }
    int k = 0;
    for (; k + 1 < C; k += 2) {
      const T* colk = S + acol(k, C) - k;
      T* colk1 = S + acol(k + 1, C) - (k + 1);
      const T d0 = colk[k], a10 = colk[k + 1], d1r = colk1[k + 1];
      const T i0 = frcp(d0);
      const T l10 = a10 * i0;
      const T d1 = d1r - l10 * a10;
      const T i1 = frcp(d1);
#pragma unroll
      for (int u = 0; u < E; ++u) {
        const int e = tid + u * NT;
        if (jj[u] >= k + 2) {
          const T a = colk[ii[u]], b = colk[jj[u]], c = colk1[ii[u]], dd = colk1[jj[u]];
          const T sv = S[e];
          const T ci1 = c - a * l10, cj1 = dd - b * l10;
          S[e] = sv - a * b * i0 - ci1 * cj1 * i1;
        }
      }
      __syncthreads();
      for (int i = k + 1 + tid; i <= C; i += NT) colk1[i] = (i == k + 1) ? d1 : colk1[i] - colk[i] * l10;
      if (tid == 0) { invd[k] = i0; invd[k + 1] = i1; }
      __syncthreads();
    }
    for (; k < C; ++k) {
      const T* colk = S + acol(k, C) - k;
      const T d = colk[k];
      const T inv = frcp(d);
#pragma unroll
      for (int u = 0; u < E; ++u) {
        const int e = tid + u * NT;
        if (jj[u] > k) S[e] -= colk[ii[u]] * colk[jj[u]] * inv;
      }
      if (tid == 0) invd[k] = inv;
      __syncthreads();
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) cyc[0] = tot / reps;
  for (int i = tid; i < CA; i += NT) out[i] = S[i];
}

// rank-1 steps, fast reciprocal, register-held (i,j)
template <typename T>
__global__ void bench_r1f(const T* __restrict__ Ain, int C, int reps, long long* cyc, T* out) {
  __shared__ T S[MAXCA], S0[MAXCA], invd[64];
  __shared__ unsigned short tab[MAXCA];
  const int tid = threadIdx.x;
  const int CA = C * (C + 3) / 2;
  for (int i = tid; i < CA; i += NT) S0[i] = Ain[i];
  for (int j = tid; j < C; j += NT) {
    const int a0 = acol(j, C);
    for (int i = j; i <= C; ++i) tab[a0 + i - j] = (unsigned short)((i << 8) | j);
  }
  __syncthreads();
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = tid; i < CA; i += NT) S[i] = S0[i];
    __syncthreads();
    long long t0 = clock64();
    constexpr int E = 5;
    int ii[E], jj[E];
#pragma unroll
    for (int u = 0; u < E; ++u) {
      const int e = tid + u * NT;
      const unsigned ij = e < CA ? tab[e] : 0u;
      ii[u] = e < CA ? (int)(ij >> 8) : 0;
      jj[u] = e < CA ? (int)(ij & 255u) : -1;
    }
    for (int k = 0; k < C; ++k) {
      const T* colk = S + acol(k, C) - k;
      const T d = colk[k];
      const T inv = frcp(d);
#pragma unroll
      for (int u = 0; u < E; ++u) {
        const int e = tid + u * NT;
        if (jj[u] > k) S[e] -= colk[ii[u]] * colk[jj[u]] * inv;
      }
      if (tid == 0) invd[k] = inv;
      __syncthreads();
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) cyc[0] = tot / reps;
  for (int i = tid; i < CA; i += NT) out[i] = S[i];
}


// rank-2 steps with ONE barrier per step: column k+1 is finalised lazily in the
// next step (nobody reads it there); fast reciprocals; register-held (i,j)
template <typename T>
__global__ void bench_r2b(const T* __restrict__ Ain, int C, int reps, long long* cyc, T* out) {
  __shared__ T S[MAXCA], S0[MAXCA], invd[64], l10s[64];
  __shared__ unsigned short tab[MAXCA];
  const int tid = threadIdx.x;
  const int CA = C * (C + 3) / 2;
  for (int i = tid; i < CA; i += NT) S0[i] = Ain[i];
  for (int j = tid; j < C; j += NT) {
    const int a0 = acol(j, C);
    for (int i = j; i <= C; ++i) tab[a0 + i - j] = (unsigned short)((i << 8) | j);
  }
  __syncthreads();
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = tid; i < CA; i += NT) S[i] = S0[i];
    __syncthreads();
    long long t0 = clock64();
    constexpr int E = 5;
    int ii[E], jj[E];
#pragma unroll
    for (int u = 0; u < E; ++u) {
      const int e = tid + u * NT;
      const unsigned ij = e < CA ? tab[e] : 0u;
      ii[u] = e < CA ? (int)(ij >> 8) : 0;
      jj[u] = e < CA ? (int)(ij & 255u) : -1;
    }
    int k = 0;
    int pend = -1;   // column waiting for its rank-1 finalisation (pend = k-1 of the previous step)
    for (; k + 1 < C; k += 2) {
      const T* colk = S + acol(k, C) - k;
      const T* colk1 = S + acol(k + 1, C) - (k + 1);
      const T d0 = colk[k], a10 = colk[k + 1], d1r = colk1[k + 1];
      const T i0 = frcp(d0);
      const T l10 = a10 * i0;
      const T d1 = d1r - l10 * a10;
      const T i1 = frcp(d1);
      if (tid == 0) { invd[k] = i0; invd[k + 1] = i1; l10s[k] = l10; }
#pragma unroll
      for (int u = 0; u < E; ++u) {
        const int e = tid + u * NT;
        if (jj[u] >= k + 2) {
          const T a = colk[ii[u]], b = colk[jj[u]], c = colk1[ii[u]], dd = colk1[jj[u]];
          const T sv = S[e];
          const T ci1 = c - a * l10, cj1 = dd - b * l10;
          S[e] = sv - a * b * i0 - ci1 * cj1 * i1;
        }
      }
      if (pend >= 0) {   // finalise column pend = k-1 (rank-1 with column k-2)
        T* cp = S + acol(pend, C) - pend;
        const T* cq = S + acol(pend - 1, C) - (pend - 1);
        const T lp = l10s[pend - 1];
        for (int i = pend + tid; i <= C; i += NT) cp[i] = (i == pend) ? cp[i] - lp * cq[pend] : cp[i] - cq[i] * lp;
      }
      pend = k + 1;
      __syncthreads();
    }
    if (pend >= 0) {
      T* cp = S + acol(pend, C) - pend;
      const T* cq = S + acol(pend - 1, C) - (pend - 1);
      const T lp = l10s[pend - 1];
      for (int i = pend + tid; i <= C; i += NT) cp[i] = (i == pend) ? cp[i] - lp * cq[pend] : cp[i] - cq[i] * lp;
      __syncthreads();
    }
    for (; k < C; ++k) {
      const T* colk = S + acol(k, C) - k;
      const T d = colk[k];
      const T inv = frcp(d);
#pragma unroll
      for (int u = 0; u < E; ++u) {
        const int e = tid + u * NT;
        if (jj[u] > k) S[e] -= colk[ii[u]] * colk[jj[u]] * inv;
      }
      if (tid == 0) invd[k] = inv;
      __syncthreads();
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) cyc[0] = tot / reps;
  for (int i = tid; i < CA; i += NT) out[i] = S[i];
}


// wavefront (fan-in, column-cyclic): warp w owns columns j = w (mod 8); for
// each own column it applies the updates of columns k < j as soon as their
// ready flags are published, then publishes its own pivot. No CTA barrier.
template <typename T>
__global__ void bench_wave(const T* __restrict__ Ain, int C, int reps, long long* cyc, T* out) {
  __shared__ T S[MAXCA], S0[MAXCA], invd[64];
  __shared__ volatile int ready[64];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NWW = NT / 32;
  const int CA = C * (C + 3) / 2;
  for (int i = tid; i < CA; i += NT) S0[i] = Ain[i];
  __syncthreads();
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = tid; i < CA; i += NT) S[i] = S0[i];
    if (tid < 64) ready[tid] = 0;
    __syncthreads();
    long long t0 = clock64();
    const int epoch = r + 1;
    for (int j = wid; j < C; j += NWW) {
      T* colj = S + acol(j, C) - j;   // colj[i] = S[i][j], i in [j, C]
      const int i0 = j + lane, i1 = j + lane + 32;
      T x0 = i0 <= C ? colj[i0] : T(0);
      T x1 = i1 <= C ? colj[i1] : T(0);
      for (int k = 0; k < j; ++k) {
        const T* colk = S + acol(k, C) - k;
        if (lane == 0) while (ready[k] != epoch) { }
        __syncwarp();
        __threadfence_block();
        const T l = colk[j] * invd[k];            // L_jk
        if (i0 <= C) x0 -= colk[i0] * l;
        if (i1 <= C) x1 -= colk[i1] * l;
      }
      const T d = __shfl_sync(0xffffffffu, x0, 0);   // row j = lane 0
      const T inv = frcp(d);
      if (i0 <= C) colj[i0] = x0;
      if (i1 <= C) colj[i1] = x1;
      if (lane == 0) invd[j] = inv;
      __threadfence_block();
      __syncwarp();
      if (lane == 0) ready[j] = epoch;
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) cyc[0] = tot / reps;
  for (int i = tid; i < CA; i += NT) out[i] = S[i];
}

template <typename T>
void run(int C) {
  const int CA = C * (C + 3) / 2;
  // random SPD matrix A = G G^T + C I, augmented with rhs
  std::vector<double> G(C * C), A(C * C);
  srand(1);
  for (auto& g : G) g = (rand() / (double)RAND_MAX) - 0.5;
  for (int i = 0; i < C; ++i) for (int j = 0; j < C; ++j) { double s = 0; for (int k = 0; k < C; ++k) s += G[i * C + k] * G[j * C + k]; A[i * C + j] = s + (i == j ? C : 0); }
  std::vector<T> h(CA);
  for (int j = 0; j < C; ++j) { for (int i = j; i < C; ++i) h[acol(j, C) + i - j] = (T)A[i * C + j]; h[acol(j, C) + C - j] = (T)(j + 1); }
  T *dA, *dO; long long* dc;
  cudaMalloc(&dA, CA * sizeof(T)); cudaMalloc(&dO, CA * sizeof(T)); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, h.data(), CA * sizeof(T), cudaMemcpyHostToDevice);
  std::vector<T> ref(CA), o(CA);
  const char* names[] = {"all-threads x4", "1 warp x4", "1 warp lane=row", "all-threads rank-2", "barrier only", "lds-sts-bar", "register-owned", "warp registers CM=43", "warp registers CM=49", "rank-2 fast-rcp regs", "rank-1 fast-rcp regs", "rank-2 1-barrier", "wavefront flags"};
  auto go = [&](auto kern, int v) {
    kern<<<1, NT>>>(dA, C, 50, dc, dO);
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(o.data(), dO, CA * sizeof(T), cudaMemcpyDeviceToHost);
    if (v == 0) ref = o;
    double err = 0; for (int i = 0; i < CA; ++i) err = fmax(err, fabs((double)o[i] - (double)ref[i]) / (1e-30 + fabs((double)ref[i])));
    printf("%s C=%d %-20s %6lld cycles  maxrel %.2e  %s\n", sizeof(T) == 4 ? "f32" : "f64", C, names[v], c, err, cudaGetErrorString(cudaGetLastError()));
  };
  go(bench<T, 0>, 0); go(bench<T, 3>, 3); go(bench_r2b<T>, 11); go(bench_wave<T>, 12);
}

int main() {
  run<float>(43); run<double>(43); run<float>(49); run<double>(49); run<double>(42);
  return 0;
}
