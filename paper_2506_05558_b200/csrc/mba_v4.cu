// mba_v4.cu -- cluster-resident Levenberg-Marquardt mini-BA (sm_100a).
//
// Same algorithm as solve_kernel (mba_solve.cu) -- lm_solve, miniba.py:223-296,
// with residuals (85-98), huber/cauchy weights (46-54), _build_blocks
// (101-132), _assemble (135-177) and solve_step(method="schur") (180-220) --
// re-mapped so that a problem's whole working set lives in SHARED MEMORY:
//
//  * One thread-block cluster of R CTAs per problem (R = 1, 2, 4, 6, 8, 9, 16 chosen
//    by the host so the problem fits). CTA r owns a contiguous, point-aligned
//    slice of the point-major observations; partial normal equations are
//    summed across the cluster through distributed shared memory (DSMEM) in
//    rank order, so every CTA holds a bit-identical reduced camera system and
//    factorises it redundantly (no broadcast, no global memory traffic).
//  * No per-observation Y = W V^-1/2 blocks are materialised. The point pass
//    stores a COMPACT Jacobian per observation -- sqrt(w)*(f/z, -fx/z^2,
//    -fy/z^2), v = R X, sqrt(w)*F, sqrt(w)*r (10 values) -- and the 3x3 point
//    factor L_p. Schur products are rebuilt algebraically:
//        A_i = Jp_i G_i,  G_i = [-[v_i]x | I],  B_i = Jp_i R_c,
//        Q_i = B_i L_p^-T (2x3),
//        Y_i Y_j^T = G_i^T (Jp_i^T (Q_i Q_j^T) Jp_j) G_j        (6x6)
//    i.e. ~126 flops and 18 loads per co-observation pair instead of 108
//    flops and 36 loads from an 18-value Y -- and 3x less memory, which is what
//    lets the scratch stay on chip.
//  * Camera jobs (U_aa, U_af, g_a, sum Y yf, sum Y z) and pair jobs
//    (S_ab = -sum Y_i Y_j^T) are warps pulling from a shared-memory job queue;
//    each job is reduced by a transposed warp butterfly (37-46 shuffles for 36-45
//    sums instead of 180-225). Results do not depend on which warp ran a job.
//  * LDL^T of the augmented reduced system (forward substitution fused), then a
//    column-oriented back substitution in one warp (no reductions).
//  * Trial cost passes read observations, points and the step from shared
//    memory; the accept/reject / lambda logic is evaluated redundantly in every
//    CTA of the cluster from identical sums.
//
// State (cameras, focal, points) is float64; T is the arithmetic type of the
// linearise/Schur/LDL^T stages (double = "f64", float = "mixed").
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cooperative_groups.h>
#include <type_traits>

#include "mba_common.cuh"
#include "mba_v4.cuh"

namespace cg = cooperative_groups;

namespace mba {
namespace v4 {

// observations per thread in flight in the cost passes (try 0 / fused tries
// 1-4). One: the passes are not latency-bound enough for unrolling to pay for
// its registers (scripts/gpu/cost_u_sweep*.sh, config 4: f64 259k at 4 / 2 ->
// 266k at 1 / 1, mixed 297k -> 312k).
#ifndef MBA_COST_U
#define MBA_COST_U 1
#endif
#ifndef MBA_COST4_U
#define MBA_COST4_U 1
#endif
constexpr int NW_MAX = 16;                       // layout bound: warps per CTA
constexpr int MAXN = 8;                          // cameras per problem
constexpr int MAXC = 6 * MAXN + 1;               // reduced system size (+ focal)
constexpr int MAXNB = MAXN * (MAXN + 1) / 2;     // camera blocks a <= b
constexpr int CA_MAX = MAXC * (MAXC + 3) / 2;    // augmented packed size
// per observation: sqrt(w) (f/z, -fx/z^2, -fy/z^2) [+ sqrt(w) r in fp32 mode, where
// re-deriving the residual from rounded factors would cancel]; v = R X, the
// focal derivative and (fp64) the residual are recomputed where used. Odd
// strides keep shared-memory accesses conflict-free.
template <typename T>
__host__ __device__ constexpr int jstr() { return sizeof(T) == 8 ? 3 : 5; }
// per point: iL00 L10 iL11 L20 L21 iL22 z0..2 yf0..2 (+1 pad); the back
// substitution overwrites z with dp (z is consumed there, by the same thread),
// so the step costs no slots: 13 instead of 15 values per point (f64: 16 B less
// per point, which lets a full batch of K = 20k problems run on 9-CTA
// clusters). The stride stays odd: thread-per-point accesses stay free of
// bank conflicts (a stride of 12 measured 2 % slower on config 4).
constexpr int PSTR = 13;
constexpr int PDP = 6;     // dp0..2 live where z0..2 were
constexpr int UST = 51;    // camera job: U_aa - sum_self Y Y^T (21) U_af(6) g_a(6) SYf(6) SYz(6) diag U_aa(6)
constexpr int JOB_PAIR0 = MAXN * UST;
constexpr int JOB_PART = JOB_PAIR0 + MAXNB * 36;
constexpr int JOB_OUT = JOB_PART + 4;
constexpr size_t kSmemLimit = 227 * 1024;

__host__ __device__ constexpr size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ __forceinline__ int acol(int j, int C) { return j * (C + 1) - (j * (j - 1)) / 2; }

template <typename T>
struct Fixed {
  static constexpr size_t oRc = 0;                                    // double[MAXN][9]
  static constexpr size_t oTc = oRc + 8 * 9 * MAXN;                   // double[MAXN][3]
  static constexpr size_t oRt = oTc + 8 * 3 * MAXN;                   // double[5][MAXN][9]
  static constexpr size_t oTt = oRt + 8 * 9 * MAXN * kBacktrackTries; // double[5][MAXN][3]
  static constexpr size_t oDc = oTt + 8 * 3 * MAXN * kBacktrackTries; // double[MAXC]
  static constexpr size_t oXch = oDc + 8 * MAXC;                      // double[2][4] cluster exchange
  static constexpr size_t oRed = oXch + 8 * 8;                        // double[NW_MAX][4]
  static constexpr size_t oS = al16(oRed + 8 * NW_MAX * 4);           // T[CA_MAX]
  static constexpr size_t oJob = al16(oS + sizeof(T) * CA_MAX);       // T[JOB_OUT] this CTA's partials
  static constexpr size_t oInvd = al16(oJob + sizeof(T) * JOB_OUT);   // T[MAXC]
  static constexpr size_t oTab = al16(oInvd + sizeof(T) * MAXC);      // u16[CA_MAX] (row<<8|col)
  static constexpr size_t oCamPtr = al16(oTab + 2 * CA_MAX);          // int[MAXN+1]
  static constexpr size_t oSlot = oCamPtr + 4 * (MAXN + 1);           // int[MAXN]
  static constexpr size_t oCos = oSlot + 4 * MAXN;                    // int[MAXN]
  static constexpr size_t oBlkOff = oCos + 4 * MAXN;                  // int[MAXNB+1]
  static constexpr size_t oBlkA = oBlkOff + 4 * (MAXNB + 1);          // u8[MAXNB]
  static constexpr size_t oBlkB = oBlkA + MAXNB;                      // u8[MAXNB]
  static constexpr size_t oRcT = al16(oBlkB + MAXNB);                 // T[MAXN][9] rotations in T
  static constexpr size_t oDcT = al16(oRcT + sizeof(T) * 9 * MAXN);   // T[MAXC] step in T
  static constexpr size_t oL10 = al16(oDcT + sizeof(T) * MAXC);       // T[MAXC] LDL^T pair multipliers
  static constexpr size_t kBytes = al16(oL10 + sizeof(T) * MAXC);
};

// bytes per local observation / observed point in the arena (plus pairs, 4 B each)
template <typename T>
__host__ __device__ constexpr size_t obs_bytes() { return 16 + sizeof(T) * jstr<T>() + 2; }
template <typename T>
__host__ __device__ constexpr size_t pt_bytes() { return 24 + sizeof(T) * PSTR + 4 + 2; }

// Optional per-phase cycle counters (-DMBA_PHASE_PROF, scripts/phase_prof.py):
// thread 0 of every CTA accumulates clock64() deltas between phase marks.
enum { PH_SETUP, PH_COST0, PH_POINT, PH_JOBS, PH_ASM, PH_CHOL, PH_SOLVE, PH_TRIAL, PH_COMMIT, PH_CHA, PH_CHB, PH_LCAM, PH_NCAM, PH_LPAIR, PH_NPAIR, PH_N };
#ifdef MBA_PHASE_PROF
#define LANES_PROF(sum_slot, n_slot) { const unsigned am_ = __activemask(); if (threadIdx.x == 0) { s_prof[sum_slot] += __popc(am_); s_prof[n_slot] += 1; } }
#else
#define LANES_PROF(sum_slot, n_slot)
#endif
#ifdef MBA_PHASE_PROF
static __device__ unsigned long long* g_prof = nullptr;
#define PROF_DECL __shared__ long long s_prof[PH_N]; long long prof_t = clock64(); \
  if (threadIdx.x == 0) for (int i = 0; i < PH_N; ++i) s_prof[i] = 0;
#define PROF_MARK(ph) if (threadIdx.x == 0) { long long now = clock64(); s_prof[ph] += now - prof_t; prof_t = now; }
#define PROF_FLUSH if (threadIdx.x == 0 && g_prof) for (int i = 0; i < PH_N; ++i) atomicAdd(g_prof + i, (unsigned long long)s_prof[i]);
#ifdef MBA_V4_F32
void set_prof_f32(unsigned long long* p) { cudaMemcpyToSymbol(g_prof, &p, sizeof(p)); }
#else
void set_prof_f64(unsigned long long* p) { cudaMemcpyToSymbol(g_prof, &p, sizeof(p)); }
#endif
#else
#define PROF_DECL
#define PROF_MARK(ph)
#define PROF_FLUSH
#endif

struct Params {
  MbaBatchDesc d;
  MbaLmConfig cfg;
  MbaOutputs o;
  size_t arena;   // bytes of dynamic shared memory after the fixed part
  unsigned char* gcache;   // optional per-SM linearisation caches (one CTA per SM plans)
  size_t gcache_slot;      // bytes per SM
  int gcache_slots;        // number of SM slots
};

// ---------------------------------------------------------------------------
// warp helpers

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Deterministic block sum of N doubles (result to every thread).
template <int NW, int N>
__device__ __forceinline__ void block_sum_d(double (&v)[N], double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < N; ++i) red[wid * 4 + i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w * 4 + i];
    v[i] = s;
  }
  __syncthreads();
}

template <int R>
struct Clu {
  __device__ static __forceinline__ void sync() {
    if constexpr (R > 1) cg::this_cluster().sync();
    else __syncthreads();
  }
  __device__ static __forceinline__ int rank() {
    if constexpr (R > 1) return (int)cg::this_cluster().block_rank();
    else return 0;
  }
  template <typename U>
  __device__ static __forceinline__ U* remote(U* p, int r) {
    if constexpr (R > 1) return cg::this_cluster().map_shared_rank(p, r);
    else return p;
  }
};

// Cluster-wide sum of N (<= 4) doubles that every thread holds (after a block
// sum); rank-ordered, so every CTA gets bit-identical totals. Double-buffered
// exchange slots -> one cluster barrier per call.
template <int R, int N>
__device__ __forceinline__ void cluster_sum(double (&v)[N], double* xch, int& epoch) {
  if constexpr (R > 1) {
    double* slot = xch + 4 * (epoch & 1);
    ++epoch;
    if (threadIdx.x == 0)
#pragma unroll
      for (int i = 0; i < N; ++i) slot[i] = v[i];
    Clu<R>::sync();
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double* q = Clu<R>::remote(slot, r);
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] += q[i];
    }
  }
}

// fp64 projection with the reciprocal depth kept (miniba.py:85-98; one
// reciprocal instead of two divisions, <= 1 ulp from the reference's (f x)/z)
struct ProjZ {
  double pc[3], v[3], ru, rv, iz;
  bool behind;
};
__device__ __forceinline__ ProjZ proj_z(const double* __restrict__ R, const double* __restrict__ t,
                                        const double X[3], double f, double cx, double cy, double u,
                                        double vv) {
  ProjZ o;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    o.pc[i] = R[i * 3 + 0] * X[0] + R[i * 3 + 1] * X[1] + R[i * 3 + 2] * X[2] + t[i];
    o.v[i] = o.pc[i] - t[i];  // R X recovered as p_cam - t, as miniba.py:117 does
  }
  o.behind = !(o.pc[2] > kZMin);
  o.iz = 1.0 / (o.behind ? kZMin : o.pc[2]);
  o.ru = o.behind ? kBadResidual : f * o.pc[0] * o.iz + cx - u;
  o.rv = o.behind ? kBadResidual : f * o.pc[1] * o.iz + cy - vv;
  return o;
}

// reciprocal for the factorisation pivots: fp64 MUFU seed + two Newton steps
// (<= 1 ulp), fp32 correctly rounded
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ float fast_rcp(float x) { return 1.0f / x; }

// robust cost from the squared residual norm (miniba.py:46-50 + Cauchy): the
// square root is only taken for Huber observations beyond delta
__device__ __forceinline__ double rho_e2(double e2, double delta, int loss) {
  if (loss == MBA_LOSS_CAUCHY) return 0.5 * delta * delta * log1p(e2 / (delta * delta));
  if (e2 <= delta * delta) return 0.5 * e2;
  const double e = sqrt(e2);
  return e <= delta ? 0.5 * e * e : delta * (e - 0.5 * delta);
}

// sqrt of the IRLS weight (miniba.py:52-54 + Cauchy). e2 <= delta^2 implies
// sqrt(e2) <= delta after rounding, so inliers need no square root at all.
__device__ __forceinline__ double sqrt_w_e2(double e2, double delta, int loss) {
  if (loss == MBA_LOSS_CAUCHY) return sqrt(1.0 / (1.0 + e2 / (delta * delta)));
  if (e2 <= delta * delta) return 1.0;
  const double e = sqrt(e2);
  return e <= delta ? 1.0 : sqrt(delta / fmax(e, 1e-300));
}

// fp64 projection of point X by camera (R, t), residual, robust weight and the
// compact Jacobian (miniba.py:85-132 + 46-54), scaled by sqrt(w).
template <typename T>
struct CompactJ {
  T J0, J1, J2, v0, v1, v2, F0, F1, r0, r1;
};

template <typename T>
__device__ __forceinline__ CompactJ<T> linearise(const double* __restrict__ Rm, const double* __restrict__ t,
                                                 const double X[3], double f, double cx, double cy,
                                                 double u, double vv, double delta, int loss) {
  const ProjZ pr = proj_z(Rm, t, X, f, cx, cy, u, vv);
  const double s = sqrt_w_e2(pr.ru * pr.ru + pr.rv * pr.rv, delta, loss);
  CompactJ<T> c;
  c.r0 = T(s * pr.ru);
  c.r1 = T(s * pr.rv);
  if (pr.behind) {  // miniba.py:114,131: rows of behind-camera observations are zeroed
    c.J0 = c.J1 = c.J2 = c.v0 = c.v1 = c.v2 = c.F0 = c.F1 = T(0);
    return c;
  }
  const double iz = pr.iz;
  const double fz = f * iz;
  c.J0 = T(s * fz);
  c.J1 = T(-s * fz * pr.pc[0] * iz);
  c.J2 = T(-s * fz * pr.pc[1] * iz);
  c.v0 = T(pr.v[0]);
  c.v1 = T(pr.v[1]);
  c.v2 = T(pr.v[2]);
  c.F0 = T(s * pr.pc[0] * iz);
  c.F1 = T(s * pr.pc[1] * iz);
  return c;
}

// Q = (Jp R) L^-T for one observation: two rows of 3 (forward substitution
// with the point factor; L diagonal stored inverted).
template <typename T>
__device__ __forceinline__ void q_rows(T J0, T J1, T J2, const T* Rt, const T* __restrict__ L, T q[6]) {
  const T iL00 = L[0], L10 = L[1], iL11 = L[2], L20 = L[3], L21 = L[4], iL22 = L[5];
  T b[6];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    b[c] = J0 * Rt[c] + J1 * Rt[6 + c];
    b[3 + c] = J0 * Rt[3 + c] + J2 * Rt[6 + c];
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const T x0 = b[3 * r] * iL00;
    const T x1 = (b[3 * r + 1] - L10 * x0) * iL11;
    const T x2 = (b[3 * r + 2] - L20 * x0 - L21 * x1) * iL22;
    q[3 * r] = x0;
    q[3 * r + 1] = x1;
    q[3 * r + 2] = x2;
  }
}

// A = Jp [-[v]x | I] (2x6), rotation columns first (miniba.py:116-128)
template <typename T>
__device__ __forceinline__ void expand_A(T J0, T J1, T J2, T v0, T v1, T v2, T a[12]) {
  a[0] = J1 * v1;
  a[1] = J0 * v2 - J1 * v0;
  a[2] = -J0 * v1;
  a[3] = J0;
  a[4] = T(0);
  a[5] = J1;
  a[6] = J2 * v1 - J0 * v2;
  a[7] = -J2 * v0;
  a[8] = J0 * v0;
  a[9] = T(0);
  a[10] = J0;
  a[11] = J2;
}

// ---------------------------------------------------------------------------

template <typename T, int R, int NT>
__device__ void solve_problem(const Params& P, unsigned char* smem) {
  constexpr int NW = NT / 32;
  using F = Fixed<T>;
  constexpr int JSTR = jstr<T>();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rank = Clu<R>::rank();
  const int b = (int)(blockIdx.x / R);
  const bool lead = rank == 0 && tid == 0;
  const MbaBatchDesc& D = P.d;
  const MbaLmConfig& cfg = P.cfg;
  const MbaOutputs& O = P.o;

  double* Rc = (double*)(smem + F::oRc);
  double* tc = (double*)(smem + F::oTc);
  double* Rt = (double*)(smem + F::oRt);
  double* tt = (double*)(smem + F::oTt);
  double* dc = (double*)(smem + F::oDc);
  double* xch = (double*)(smem + F::oXch);
  double* red = (double*)(smem + F::oRed);
  T* S = (T*)(smem + F::oS);
  T* job = (T*)(smem + F::oJob);
  T* invd = (T*)(smem + F::oInvd);
  unsigned short* tab = (unsigned short*)(smem + F::oTab);
  int* cam_ptr = (int*)(smem + F::oCamPtr);
  int* slot = (int*)(smem + F::oSlot);
  int* cslot = (int*)(smem + F::oCos);
  int* blk_off = (int*)(smem + F::oBlkOff);
  unsigned char* blk_a = smem + F::oBlkA;
  unsigned char* blk_b = smem + F::oBlkB;
  unsigned char* arena = smem + F::kBytes;
  T* RcT = (T*)(smem + F::oRcT);
  T* dcT = (T*)(smem + F::oDcT);
  T* l10s = (T*)(smem + F::oL10);

  __shared__ int s_flag, s_nf, s_nlp, s_npairs, s_job, s_gcam;
  __shared__ unsigned char s_jorder[MAXN + MAXNB];   // job queue order: longest first
  __shared__ int s_wtot[NW_MAX];
  int epoch = 0;
  PROF_DECL

  const int64_t cb = D.cam_off[b], pb = D.pt_off[b], ob = D.obs_off[b];
  const int n = (int)(D.cam_off[b + 1] - cb);
  const int Pn = (int)(D.pt_off[b + 1] - pb);
  const int K = (int)(D.obs_off[b + 1] - ob);
  const uint8_t fl = D.flags[b];
  const bool has_f = fl & 1, opt_pts = (fl >> 1) & 1;
  const double cx = D.cx[b], cy = D.cy[b];
  const double delta = cfg.delta, nu = cfg.nu;
  const int loss = cfg.loss, max_it = cfg.max_iters;
  const MbaObs* __restrict__ gobs = D.obs + ob;
  const float* __restrict__ glo = D.obs_lo ? D.obs_lo + 2 * ob : nullptr;

  // ---------------- setup ----------------
  for (int i = tid; i < n * 9; i += NT) Rc[i] = O.R_in[cb * 9 + i];
  for (int i = tid; i < n * 3; i += NT) tc[i] = O.t_in[cb * 3 + i];
  if (tid == 0) {
    int nf = 0;
    for (int c = 0; c < n; ++c) {
      if (D.fixed[cb + c]) {
        slot[c] = -1;
      } else {
        slot[c] = nf;
        cslot[nf] = c;
        ++nf;
      }
    }
    int q = 0;
    for (int a = 0; a < nf; ++a)
      for (int bb = a; bb < nf; ++bb, ++q) {
        blk_a[q] = (unsigned char)a;
        blk_b[q] = (unsigned char)bb;
      }
    s_nf = nf;
    s_flag = (n > MAXN) ? 1 : 0;
    // the one fixed camera of a problem with a free scale gauge (see the step
    // projection below); -1 when the gauge is pinned or not a pure scale
    int gc = -1;
    for (int c = 0; c < n; ++c)
      if (slot[c] < 0) gc = (nf == n - 1) ? c : -1;
    s_gcam = ((fl >> 1) & 1) ? gc : -1;
  }
  __syncthreads();
  const int nf = s_nf, C = 6 * nf + (has_f ? 1 : 0), FI = C - 1, CA = C * (C + 3) / 2;
  const int nb = opt_pts ? nf * (nf + 1) / 2 : 0;
  double f = O.focal_in[b];

  // this CTA's observation slice [k0, k1): point-aligned cut near K r / R
  // (binary search on the point-major order, verified below)
  auto lower_bound_pt = [&](int p) {
    int lo_i = 0, hi_i = K;
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i) >> 1;
      if (__ldg(&gobs[mid].pt) < p) lo_i = mid + 1; else hi_i = mid;
    }
    return lo_i;
  };
  int k0 = 0, k1 = K;
  if (R > 1 && K > 0) {
    if (rank > 0) k0 = lower_bound_pt(__ldg(&gobs[(int)((int64_t)K * rank / R)].pt));
    if (rank < R - 1) k1 = lower_bound_pt(__ldg(&gobs[(int)((int64_t)K * (rank + 1) / R)].pt));
  }
  const int nlo = k1 > k0 ? k1 - k0 : 0;
  // stage the slice's 16-byte records in shared memory (one coalesced pass) and
  // validate it there: index ranges, point-major order, slice boundary
  float4* sobs = (float4*)arena;                                        // [nlo] u, v, cam, point slot
  unsigned char* newpt = arena + al16(16 * (size_t)nlo);               // [nlo] scratch (setup only)
  bool overflow = al16(16 * (size_t)nlo) + nlo > P.arena || nlo >= 65535;
  if (tid == 0 && k1 < k0) s_flag = 1;
  if (!overflow) {
    // eight 16-byte loads in flight per thread (one HBM round trip per 2k records)
    for (int k8 = tid; k8 < nlo; k8 += 8 * NT) {
      float4 rec[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k8 + u * NT < nlo) rec[u] = __ldg(reinterpret_cast<const float4*>(gobs) + k0 + k8 + u * NT);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (k8 + u * NT >= nlo) continue;
        const int c = __float_as_int(rec[u].z), pt = __float_as_int(rec[u].w);
        if (pt < 0 || pt >= Pn || c < 0 || c >= n) s_flag = 1;
        sobs[k8 + u * NT] = rec[u];
      }
    }
    __syncthreads();
    int cnt = 0;
    for (int kl = tid; kl < nlo; kl += NT) {
      const int pt = __float_as_int(sobs[kl].w);
      const int prev = kl > 0 ? __float_as_int(sobs[kl - 1].w) : -1;
      if (prev > pt) s_flag = 1;
      newpt[kl] = prev != pt;
      cnt += prev != pt;
    }
    if (tid == 0 && nlo > 0 && k1 < K && __ldg(&gobs[k1].pt) < __float_as_int(sobs[nlo - 1].w)) s_flag = 1;
    double v[1] = {(double)cnt};
    block_sum_d<NW, 1>(v, red);
    if (tid == 0) s_nlp = (int)v[0];
  }
  __syncthreads();
  {  // the cluster agrees on validity (malformed problems keep their parameters)
    double v[1] = {s_flag ? 1.0 : 0.0};
    __syncthreads();
    cluster_sum<R, 1>(v, xch, epoch);
    if (v[0] != 0.0) {
      if (lead) {
        O.n_iters[b] = 0;
        O.status[b] = -1;
        O.focal_out[b] = f;
      }
      if (rank == 0) {
        for (int i = tid; i < n * 9; i += NT) O.R_out[cb * 9 + i] = O.R_in[cb * 9 + i];
        for (int i = tid; i < n * 3; i += NT) O.t_out[cb * 3 + i] = O.t_in[cb * 3 + i];
      }
      for (int i = rank * NT + tid; i < Pn * 3; i += R * NT)
        O.points_out[pb * 3 + i] = O.points_in[pb * 3 + i];
      Clu<R>::sync();
      return;
    }
  }
  // points [p_lo, p_hi) belong to this rank (unobserved points included: they
  // keep their value, dp = 0, as in the reference)
  const int p_lo = rank == 0 ? 0 : (k0 < K ? __ldg(&gobs[k0].pt) : Pn);
  const int p_hi = rank == R - 1 ? Pn : (k1 < K ? __ldg(&gobs[k1].pt) : Pn);
  if (O.points_in != O.points_out)
    for (int i = p_lo * 3 + tid; i < p_hi * 3; i += NT) O.points_out[pb * 3 + i] = O.points_in[pb * 3 + i];

  const int nlp = overflow ? 0 : s_nlp;
  // arena layout (newpt scratch aliases the start of Xs; it is consumed first)
  double* Xs = (double*)(arena + al16(16 * (size_t)nlo));               // [nlp][3]
  T* jac = (T*)((unsigned char*)Xs + al16(24 * (size_t)nlp));           // [nlo][JSTR]
  T* pf = (T*)((unsigned char*)jac + al16(sizeof(T) * JSTR * (size_t)nlo));  // [nlp][PSTR]
  int* lpt = (int*)((unsigned char*)pf + al16(sizeof(T) * PSTR * (size_t)nlp));  // [nlp]
  unsigned short* perm = (unsigned short*)((unsigned char*)lpt + al16(4 * (size_t)nlp));  // [nlo]
  unsigned short* ptr = (unsigned short*)((unsigned char*)perm + al16(2 * (size_t)nlo));  // [nlp+1]
  unsigned* pairs = (unsigned*)((unsigned char*)ptr + al16(2 * (size_t)(nlp + 1)));
  const size_t fixed_need = (size_t)((unsigned char*)pairs - arena);
  overflow = overflow || fixed_need > P.arena;

  if (!overflow) {
    // point slots: block-wide scan of "first observation of a point"
    int base = 0;
    for (int c0 = 0; c0 < nlo; c0 += NT) {
      const int kl = c0 + tid;
      const int flag = kl < nlo ? newpt[kl] : 0;
      const int inc = warp_incl_scan(flag, lane);
      if (lane == 31) s_wtot[wid] = inc;
      __syncthreads();
      int pre = base;
      for (int w = 0; w < wid; ++w) pre += s_wtot[w];
      int tot = 0;
      for (int w = 0; w < NW; ++w) tot += s_wtot[w];
      if (kl < nlo) {
        const int sl = pre + inc - 1;
        if (flag) {
          lpt[sl] = __float_as_int(sobs[kl].w);
          ptr[sl] = (unsigned short)kl;
        }
        sobs[kl].w = __int_as_float(sl);
      }
      base += tot;
      __syncthreads();
    }
    if (tid == 0) ptr[nlp] = (unsigned short)nlo;
    __syncthreads();
    for (int i8 = tid; i8 < nlp * 3; i8 += 8 * NT) {   // gathered point loads, eight in flight
      double xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i8 + u * NT;
        if (i < nlp * 3) xv[u] = __ldg(O.points_in + (pb + lpt[i / 3]) * 3 + i % 3);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i8 + u * NT < nlp * 3) Xs[i8 + u * NT] = xv[u];
    }
    // camera-major permutation of the slice (warp per camera, ballot sweeps)
    for (int c = wid; c < n; c += NW) {
      int cnt = 0;
      for (int q0 = 0; q0 < nlo; q0 += 32) {
        const int q = q0 + lane;
        cnt += __popc(__ballot_sync(0xffffffffu, q < nlo && __float_as_int(sobs[q].z) == c));
      }
      if (lane == 0) cam_ptr[c + 1] = cnt;
    }
    __syncthreads();
    if (tid == 0) {
      cam_ptr[0] = 0;
      for (int c = 0; c < n; ++c) cam_ptr[c + 1] += cam_ptr[c];
    }
    __syncthreads();
    for (int c = wid; c < n; c += NW) {
      int basec = cam_ptr[c];
      for (int q0 = 0; q0 < nlo; q0 += 32) {
        const int q = q0 + lane;
        const bool hit = q < nlo && __float_as_int(sobs[q].z) == c;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (hit) perm[basec + __popc(m & ((1u << lane) - 1u))] = (unsigned short)q;
        basec += __popc(m);
      }
    }
    __syncthreads();
    // per point, where each camera's observation sits: nibble c of cpos[sl] is
    // 0 (camera c does not see the point), 1..14 (offset + 1 of its only
    // observation) or 15 (several observations / long track: scan). Scratch in
    // the (not yet used) Jacobian area.
    unsigned* cpos = reinterpret_cast<unsigned*>(jac);
    for (int sl = tid; sl < nlp; sl += NT) {
      unsigned m = 0u;
      const int j0 = ptr[sl], j1 = ptr[sl + 1];
      for (int j = j0; j < j1; ++j) {
        const int c = __float_as_int(sobs[j].z), sh = 4 * c;
        const unsigned cur = (m >> sh) & 15u;
        const unsigned v = (cur == 0u && j - j0 < 14) ? (unsigned)(j - j0 + 1) : 15u;
        m = (m & ~(15u << sh)) | (v << sh);
      }
      cpos[sl] = m;
    }
    __syncthreads();
    // co-observation pair lists per free camera block (a <= b): count, scan, fill
    for (int pass = 0; pass < 2; ++pass) {
      for (int blk = wid; blk < nb; blk += NW) {
        const int ca = cslot[blk_a[blk]], cbb = cslot[blk_b[blk]];
        const int q1 = cam_ptr[ca + 1];
        int basep = pass ? blk_off[blk] : 0;
        const unsigned lt = (1u << lane) - 1u;
        // two 32-observation chunks per step (their loads overlap); 0/1
        // multiplicities -- one observation per (camera, point), the usual
        // case -- are counted / compacted with ballots
        for (int q0 = cam_ptr[ca]; q0 < q1; q0 += 64) {
          int i[2], j0[2], m[2];
          unsigned nib[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int q = q0 + 32 * u + lane;
            i[u] = -1;
            j0[u] = 0;
            nib[u] = 0u;
            if (q < q1) {
              i[u] = perm[q];
              const int sl = __float_as_int(sobs[i[u]].w);
              j0[u] = ptr[sl];
              nib[u] = (cpos[sl] >> (4 * cbb)) & 15u;
            }
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            // self pairs (j == i) are folded into the camera jobs
            m[u] = 0;
            if (nib[u] == 15u) {
              const int j1 = ptr[__float_as_int(sobs[i[u]].w) + 1];
              for (int j = j0[u]; j < j1; ++j) m[u] += __float_as_int(sobs[j].z) == cbb && j != i[u];
            } else {
              m[u] = (nib[u] != 0u && j0[u] + (int)nib[u] - 1 != i[u]) ? 1 : 0;
            }
            int excl, cnt;
            if (!__any_sync(0xffffffffu, nib[u] == 15u)) {
              const unsigned bal = __ballot_sync(0xffffffffu, m[u] != 0);
              excl = __popc(bal & lt);
              cnt = __popc(bal);
            } else {
              excl = warp_incl_scan(m[u], lane) - m[u];
              cnt = warp_sum(m[u]);
            }
            if (pass && m[u]) {
              int pos = basep + excl;
              if (nib[u] == 15u) {
                const int j1 = ptr[__float_as_int(sobs[i[u]].w) + 1];
                for (int j = j0[u]; j < j1; ++j)
                  if (__float_as_int(sobs[j].z) == cbb && j != i[u]) pairs[pos++] = ((unsigned)i[u] << 16) | (unsigned)j;
              } else {
                pairs[pos] = ((unsigned)i[u] << 16) | (unsigned)(j0[u] + (int)nib[u] - 1);
              }
            }
            basep += cnt;
          }
        }
        if (!pass && lane == 0) blk_off[blk + 1] = basep;
      }
      __syncthreads();
      if (!pass) {
        if (tid == 0) {
          blk_off[0] = 0;
          for (int q = 0; q < nb; ++q) blk_off[q + 1] += blk_off[q];
          s_npairs = blk_off[nb];
        }
        __syncthreads();
        if (fixed_need + 4 * (size_t)s_npairs > P.arena) {
          overflow = true;
          break;
        }
      }
    }
  }
  // job queue order, longest first (results do not depend on the order):
  // job q's rank = number of jobs that are heavier (ties by index)
  if (!overflow) {
    __shared__ int s_w[MAXN + MAXNB];
    const int nj = nf + nb;
    for (int q = tid; q < nj; q += NT)
      s_w[q] = q < nf ? 3 * (cam_ptr[cslot[q] + 1] - cam_ptr[cslot[q]]) / 2
                      : blk_off[q - nf + 1] - blk_off[q - nf];
    __syncthreads();
    for (int q = tid; q < nj; q += NT) {
      int rk = 0;
      for (int r = 0; r < nj; ++r) rk += s_w[r] > s_w[q] || (s_w[r] == s_w[q] && r < q);
      s_jorder[rk] = (unsigned char)q;
    }
  }
  // packed position -> (row, col) table of the augmented system
  for (int j = tid; j < C; j += NT) {
    const int a0 = acol(j, C);
    for (int i = j; i <= C; ++i) tab[a0 + i - j] = (unsigned short)((i << 8) | j);
  }
  {  // the cluster agrees on overflow (the CTA kernel then re-solves this problem)
    double v[1] = {overflow ? 1.0 : 0.0};
    cluster_sum<R, 1>(v, xch, epoch);
    if (v[0] != 0.0) {
      if (lead) O.status[b] = kStatusPlanOverflow;
      Clu<R>::sync();
      return;
    }
  }
  __syncthreads();

  auto obs_uv = [&](int kl, const float4& o, double& u, double& vv) {
    u = (double)o.x;
    vv = (double)o.y;
    if (glo != nullptr) {
      const float2 l = __ldg(reinterpret_cast<const float2*>(glo) + k0 + kl);
      u += (double)l.x;
      vv += (double)l.y;
    }
  };

  // cost pass over the slice with camera set (Rs, ts), focal ft and points
  // X + frac * dp; cluster-summed (sum rho, sum e, sum e^2)
  // (full: also sum e and sum e^2 for final_rms / mean_err, miniba.py:295-296)
  auto cost = [&](auto full, const double* Rs, const double* ts, double ft, double frac, bool use_dp,
                  double out[3]) {
    constexpr bool FULL = decltype(full)::value;
    double acc[3] = {0.0, 0.0, 0.0};
    constexpr int U = MBA_COST_U;
    for (int c0 = tid; c0 < nlo; c0 += U * NT) {
      float4 o[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c0 + u * NT < nlo) o[u] = sobs[c0 + u * NT];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kl = c0 + u * NT;
        if (kl >= nlo) continue;
        const int sl = __float_as_int(o[u].w), c = __float_as_int(o[u].z);
        double Xp[3] = {Xs[3 * sl], Xs[3 * sl + 1], Xs[3 * sl + 2]};
        if (use_dp) {
          const T* dp = pf + (size_t)sl * PSTR + PDP;
          Xp[0] = Xp[0] + frac * (double)dp[0];
          Xp[1] = Xp[1] + frac * (double)dp[1];
          Xp[2] = Xp[2] + frac * (double)dp[2];
        }
        double uu, vv;
        obs_uv(kl, o[u], uu, vv);
        const ProjZ pr = proj_z(Rs + 9 * c, ts + 3 * c, Xp, ft, cx, cy, uu, vv);
        const double e2 = pr.ru * pr.ru + pr.rv * pr.rv;
        acc[0] += rho_e2(e2, delta, loss);
        if constexpr (FULL) {
          const double e = sqrt(e2);
          acc[1] += e;
          acc[2] += e * e;
        }
      }
    }
    if constexpr (FULL) {
      block_sum_d<NW, 3>(acc, red);
      cluster_sum<R, 3>(acc, xch, epoch);
    } else {
      double a1[1] = {acc[0]};
      block_sum_d<NW, 1>(a1, red);
      cluster_sum<R, 1>(a1, xch, epoch);
      acc[0] = a1[0];
    }
    out[0] = acc[0];
    out[1] = acc[1];
    out[2] = acc[2];
  };

  // backtracking tries 1..4 (fractions 1/2 .. 1/16) in ONE pass over the
  // observations: four camera sets / focals / point offsets per observation,
  // four rank-ordered sums (identical to four separate passes)
  auto cost4 = [&](const double (&fts)[4], double (&out)[4]) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    constexpr int U = MBA_COST4_U;
    for (int c0 = tid; c0 < nlo; c0 += U * NT) {
      float4 o[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c0 + u * NT < nlo) o[u] = sobs[c0 + u * NT];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kl = c0 + u * NT;
        if (kl >= nlo) continue;
        const int sl = __float_as_int(o[u].w), c = __float_as_int(o[u].z);
        const double X0 = Xs[3 * sl], X1 = Xs[3 * sl + 1], X2 = Xs[3 * sl + 2];
        double d0 = 0.0, d1 = 0.0, d2 = 0.0;
        if (opt_pts) {
          const T* dp = pf + (size_t)sl * PSTR + PDP;
          d0 = (double)dp[0];
          d1 = (double)dp[1];
          d2 = (double)dp[2];
        }
        double uu, vv;
        obs_uv(kl, o[u], uu, vv);
#pragma unroll
        for (int bt = 1; bt < kBacktrackTries; ++bt) {
          const double frac = 1.0 / (double)(1 << bt);
          const double Xp[3] = {X0 + frac * d0, X1 + frac * d1, X2 + frac * d2};
          const ProjZ pr = proj_z(Rt + (size_t)(bt * n + c) * 9, tt + (size_t)(bt * n + c) * 3, Xp,
                                  fts[bt - 1], cx, cy, uu, vv);
          acc[bt - 1] += rho_e2(pr.ru * pr.ru + pr.rv * pr.rv, delta, loss);
        }
      }
    }
    block_sum_d<NW, 4>(acc, red);
    cluster_sum<R, 4>(acc, xch, epoch);
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = acc[i];
  };

  // Linearisation cache (when the arena has room): per point the undamped
  // V_p, g_p, Wf_p and per thread its focal partials. An iteration that
  // follows a rejected one re-linearises at unchanged parameters (the
  // reference rebuilds the same system with a larger lambda, miniba.py:
  // 223-296), so its point pass only re-damps and re-factorises (40 % of
  // config-4 iterations are full rejections on the plateau). Same values,
  // same order -> results bit-identical to recomputing.
  constexpr int VCS = 13;   // 12 values per point, odd stride
  T* vcache = reinterpret_cast<T*>(
      reinterpret_cast<unsigned char*>(pairs) + al16(4 * (size_t)(overflow ? 0 : s_npairs)));
  T* pcache = vcache + (size_t)VCS * nlp;   // [NT][2]
  bool cache_ok = !overflow && fixed_need + al16(4 * (size_t)s_npairs) +
                                   sizeof(T) * ((size_t)VCS * nlp + 2 * NT) <= P.arena;
  if (!cache_ok && !overflow && P.gcache != nullptr) {
    // no room in shared memory (fp64): the slot of this SM in global memory
    // (L2-resident; one point's 12 values are one round trip). Only plans with
    // one CTA per SM pass gcache, so the slot has a single owner.
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if ((int)smid < P.gcache_slots && sizeof(T) * ((size_t)VCS * nlp + 2 * NT) <= P.gcache_slot) {
      vcache = reinterpret_cast<T*>(P.gcache + (size_t)smid * P.gcache_slot);
      pcache = vcache + (size_t)VCS * nlp;
      cache_ok = true;
    }
  }
  bool reuse = false;

  double* costs = O.costs + (size_t)b * (max_it + 1);
  double* lambdas = O.lambdas + (size_t)b * max_it;
  uint8_t* accepted = O.accepted + (size_t)b * max_it;
  uint8_t* evals = O.evals + (size_t)b * max_it;

  for (int i = tid; i < n * 9; i += NT) RcT[i] = T(Rc[i]);
  __syncthreads();
  PROF_MARK(PH_SETUP)
  // initial cost (miniba.py:232-235)
  double st[3];
  cost(std::false_type(), Rc, tc, f, 0.0, false, st);
  PROF_MARK(PH_COST0)
  double cur = st[0];
  double lam = cfg.lambda_init;
  if (lead) costs[0] = cur;
  int it = 0, stop_reason = MBA_SOLVE_MAX_ITERS;

  for (; it < max_it;) {
    const T tlam = T(lam);
    const T inv_f = T(1.0 / f);
    // ---------- point pass: compact Jacobians, V_p / g_p / Wf_p, point factor ----------
    T part[4] = {T(0), T(0), T(0), T(0)};  // U_ff, g_f, sum yf.yf, sum yf.z
    if (reuse) {
      part[0] = pcache[2 * tid];
      part[1] = pcache[2 * tid + 1];
    }
    for (int sl = tid; sl < nlp; sl += NT) {
      const double Xp[3] = {Xs[3 * sl], Xs[3 * sl + 1], Xs[3 * sl + 2]};
      T V[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};  // 00 10 11 20 21 22
      T g[3] = {T(0), T(0), T(0)}, wf[3] = {T(0), T(0), T(0)};
      const int j0 = ptr[sl], j1 = ptr[sl + 1];
      T* vc = vcache + (size_t)sl * VCS;
      if (reuse) {
#pragma unroll
        for (int i = 0; i < 6; ++i) V[i] = vc[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          g[i] = vc[6 + i];
          wf[i] = vc[9 + i];
        }
      }
      for (int kl = reuse ? j1 : j0; kl < j1; ++kl) {
        const float4 o = sobs[kl];
        const int c = __float_as_int(o.z);
        double uu, vv;
        obs_uv(kl, o, uu, vv);
        const CompactJ<T> cj = linearise<T>(Rc + 9 * c, tc + 3 * c, Xp, f, cx, cy, uu, vv, delta, loss);
        T* jk = jac + (size_t)kl * JSTR;
        jk[0] = cj.J0; jk[1] = cj.J1; jk[2] = cj.J2;
        if constexpr (JSTR == 5) { jk[3] = cj.r0; jk[4] = cj.r1; }
        if (has_f) {
          part[0] += cj.F0 * cj.F0 + cj.F1 * cj.F1;
          part[1] += cj.F0 * cj.r0 + cj.F1 * cj.r1;
        }
        if (opt_pts) {
          const T* Rk = RcT + 9 * c;
          T B0[3], B1[3];
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            B0[q] = cj.J0 * Rk[q] + cj.J1 * Rk[6 + q];
            B1[q] = cj.J0 * Rk[3 + q] + cj.J2 * Rk[6 + q];
          }
          V[0] += B0[0] * B0[0] + B1[0] * B1[0];
          V[1] += B0[1] * B0[0] + B1[1] * B1[0];
          V[2] += B0[1] * B0[1] + B1[1] * B1[1];
          V[3] += B0[2] * B0[0] + B1[2] * B1[0];
          V[4] += B0[2] * B0[1] + B1[2] * B1[1];
          V[5] += B0[2] * B0[2] + B1[2] * B1[2];
#pragma unroll
          for (int q = 0; q < 3; ++q) g[q] += B0[q] * cj.r0 + B1[q] * cj.r1;
          if (has_f)
#pragma unroll
            for (int q = 0; q < 3; ++q) wf[q] += B0[q] * cj.F0 + B1[q] * cj.F1;
        }
      }
      if (cache_ok && !reuse) {
#pragma unroll
        for (int i = 0; i < 6; ++i) vc[i] = V[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          vc[6 + i] = g[i];
          vc[9 + i] = wf[i];
        }
      }
      if (!opt_pts) continue;
      // damping (miniba.py:191-193) and 3x3 Cholesky of Vd
      V[0] += tlam * (V[0] > T(kDiagFloor) ? V[0] : T(kDiagFloor));
      V[2] += tlam * (V[2] > T(kDiagFloor) ? V[2] : T(kDiagFloor));
      V[5] += tlam * (V[5] > T(kDiagFloor) ? V[5] : T(kDiagFloor));
      const T L00 = sqrt(V[0]);
      const T i00 = T(1) / L00;
      const T L10 = V[1] * i00, L20 = V[3] * i00;
      const T L11 = sqrt(V[2] - L10 * L10);
      const T i11 = T(1) / L11;
      const T L21 = (V[4] - L20 * L10) * i11;
      const T L22 = sqrt(V[5] - L20 * L20 - L21 * L21);
      const T i22 = T(1) / L22;
      const T z0 = g[0] * i00, z1 = (g[1] - L10 * z0) * i11, z2 = (g[2] - L20 * z0 - L21 * z1) * i22;
      const T f0 = wf[0] * i00, f1 = (wf[1] - L10 * f0) * i11, f2 = (wf[2] - L20 * f0 - L21 * f1) * i22;
      part[2] += f0 * f0 + f1 * f1 + f2 * f2;
      part[3] += f0 * z0 + f1 * z1 + f2 * z2;
      T* pw = pf + (size_t)sl * PSTR;
      pw[0] = i00; pw[1] = L10; pw[2] = i11; pw[3] = L20; pw[4] = L21; pw[5] = i22;
      pw[6] = z0; pw[7] = z1; pw[8] = z2;
      pw[9] = f0; pw[10] = f1; pw[11] = f2;
    }
    if (cache_ok && !reuse) {
      pcache[2 * tid] = part[0];
      pcache[2 * tid + 1] = part[1];
    }
    {  // this CTA's focal partials
      double pd[4] = {(double)part[0], (double)part[1], (double)part[2], (double)part[3]};
#pragma unroll
      for (int i = 0; i < 4; ++i) pd[i] = (double)warp_sum(part[i]);
      if (lane == 0)
#pragma unroll
        for (int i = 0; i < 4; ++i) red[wid * 4 + i] = pd[i];
      if (tid == 0) s_job = 0;
      __syncthreads();
      if (tid < 4) {
        T s_ = T(0);
        for (int w = 0; w < NW; ++w) s_ += T(red[w * 4 + tid]);
        job[JOB_PART + tid] = s_;
      }
    }

    PROF_MARK(PH_POINT)
    // ---------- camera jobs + pair jobs (warps pull jobs from a queue) ----------
    for (;;) {
      int jb = 0;
      if (lane == 0) jb = atomicAdd(&s_job, 1);
      jb = __shfl_sync(0xffffffffu, jb, 0);
      if (jb >= nf + nb) break;
      jb = s_jorder[jb];
      if (jb < nf) {
        const int s = jb, c = cslot[s];
        const T* Rt9 = RcT + 9 * c;
        const T t0 = T(tc[3 * c]), t1 = T(tc[3 * c + 1]), t2 = T(tc[3 * c + 2]);
        T acc[UST];
#pragma unroll
        for (int i = 0; i < UST; ++i) acc[i] = T(0);
        // uniform trip count + __syncwarp per step: the lane-strided loop
        // otherwise ran with ~9 of 32 lanes active (lanes never reconverged
        // after the previous job; measured with LANES_PROF)
        const int qa = cam_ptr[c], qb = cam_ptr[c + 1];
        for (int q0 = qa; q0 < qb; q0 += 32) {
          __syncwarp();
          const int q = q0 + lane;
          if (q >= qb) continue;
          LANES_PROF(PH_LCAM, PH_NCAM)
          const int kl = perm[q];
          const float4 ob = sobs[kl];
          const int sl = __float_as_int(ob.w);
          const T* jk = jac + (size_t)kl * JSTR;
          const T J0 = jk[0], J1 = jk[1], J2 = jk[2];
          // v = R X; F = sqrt(w) (x, y)/z = (J0/f)(x, y); r (fp64) = J0 x + (J0 z/f)(c - u)
          const T X0 = T(Xs[3 * sl]), X1 = T(Xs[3 * sl + 1]), X2 = T(Xs[3 * sl + 2]);
          const T v0 = Rt9[0] * X0 + Rt9[1] * X1 + Rt9[2] * X2;
          const T v1 = Rt9[3] * X0 + Rt9[4] * X1 + Rt9[5] * X2;
          const T v2 = Rt9[6] * X0 + Rt9[7] * X1 + Rt9[8] * X2;
          const T sz = J0 * inv_f;   // sqrt(w) / z
          const T F0 = (v0 + t0) * sz, F1 = (v1 + t1) * sz;
          T r0, r1;
          if constexpr (JSTR == 5) {
            r0 = jk[3];
            r1 = jk[4];
          } else {
            double uu, vv;
            obs_uv(kl, ob, uu, vv);
            const T sw = sz * (v2 + t2);   // sqrt(w)
            r0 = J0 * (v0 + t0) + sw * T(cx - uu);
            r1 = J0 * (v1 + t1) + sw * T(cy - vv);
          }
          T a[12];
          expand_A(J0, J1, J2, v0, v1, v2, a);
          // self co-observation product of the diagonal block, folded in:
          // U_aa - Y_i Y_i^T = A^T A - A^T (Q Q^T) A = A^T (A - P), P = (Q Q^T) A
          T p[12];
#pragma unroll
          for (int i = 0; i < 12; ++i) p[i] = T(0);
          if (opt_pts) {
            const T* pw = pf + (size_t)sl * PSTR;
            T qv[6];
            q_rows(J0, J1, J2, Rt9, pw, qv);
            const T qf0 = qv[0] * pw[9] + qv[1] * pw[10] + qv[2] * pw[11];
            const T qf1 = qv[3] * pw[9] + qv[4] * pw[10] + qv[5] * pw[11];
            const T qz0 = qv[0] * pw[6] + qv[1] * pw[7] + qv[2] * pw[8];
            const T qz1 = qv[3] * pw[6] + qv[4] * pw[7] + qv[5] * pw[8];
            const T m00 = qv[0] * qv[0] + qv[1] * qv[1] + qv[2] * qv[2];
            const T m01 = qv[0] * qv[3] + qv[1] * qv[4] + qv[2] * qv[5];
            const T m11 = qv[3] * qv[3] + qv[4] * qv[4] + qv[5] * qv[5];
#pragma unroll
            for (int r = 0; r < 6; ++r) {
              acc[33 + r] += a[r] * qf0 + a[6 + r] * qf1;
              acc[39 + r] += a[r] * qz0 + a[6 + r] * qz1;
              p[r] = m00 * a[r] + m01 * a[6 + r];
              p[6 + r] = m01 * a[r] + m11 * a[6 + r];
            }
          }
          int idx = 0;
#pragma unroll
          for (int r = 0; r < 6; ++r) {
#pragma unroll
            for (int cc = 0; cc <= r; ++cc) acc[idx++] += a[r] * (a[cc] - p[cc]) + a[6 + r] * (a[6 + cc] - p[6 + cc]);
            acc[21 + r] += a[r] * F0 + a[6 + r] * F1;
            acc[27 + r] += a[r] * r0 + a[6 + r] * r1;
            acc[45 + r] += a[r] * a[r] + a[6 + r] * a[6 + r];
          }
        }
        warp_reduce_to<T, UST>(acc, job + s * UST, lane);
      } else {
        const int blk = jb - nf;
        if (blk_off[blk + 1] == blk_off[blk]) {   // no co-observations (e.g. diagonal blocks)
          T* o = job + JOB_PAIR0 + blk * 36;
          for (int i = lane; i < 36; i += 32) o[i] = T(0);
          continue;
        }
        const int ca = cslot[blk_a[blk]], cbb = cslot[blk_b[blk]];
        // rotations read from shared memory (uniform broadcast loads) rather
        // than held in registers: keeps the fp64 job within the register budget
        const T* Ra = RcT + 9 * ca;
        const T* Rb = RcT + 9 * cbb;
        T acc[36];
#pragma unroll
        for (int i = 0; i < 36; ++i) acc[i] = T(0);
        const int q1 = blk_off[blk + 1];
        for (int q0 = blk_off[blk]; q0 < q1; q0 += 32) {
          __syncwarp();
          const int q = q0 + lane;
          if (q >= q1) continue;
          LANES_PROF(PH_LPAIR, PH_NPAIR)
          const unsigned pr = pairs[q];
          const int i = (int)(pr >> 16), j = (int)(pr & 0xffffu);
          const int sl = __float_as_int(sobs[i].w);
          const T* pw = pf + (size_t)sl * PSTR;
          const T* ji = jac + (size_t)i * JSTR;
          const T* jj = jac + (size_t)j * JSTR;
          const T Ji0 = ji[0], Ji1 = ji[1], Ji2 = ji[2];
          const T Jj0 = jj[0], Jj1 = jj[1], Jj2 = jj[2];
          // v_i = R_a X_p, v_j = R_b X_p (same point)
          const T X0 = T(Xs[3 * sl]), X1 = T(Xs[3 * sl + 1]), X2 = T(Xs[3 * sl + 2]);
          const T vi0 = Ra[0] * X0 + Ra[1] * X1 + Ra[2] * X2;
          const T vi1 = Ra[3] * X0 + Ra[4] * X1 + Ra[5] * X2;
          const T vi2 = Ra[6] * X0 + Ra[7] * X1 + Ra[8] * X2;
          const T vj0 = Rb[0] * X0 + Rb[1] * X1 + Rb[2] * X2;
          const T vj1 = Rb[3] * X0 + Rb[4] * X1 + Rb[5] * X2;
          const T vj2 = Rb[6] * X0 + Rb[7] * X1 + Rb[8] * X2;
          T qi[6], qj[6];
          q_rows(Ji0, Ji1, Ji2, Ra, pw, qi);
          q_rows(Jj0, Jj1, Jj2, Rb, pw, qj);
          // M = Q_i Q_j^T (2x2)
          const T m00 = qi[0] * qj[0] + qi[1] * qj[1] + qi[2] * qj[2];
          const T m01 = qi[0] * qj[3] + qi[1] * qj[4] + qi[2] * qj[5];
          const T m10 = qi[3] * qj[0] + qi[4] * qj[1] + qi[5] * qj[2];
          const T m11 = qi[3] * qj[3] + qi[4] * qj[4] + qi[5] * qj[5];
          // N = M Jp_j (2x3), M3 = Jp_i^T N (3x3)
          const T n00 = m00 * Jj0, n01 = m01 * Jj0, n02 = m00 * Jj1 + m01 * Jj2;
          const T n10 = m10 * Jj0, n11 = m11 * Jj0, n12 = m10 * Jj1 + m11 * Jj2;
          T M3[9];
          M3[0] = Ji0 * n00; M3[1] = Ji0 * n01; M3[2] = Ji0 * n02;
          M3[3] = Ji0 * n10; M3[4] = Ji0 * n11; M3[5] = Ji0 * n12;
          M3[6] = Ji1 * n00 + Ji2 * n10; M3[7] = Ji1 * n01 + Ji2 * n11; M3[8] = Ji1 * n02 + Ji2 * n12;
          // H = M3 G_j = [E | M3], E row r = -(M3 row r) x v_j
          T H[18];  // row-major 3x6
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const T a0 = M3[3 * r], a1 = M3[3 * r + 1], a2 = M3[3 * r + 2];
            H[6 * r + 0] = a2 * vj1 - a1 * vj2;
            H[6 * r + 1] = a0 * vj2 - a2 * vj0;
            H[6 * r + 2] = a1 * vj0 - a0 * vj1;
            H[6 * r + 3] = a0;
            H[6 * r + 4] = a1;
            H[6 * r + 5] = a2;
          }
          // block = G_i^T H = [[v_i]x H ; H]
#pragma unroll
          for (int cc = 0; cc < 6; ++cc) {
            const T h0 = H[cc], h1 = H[6 + cc], h2 = H[12 + cc];
            acc[0 * 6 + cc] += vi1 * h2 - vi2 * h1;
            acc[1 * 6 + cc] += vi2 * h0 - vi0 * h2;
            acc[2 * 6 + cc] += vi0 * h1 - vi1 * h0;
            acc[3 * 6 + cc] += h0;
            acc[4 * 6 + cc] += h1;
            acc[5 * 6 + cc] += h2;
          }
        }
        warp_reduce_to<T, 36>(acc, job + JOB_PAIR0 + blk * 36, lane);
      }
    }
    Clu<R>::sync();  // every CTA's job outputs are complete and visible
    // cluster totals of the job outputs, summed in rank order on access
    const T* rjob[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rjob[r] = Clu<R>::remote(job, r);
    auto jsum_at = [&](int i) {
      T s_ = rjob[0][i];
#pragma unroll
      for (int r = 1; r < R; ++r) s_ += rjob[r][i];
      return s_;
    };
    PROF_MARK(PH_JOBS)
    // ---------- assemble the damped augmented reduced system (miniba.py:188-213) ----------
    for (int e = tid; e < CA; e += NT) {
      const unsigned ij = tab[e];
      const int i = (int)(ij >> 8), j = (int)(ij & 255u);
      T val;
      if (i == C) {                       // rhs row
        if (j == FI && has_f) {
          val = -jsum_at(JOB_PART + 1) + (opt_pts ? jsum_at(JOB_PART + 3) : T(0));
        } else {
          const int u = (j / 6) * UST;
          val = -jsum_at(u + 27 + j % 6) + (opt_pts ? jsum_at(u + 39 + j % 6) : T(0));
        }
      } else if (has_f && i == FI) {      // focal row
        if (j == FI) {
          const T uff = jsum_at(JOB_PART + 0);
          val = uff + tlam * (uff > T(kDiagFloor) ? uff : T(kDiagFloor)) -
                (opt_pts ? jsum_at(JOB_PART + 2) : T(0));
        } else {
          const int u = (j / 6) * UST;
          val = jsum_at(u + 21 + j % 6) - (opt_pts ? jsum_at(u + 33 + j % 6) : T(0));
        }
      } else {                            // camera-camera: i >= j
        const int sb = i / 6, sa = j / 6, ri = i % 6, rj = j % 6;
        T schur = T(0);
        val = T(0);
        if (sa == sb) {
          const int r = ri, cc = rj;  // r >= cc
          T ud = jsum_at(sa * UST + r * (r + 1) / 2 + cc);   // U_aa - sum_self Y Y^T
          if (r == cc) {
            const T u0 = jsum_at(sa * UST + 45 + r);         // U_aa diagonal (damping, miniba.py:190)
            ud += tlam * (u0 > T(kDiagFloor) ? u0 : T(kDiagFloor));
          }
          val = ud;
          if (opt_pts) {
            const int q = sa * nf - sa * (sa - 1) / 2;   // block (sa, sa)
            schur = jsum_at(JOB_PAIR0 + q * 36 + r * 6 + cc);
          }
        } else if (opt_pts) {
          const int q = sa * nf - sa * (sa - 1) / 2 + (sb - sa);   // block (sa, sb)
          schur = jsum_at(JOB_PAIR0 + q * 36 + rj * 6 + ri);
        }
        val -= schur;
      }
      S[e] = val;
    }
    __syncthreads();

    PROF_MARK(PH_ASM)
    // ---------- LDL^T of the augmented system ----------
    // Right-looking, two pivots per step and ONE barrier per step: pivots k and
    // k+1 (d_k, l = S[k+1][k]/d_k, d_{k+1} = S[k+1][k+1] - l S[k+1][k]) are
    // formed redundantly by every thread, the trailing entries get the rank-2
    // update with column k+1 corrected on the fly, and column k+1 itself is
    // finalised lazily during the next step (nobody reads it there). Each
    // thread owns fixed packed entries whose (row, column) stay in registers;
    // reciprocals are MUFU-seeded with Newton refinement in fp64. S[k][k] keeps
    // d_k, S[i][k] keeps L_ik d_k; the rhs row C receives y = L^-1 b.
    // (B200: a shared store -> barrier -> load round trip costs ~200 cycles,
    // scripts/micro/ldl_bench.cu; this variant measured 14.8k cycles for C=43
    // in fp64 against 22.1k for one barrier per column.)
    bool chol_fail = false;
    {
      constexpr int E = (CA_MAX + NT - 1) / NT;
      int ii[E], jj[E];
#pragma unroll
      for (int u = 0; u < E; ++u) {
        const int e = tid + u * NT;
        const unsigned ij = e < CA ? tab[e] : 0u;
        ii[u] = e < CA ? (int)(ij >> 8) : 0;
        jj[u] = e < CA ? (int)(ij & 255u) : -1;
      }
      auto bad_pivot = [](T d) { return !(d > T(0)) || !isfinite(d); };
      int k = 0, pend = -1;   // pend: column awaiting its rank-1 finalisation
      for (; k + 1 < C; k += 2) {
        const T* colk = S + acol(k, C) - k;
        const T* colk1 = S + acol(k + 1, C) - (k + 1);
        const T d0 = colk[k], a10 = colk[k + 1], d1r = colk1[k + 1];
        if (bad_pivot(d0)) {
          chol_fail = true;
          break;
        }
        const T i0 = fast_rcp(d0);
        const T l10 = a10 * i0;
        const T d1 = d1r - l10 * a10;
        if (bad_pivot(d1)) {
          chol_fail = true;
          break;
        }
        const T i1 = fast_rcp(d1);
        if (tid == 0) {
          invd[k] = i0;
          invd[k + 1] = i1;
          l10s[k] = l10;
        }
#pragma unroll
        for (int u = 0; u < E; ++u) {
          if (jj[u] >= k + 2) {
            const int e = tid + u * NT;
            const T ai = colk[ii[u]], aj = colk[jj[u]], ci = colk1[ii[u]], cj = colk1[jj[u]];
            const T sv = S[e];
            const T ci1 = ci - ai * l10, cj1 = cj - aj * l10;
            S[e] = sv - ai * aj * i0 - ci1 * cj1 * i1;
          }
        }
        if (pend >= 0) {   // finalise column pend (= k - 1) against column pend - 1
          T* cp = S + acol(pend, C) - pend;
          const T* cq = S + acol(pend - 1, C) - (pend - 1);
          const T lp = l10s[pend - 1];
          for (int i = pend + tid; i <= C; i += NT) cp[i] = cp[i] - cq[i] * lp;
        }
        pend = k + 1;
        __syncthreads();
      }
      if (!chol_fail) {
        if (pend >= 0) {
          T* cp = S + acol(pend, C) - pend;
          const T* cq = S + acol(pend - 1, C) - (pend - 1);
          const T lp = l10s[pend - 1];
          for (int i = pend + tid; i <= C; i += NT) cp[i] = cp[i] - cq[i] * lp;
          __syncthreads();
        }
        if (k < C) {   // odd C: the last pivot alone
          const T* colk = S + acol(k, C) - k;
          const T d = colk[k];
          if (bad_pivot(d)) {
            chol_fail = true;
          } else {
            const T inv = fast_rcp(d);
#pragma unroll
            for (int u = 0; u < E; ++u)
              if (jj[u] > k) S[tid + u * NT] -= colk[ii[u]] * colk[jj[u]] * inv;
            if (tid == 0) invd[k] = inv;
          }
          __syncthreads();
        }
      }
    }
    PROF_MARK(PH_CHA)
    if (it < 64 && ((cfg.fail_iters_mask >> it) & 1ull)) chol_fail = true;
    PROF_MARK(PH_CHOL)

    if (!chol_fail) {
      // column-oriented back substitution D L^T x = y in warp 0 (no reductions):
      // x_k = u_k / d_k, then u_j -= S[k][j] x_k for j < k
      if (wid == 0) {
        T u0 = lane < C ? S[acol(lane, C) + C - lane] : T(0);
        T u1 = lane + 32 < C ? S[acol(lane + 32, C) + C - lane - 32] : T(0);
        for (int k = C - 1; k >= 0; --k) {
          const T uk = __shfl_sync(0xffffffffu, k < 32 ? u0 : u1, k & 31);
          const T xk = uk * invd[k];
          if (lane == (k & 31)) {
            if (k < 32) u0 = xk; else u1 = xk;
          }
          if (lane < k) u0 -= S[acol(lane, C) + k - lane] * xk;
          if (lane + 32 < k) u1 -= S[acol(lane + 32, C) + k - lane - 32] * xk;
        }
        if (lane < C) { dc[lane] = (double)u0; dcT[lane] = u0; }
        if (lane + 32 < C) { dc[lane + 32] = (double)u1; dcT[lane + 32] = u1; }
      }
      __syncthreads();
      PROF_MARK(PH_CHB)
      // trial cameras of all five tries (R <- exp(frac dw) R, t + frac dt,
      // miniba.py:264-266), by the highest-numbered threads, overlapped with
      // the point back substitution (the barrier after it publishes both)
      for (int q = NT - 1 - tid; q < kBacktrackTries * n; q += NT) {
        const int bt = q / n, c = q % n, s = slot[c];
        const double frac = ldexp(1.0, -bt);
        double* Rq = Rt + (size_t)(bt * n + c) * 9;
        double* tq = tt + (size_t)(bt * n + c) * 3;
        if (s < 0) {
          for (int i = 0; i < 9; ++i) Rq[i] = Rc[9 * c + i];
          for (int i = 0; i < 3; ++i) tq[i] = tc[3 * c + i];
        } else {
          double w[3] = {frac * dc[6 * s], frac * dc[6 * s + 1], frac * dc[6 * s + 2]};
          double E[9];
          exp_so3(w, E);
          matmul33(E, Rc + 9 * c, Rq);
          for (int i = 0; i < 3; ++i) tq[i] = tc[3 * c + i] + frac * dc[6 * s + 3 + i];
        }
      }
      const bool gauge = sizeof(T) == 4 && s_gcam >= 0;
      double c0[3] = {0.0, 0.0, 0.0}, gacc[2] = {0.0, 0.0};
      double gDp = 0.0;
      if (gauge) {
        const int g = s_gcam;
#pragma unroll
        for (int i = 0; i < 3; ++i)
          c0[i] = -(Rc[9 * g + i] * tc[3 * g] + Rc[9 * g + 3 + i] * tc[3 * g + 1] + Rc[9 * g + 6 + i] * tc[3 * g + 2]);
        gDp = 1.0 / (1.0 + lam);
      }
      // point back substitution (miniba.py:216-217): dp = -L^-T (z + yf df + sum Y_i^T dc_a)
      if (opt_pts) {
        const T df = has_f ? dcT[FI] : T(0);
        for (int sl = tid; sl < nlp; sl += NT) {
          T* pw = pf + (size_t)sl * PSTR;
          const T X0 = T(Xs[3 * sl]), X1 = T(Xs[3 * sl + 1]), X2 = T(Xs[3 * sl + 2]);
          T u0 = pw[6] + pw[9] * df, u1 = pw[7] + pw[10] * df, u2 = pw[8] + pw[11] * df;
          for (int kl = ptr[sl]; kl < ptr[sl + 1]; ++kl) {
            const int c = __float_as_int(sobs[kl].z);
            const int s = slot[c];
            if (s < 0) continue;
            const T* jk = jac + (size_t)kl * JSTR;
            const T J0 = jk[0], J1 = jk[1], J2 = jk[2];
            const T* Rk = RcT + 9 * c;
            const T v0 = Rk[0] * X0 + Rk[1] * X1 + Rk[2] * X2;
            const T v1 = Rk[3] * X0 + Rk[4] * X1 + Rk[5] * X2;
            const T v2 = Rk[6] * X0 + Rk[7] * X1 + Rk[8] * X2;
            const T* dca = dcT + 6 * s;
            const T w0 = dca[0], w1 = dca[1], w2 = dca[2];
            // G dc = -(v x w) + dt ; A dc = Jp (G dc)
            const T g0 = -(v1 * w2 - v2 * w1) + dca[3];
            const T g1 = -(v2 * w0 - v0 * w2) + dca[4];
            const T g2 = -(v0 * w1 - v1 * w0) + dca[5];
            const T ad0 = J0 * g0 + J1 * g2, ad1 = J0 * g1 + J2 * g2;
            T qv[6];
            q_rows(J0, J1, J2, RcT + 9 * c, pw, qv);
            u0 += qv[0] * ad0 + qv[3] * ad1;
            u1 += qv[1] * ad0 + qv[4] * ad1;
            u2 += qv[2] * ad0 + qv[5] * ad1;
          }
          const T iL00 = pw[0], L10 = pw[1], iL11 = pw[2], L20 = pw[3], L21 = pw[4], iL22 = pw[5];
          const T x2 = u2 * iL22;
          const T x1 = (u1 - L21 * x2) * iL11;
          const T x0 = (u0 - L10 * x1 - L20 * x2) * iL00;
          pw[PDP] = -x0;
          pw[PDP + 1] = -x1;
          pw[PDP + 2] = -x2;
          if (gauge) {   // n_p^T D_p dp, n_p^T D_p n_p (step projection below)
            const double l00 = 1.0 / (double)iL00, l11 = 1.0 / (double)iL11, l22 = 1.0 / (double)iL22;
            const double Dp[3] = {l00 * l00 * gDp, ((double)L10 * L10 + l11 * l11) * gDp,
                                  ((double)L20 * L20 + (double)L21 * L21 + l22 * l22) * gDp};
            const double xs[3] = {-(double)x0, -(double)x1, -(double)x2};
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              const double nv = Xs[3 * sl + i] - c0[i];
              gacc[0] += nv * Dp[i] * xs[i];
              gacc[1] += nv * nv * Dp[i];
            }
          }
        }
      }
      if (gauge) {
        // Gauge-consistent step (fp32 Schur only). With one fixed camera the
        // cost is invariant under scaling the scene about that camera's centre
        // c0: H n = 0 and g.n = 0 for n = (dt_c = t_c + R_c c0, dX_p = X_p - c0),
        // so the exact damped step (H + lam D) d = -g satisfies n^T D d = 0
        // (D = max(diag H, 1e-12), miniba.py:188-193). fp32 Jacobians break the
        // invariance at the 1e-7 level and, with lam -> 1e-15, the solve then
        // moves freely along n (config 4: translations 5e-4 off the fp64
        // reference at identical cost). Restore the exact-arithmetic property
        // by removing the D-weighted component along n.
        double acc[2] = {gacc[0], gacc[1]};
        block_sum_d<NW, 2>(acc, red);
        cluster_sum<R, 2>(acc, xch, epoch);
        for (int s = 0; s < nf; ++s) {   // camera part: identical in every thread
          const int c = cslot[s];
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const double nv = tc[3 * c + i] + Rc[9 * c + 3 * i] * c0[0] + Rc[9 * c + 3 * i + 1] * c0[1] +
                              Rc[9 * c + 3 * i + 2] * c0[2];
            const double u = (double)jsum_at(s * UST + 45 + 3 + i);
            const double Dc = u > kDiagFloor ? u : kDiagFloor;
            acc[0] += nv * Dc * dc[6 * s + 3 + i];
            acc[1] += nv * nv * Dc;
          }
        }
        const double alpha = acc[1] > 0.0 ? acc[0] / acc[1] : 0.0;
        __syncthreads();   // every thread has read dc; the trial cameras are complete
        for (int sl = tid; sl < nlp; sl += NT) {
          T* pw = pf + (size_t)sl * PSTR;
#pragma unroll
          for (int i = 0; i < 3; ++i) pw[PDP + i] = T((double)pw[PDP + i] - alpha * (Xs[3 * sl + i] - c0[i]));
        }
        for (int q = tid; q < 3 * nf; q += NT) {
          const int s = q / 3, i = q % 3, c = cslot[s];
          const double nv = tc[3 * c + i] + Rc[9 * c + 3 * i] * c0[0] + Rc[9 * c + 3 * i + 1] * c0[1] +
                            Rc[9 * c + 3 * i + 2] * c0[2];
          dc[6 * s + 3 + i] -= alpha * nv;
          for (int bt = 0; bt < kBacktrackTries; ++bt)
            tt[(size_t)(bt * n + c) * 3 + i] = tc[3 * c + i] + ldexp(1.0, -bt) * dc[6 * s + 3 + i];
        }
      }
    }

    __syncthreads();
    PROF_MARK(PH_SOLVE)
    // ---------- trials, accept / reject, lambda (miniba.py:244-293) ----------
    if (lead) lambdas[it] = lam;
    int tries = 0, took = -1;
    double tc_[3] = {0, 0, 0};
    double ft = f;
    if (!chol_fail) {
      // try 0 (the full step) alone; if it is rejected, tries 1..4 in one
      // fused pass. `tries` keeps the reference's count (first accepted try + 1,
      // or 5), miniba.py:262-276.
      ft = has_f ? f + dc[FI] : f;
      cost(std::false_type(), Rt, tt, ft, 1.0, opt_pts, tc_);
      tries = 1;
      if (tc_[0] < cur && isfinite(tc_[0])) {
        took = 0;
      } else {
        double fts[4], c4[4];
#pragma unroll
        for (int bt = 1; bt < kBacktrackTries; ++bt)
          fts[bt - 1] = has_f ? f + (1.0 / (double)(1 << bt)) * dc[FI] : f;
        cost4(fts, c4);
        tries = kBacktrackTries;
        for (int bt = 1; bt < kBacktrackTries; ++bt) {
          if (c4[bt - 1] < cur && isfinite(c4[bt - 1])) {
            took = bt;
            tries = bt + 1;
            tc_[0] = c4[bt - 1];
            ft = fts[bt - 1];
            break;
          }
        }
      }
    } else {
      Clu<R>::sync();  // job buffers are rewritten next iteration: peers must be done reading
    }
    PROF_MARK(PH_TRIAL)
    if (lead) evals[it] = (uint8_t)tries;
    bool stop = false;
    if (took >= 0) {
      const double frac = ldexp(1.0, -took);
      for (int i = tid; i < n * 9; i += NT) Rc[i] = Rt[(size_t)took * n * 9 + i];
      for (int i = tid; i < n * 3; i += NT) tc[i] = tt[(size_t)took * n * 3 + i];
      for (int i = tid; i < n * 9; i += NT) RcT[i] = T(Rt[(size_t)took * n * 9 + i]);
      if (opt_pts)
        for (int i = tid; i < nlp * 3; i += NT) {
          const T* dp = pf + (size_t)(i / 3) * PSTR + PDP;
          Xs[i] = Xs[i] + frac * (double)dp[i % 3];
        }
      f = ft;
      lam = took == 0 ? fmax(lam / nu, 1e-15) : fmin(lam * nu, kLambdaMax);
      const double improve = cur - tc_[0];
      cur = tc_[0];
      if (lead) accepted[it] = 1;
      if (improve <= 1e-15 * fmax(cur, 1.0)) {
        stop = true;
        stop_reason = MBA_SOLVE_CONVERGED;
      }
    } else {
      lam = fmin(lam * nu, kLambdaMax);
      if (lead) accepted[it] = 0;
      if (!chol_fail && lam >= kLambdaMax) {
        stop = true;
        stop_reason = MBA_SOLVE_LAMBDA_CAP;
      }
    }
    if (lead) costs[it + 1] = cur;
    reuse = cache_ok && took < 0;   // parameters unchanged: the next linearisation is this one
    ++it;
    __syncthreads();
    PROF_MARK(PH_COMMIT)
    if (stop) break;
  }

  // ---------------- outputs ----------------
  cost(std::true_type(), Rc, tc, f, 0.0, false, st);   // sum e, sum e^2 of the final state
  const double se = st[1], se2 = st[2];
  for (int i = tid; i < nlp * 3; i += NT) O.points_out[(pb + lpt[i / 3]) * 3 + i % 3] = Xs[i];
  if (rank == 0) {
    for (int i = tid; i < n * 9; i += NT) O.R_out[cb * 9 + i] = Rc[i];
    for (int i = tid; i < n * 3; i += NT) O.t_out[cb * 3 + i] = tc[i];
  }
  if (lead) {
    O.focal_out[b] = f;
    O.n_iters[b] = it;
    O.status[b] = stop_reason;
    O.final_stats[4 * b + 0] = cur;
    O.final_stats[4 * b + 1] = se;
    O.final_stats[4 * b + 2] = se2;
    O.final_stats[4 * b + 3] = (double)K;
  }
  PROF_FLUSH
  Clu<R>::sync();  // no CTA leaves while a peer may still read its shared memory
}

template <typename T, int R, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) solve_v4_kernel(Params P) {
  extern __shared__ __align__(16) unsigned char smem[];
  solve_problem<T, R, NT>(P, smem);
}

// ---------------------------------------------------------------------------
// host side

template <typename T>
static size_t need_bytes(const MbaBatchDesc* d, int R) {
  const int64_t mt = d->max_track > 0 ? d->max_track : d->max_obs;
  const int64_t obs = (d->max_obs + R - 1) / R + mt;
  const int64_t pts = (d->max_points + R - 1) / R + mt;
  const int64_t prs = (d->max_pairs + R - 1) / R + mt * mt;
  return Fixed<T>::kBytes + obs * obs_bytes<T>() + pts * pt_bytes<T>() + 4 * prs + 8 * 16;
}

// dynamic shared memory a CTA can use at `per_sm` CTAs per SM (228 KB per SM,
// 1 KB reserved per CTA, static shared memory of the kernel excluded)
static size_t smem_per_cta(int per_sm, size_t static_bytes) {
  size_t per = (228 * 1024) / (size_t)per_sm - 1024 - static_bytes;
  return per < kSmemLimit - static_bytes ? per : kSmemLimit - static_bytes;
}

struct Plan {
  int R, nt, per_sm;
};

// Clusters of R CTAs the device keeps resident at once (a cluster must fit in
// one GPC, so this is not 148 / R). Cached per process (one device per rank).
template <typename T, int R>
static int active_clusters_t() {
  static int cached = -1;
  if (cached >= 0) return cached;
  auto kern = solve_v4_kernel<T, R, 256, 1>;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return cached = 0;
  const size_t smem = smem_per_cta(1, fa.sharedSizeBytes);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (R > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(R * 1024);
  lc.blockDim = dim3(256);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = R;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &lc) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  return cached = n;
}

template <typename T>
static int active_clusters(int R) {
  switch (R) {
    case 8: return active_clusters_t<T, 8>();
    case 9: return active_clusters_t<T, 9>();
    case 10: return active_clusters_t<T, 10>();
    case 12: return active_clusters_t<T, 12>();
    case 16: return active_clusters_t<T, 16>();
  }
  return 0;
}

// Smallest cluster that fits (every CTA of a cluster repeats the serial
// phases -- LDL^T, substitutions, step control -- so splitting a problem costs
// more than it gains; measured on config 4: R=1 247k problems/s (mixed) vs R=2
// 149k); at equal R prefer two co-resident problems per SM. Overrides:
// MBA_V4_R, MBA_V4_NT, MBA_V4_PERSM.
template <typename T>
static Plan plan_t(const MbaBatchDesc* d) {
  const int eR = getenv("MBA_V4_R") ? atoi(getenv("MBA_V4_R")) : 0;
  const int eP = getenv("MBA_V4_PERSM") ? atoi(getenv("MBA_V4_PERSM")) : 0;
  const int eN = getenv("MBA_V4_NT") ? atoi(getenv("MBA_V4_NT")) : 0;
  const size_t st = 256;   // static shared memory bound
  // Clusters are placed inside one GPC (B200: 18-20 SMs each), so a cluster
  // size that divides a GPC poorly strands SMs: R = 8 runs 2 clusters per GPC
  // (16 of 18 SMs busy), R = 16 one (16 of 18). For batches that fill the GPU
  // the planner also tries R = 6 and R = 9 (3 / 2 clusters, 18 SMs busy, and
  // less per-CTA work than the next power of two); small batches keep the
  // powers of two, where a larger cluster only shortens the single solve.
  //
  // When the smallest fit is R >= 8 on such a batch, every fitting R in
  // {8, 9, 10, 12, 16} is scored by resident clusters x R / (R + 7): the
  // second factor models a cluster's solve speed-up with R (serial phases are
  // repeated per CTA; fitted to config 3 on B200: R = 8 / 9 / 10 / 12 / 16 run
  // 15 / 15 / 11 / 7 / 7 clusters, best f64 R = 10 at 20.0k problems/s vs
  // 12.5k at R = 16, best mixed R = 9 at 31.4k vs 29.8k at R = 8).
  const bool wide = d->n_problems >= 64;
  if (wide && !eR && !eP && !eN && need_bytes<T>(d, 4) > smem_per_cta(1, st)) {
    int best = 0;
    double best_s = 0.0;
    for (int R : {8, 9, 10, 12, 16}) {
      if (need_bytes<T>(d, R) > smem_per_cta(1, st)) continue;
      const double sc = active_clusters<T>(R) * (double)R / (R + 7.0);
      if (getenv("MBA_DEBUG")) fprintf(stderr, "mba v4 plan score R=%d: %.2f\n", R, sc);
      if (sc > best_s) {
        best_s = sc;
        best = R;
      }
    }
    if (best) return Plan{best, 256, 1};
  }
  for (int R : {1, 2, 4, 8, 9, 10, 12, 16}) {
    if (eR && R != eR) continue;
    if (!eR && (R == 9 || R == 10 || R == 12)) continue;
    for (int per_sm : {2, 1}) {
      if (eP && per_sm != eP) continue;
      if (per_sm == 2 && R > 4) continue;
      if (need_bytes<T>(d, R) <= smem_per_cta(per_sm, st)) {
        // one problem per SM: fp32 arithmetic fits 512 threads in 128 registers
        // (config 4 mixed: 324k problems/s at 512 vs 283k at 256); fp64 needs
        // the register room of 256 threads
        int nt = per_sm == 2 ? (sizeof(T) == 8 ? 128 : 256) : (sizeof(T) == 4 && R == 1 ? 512 : 256);
        if (eN == 128 || eN == 256 || (per_sm == 1 && R == 1 && (eN == 384 || eN == 512))) nt = eN;
        if (per_sm == 2 && sizeof(T) == 8) nt = 128;   // 255 registers need 128 threads at 2 CTAs/SM
        return Plan{R, nt, per_sm};
      }
    }
  }
  return Plan{0, 0, 0};
}

template <typename T, int R, int NT, int MINB>
static int launch_t(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o, cudaStream_t st,
                    void* ws, size_t ws_bytes) {
  auto kern = solve_v4_kernel<T, R, NT, MINB>;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return MBA_ERR_CUDA;
  const size_t need = need_bytes<T>(d, R);
  // take all the shared memory a CTA gets at this occupancy (slack for
  // unbalanced slices before the overflow fallback triggers)
  const size_t smem = smem_per_cta(MINB, fa.sharedSizeBytes);
  if (need > smem) return MBA_ERR_TOO_LARGE;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    if (getenv("MBA_DEBUG")) fprintf(stderr, "mba v4 smem attribute %zu rejected\n", smem);
    return MBA_ERR_CUDA;
  }
  if (R > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  Params P;
  P.d = *d;
  P.cfg = *cfg;
  P.o = *o;
  P.arena = smem - Fixed<T>::kBytes;
  P.gcache = nullptr;
  P.gcache_slot = 0;
  P.gcache_slots = 0;
  if (MINB == 1 && ws != nullptr) {   // one CTA per SM: per-SM linearisation caches in the workspace
    int dev = 0, n_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const size_t slot = al16(sizeof(T) * (13 * (size_t)d->max_points + 2 * NT));
    if (n_sm > 0 && slot * (size_t)n_sm <= ws_bytes) {
      P.gcache = static_cast<unsigned char*>(ws);
      P.gcache_slot = slot;
      P.gcache_slots = n_sm;
    }
  }
  if (const char* e = getenv("MBA_V4_ARENA_CAP")) {   // tests: force the overflow re-solve path
    const size_t cap = (size_t)atol(e);
    if (cap < P.arena) P.arena = cap;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)d->n_problems * R);
  lc.blockDim = dim3(NT);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = R;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  if (getenv("MBA_DEBUG")) {
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, kern, &lc);
    fprintf(stderr, "mba v4 R=%d NT=%d: %d active clusters (%d SMs busy)\n", R, NT, ncl, ncl * R);
  }
  const cudaError_t err = cudaLaunchKernelEx(&lc, kern, P);
  if (err != cudaSuccess && getenv("MBA_DEBUG"))
    fprintf(stderr, "mba v4 launch (R=%d, NT=%d, smem=%zu): %s\n", R, NT, smem, cudaGetErrorString(err));
  return err == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}

template <typename T>
static int launch_prec(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o, cudaStream_t st,
                       const Plan& p, void* ws, size_t ws_bytes) {
  if (getenv("MBA_DEBUG")) fprintf(stderr, "mba v4 plan: R=%d NT=%d per_sm=%d\n", p.R, p.nt, p.per_sm);
  if (p.per_sm == 2) {
    if (p.nt == 128) {
      switch (p.R) {
        case 1: return launch_t<T, 1, 128, 2>(d, cfg, o, st, ws, ws_bytes);
        case 2: return launch_t<T, 2, 128, 2>(d, cfg, o, st, ws, ws_bytes);
        case 4: return launch_t<T, 4, 128, 2>(d, cfg, o, st, ws, ws_bytes);
      }
    } else if constexpr (sizeof(T) == 4) {
      switch (p.R) {
        case 1: return launch_t<T, 1, 256, 2>(d, cfg, o, st, ws, ws_bytes);
        case 2: return launch_t<T, 2, 256, 2>(d, cfg, o, st, ws, ws_bytes);
        case 4: return launch_t<T, 4, 256, 2>(d, cfg, o, st, ws, ws_bytes);
      }
    }
    return MBA_ERR_TOO_LARGE;
  }
  if (p.nt == 512 && p.R == 1) return launch_t<T, 1, 512, 1>(d, cfg, o, st, ws, ws_bytes);
  if (p.nt == 384 && p.R == 1) return launch_t<T, 1, 384, 1>(d, cfg, o, st, ws, ws_bytes);
  switch (p.R) {
    case 1: return launch_t<T, 1, 256, 1>(d, cfg, o, st, ws, ws_bytes);
    case 2: return launch_t<T, 2, 256, 1>(d, cfg, o, st, ws, ws_bytes);
    case 4: return launch_t<T, 4, 256, 1>(d, cfg, o, st, ws, ws_bytes);
    case 8: return launch_t<T, 8, 256, 1>(d, cfg, o, st, ws, ws_bytes);
    case 9: return launch_t<T, 9, 256, 1>(d, cfg, o, st, ws, ws_bytes);
    case 10: return launch_t<T, 10, 256, 1>(d, cfg, o, st, ws, ws_bytes);
    case 12: return launch_t<T, 12, 256, 1>(d, cfg, o, st, ws, ws_bytes);
    case 16: return launch_t<T, 16, 256, 1>(d, cfg, o, st, ws, ws_bytes);
    default: return MBA_ERR_TOO_LARGE;
  }
}

// Exact shared-memory need of the largest problem on a one-CTA plan (the
// descriptor maxima bound every problem's slice): when it fits, no problem can
// overflow and the re-solve launch is skipped.
template <typename T>
static bool may_overflow_t(const MbaBatchDesc* d, const Plan& p) {
  if (p.R != 1 || getenv("MBA_V4_ARENA_CAP")) return true;
  const size_t nlo = (size_t)d->max_obs, nlp = (size_t)d->max_points;
  const size_t need = al16(16 * nlo) + al16(24 * nlp) + al16(sizeof(T) * jstr<T>() * nlo) +
                      al16(sizeof(T) * PSTR * nlp) + al16(4 * nlp) + al16(2 * nlo) + al16(2 * (nlp + 1)) +
                      4 * (size_t)d->max_pairs;
  const size_t arena = smem_per_cta(p.per_sm, 256) - Fixed<T>::kBytes;
  return nlo >= 65535 || need > arena;
}

// one arithmetic type per translation unit (see mba_v4.cuh)
#ifdef MBA_V4_F32
using TU = float;
#define V4_ENTRY(x) x##_f32
#else
using TU = double;
#define V4_ENTRY(x) x##_f64
#endif

int V4_ENTRY(plan_cluster)(const MbaBatchDesc* d) { return plan_t<TU>(d).R; }

int V4_ENTRY(may_overflow)(const MbaBatchDesc* d) {
  const Plan p = plan_t<TU>(d);
  return p.R == 0 ? 1 : (may_overflow_t<TU>(d, p) ? 1 : 0);
}

int V4_ENTRY(launch)(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o, cudaStream_t st,
                     int R, void* ws, size_t ws_bytes) {
  const Plan p = plan_t<TU>(d);
  if (p.R != R || R == 0) return MBA_ERR_TOO_LARGE;
  return launch_prec<TU>(d, cfg, o, st, p, ws, ws_bytes);
}

}  // namespace v4
}  // namespace mba
