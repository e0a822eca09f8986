// mba_solve.cu -- on-device Levenberg-Marquardt mini bundle adjustment (sm_100a).
//
// Replaces lm_solve (miniba.py:223-296) and, inside it, residuals (85-98),
// huber_cost/weights (46-54), _build_blocks (101-132), _assemble (135-177) and
// solve_step(method="schur") (180-220).
//
// Execution model: a persistent grid; each CTA pulls whole problems from an
// atomic work counter and runs the complete LM loop for that problem on chip.
//
//   setup (once per solve)
//     point CSR by binary search over the point-major observations, the
//     camera-major permutation (warp ballots), and the co-observation pair
//     lists: for every free camera block (a <= b) the list of observation
//     pairs (i in a, j in b, same point). Built once, they turn the Schur
//     accumulation into a divergence-free stream.
//   cost pass   one thread per observation, 16-byte record loads, fp64
//               residual and robust cost, deterministic block reduction
//   per iteration
//     K1+K2 point pass   one thread per point: fp64 residual, Jacobians in T,
//                        V_p / g_p accumulation in registers, W_i = w A^T B,
//                        damped 3x3 Cholesky V_p = L L^T and the Schur factors
//                        Y_i = W_i L^-T, z_p = L^-1 g_p, y_f = L^-1 Wf_p
//     K2 camera jobs     one warp per free camera: U_aa, U_af, g_a and the
//                        Schur focal column / rhs terms sum Y_i y_f, sum Y_i z
//     K3 pair jobs       one warp per camera block: S_ab = -sum Y_i Y_j^T over
//                        the block's pair list (fixed-order warp butterflies:
//                        no atomics, bit-reproducible)
//     K4 LDL^T           packed reduced camera system in shared memory, one
//                        barrier per column, then forward/back substitution
//        back-sub        dp_p = -L_p^-T (z_p + sum Y_i^T dc + y_f df)
//     K5 trials          <= 5 backtracking cost passes (fp64), accept/reject,
//                        lambda schedule and termination -- all on device
//
// State (cameras, focal, points) is float64; T selects the arithmetic of the
// linearise/Schur/factorisation stages (float = mixed-precision iterative
// refinement, SURVEY 8c design (b); double = full float64).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include <cooperative_groups.h>

#include "mba_common.cuh"
#include "mba_v4.cuh"

namespace mba {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPtStride = 17;    // per point: L(6) z(3) yf(3) dp(3) pad; odd -> no smem bank conflicts
constexpr int kYStride = 20;     // per observation: W_i then Y_i (6x3), padded for 16B vectors
constexpr int kUcamStride = 45;  // per free camera: U_aa lower(21) U_af(6) g_a(6) Sy_f(6) Sy_z(6)

// Optional per-phase cycle counters (build with -DMBA_PHASE_PROF; see
// paper_2506_05558_b200/build.py --prof). Thread 0 of every CTA accumulates
// clock64() deltas between phase boundaries; totals land in g_prof[phase].
enum { PH_SETUP, PH_COST0, PH_POINT, PH_JOBS, PH_ASM, PH_CHOL, PH_SOLVE, PH_TRIAL, PH_COMMIT, PH_JWAIT, PH_JRED, PH_ITEMS, PH_ITEMS2, PH_NCAM, PH_NPAIR, PH_BSUB, PH_JSYNC, PH_N };
#ifdef MBA_PHASE_PROF
__device__ unsigned long long* g_prof = nullptr;
#define PROF_DECL __shared__ long long s_prof[PH_N]; long long prof_t = clock64(); \
  if (threadIdx.x == 0) for (int i = 0; i < PH_N; ++i) s_prof[i] = 0;
#define PROF_MARK(ph) if (threadIdx.x == 0) { long long now = clock64(); s_prof[ph] += now - prof_t; prof_t = now; }
#define PROF_FLUSH if (threadIdx.x == 0 && g_prof) for (int i = 0; i < PH_N; ++i) atomicAdd(g_prof + i, (unsigned long long)s_prof[i]);
#else
#define PROF_DECL
#define PROF_MARK(ph)
#define PROF_FLUSH
#endif

struct SolveParams {
  MbaBatchDesc d;
  MbaLmConfig cfg;
  MbaOutputs o;
  int* counter;
  unsigned char* ws;       // per-slot workspace base
  size_t ws_slot_bytes;
  int max_cams;
  unsigned char* grid;     // cooperative (multi-CTA) mode: cross-CTA buffers
  int64_t grid_chunks;     // capacity of the job-chunk tables in `grid`
  int only_flagged;        // solve only problems the cluster kernel could not place
};

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Compile-time shared-memory layout for problems of up to MAXC cameras.
// The fixed part holds the camera state, the packed reduced camera system and
// the small index tables; in resident mode the per-problem scratch (camera
// permutation, point CSR, pair list, Y blocks, point factors) follows it, so
// the whole LM iteration runs out of shared memory.
// The reduced camera system is kept as an AUGMENTED column-major packed lower
// triangle: column j holds rows j..C-1 of S followed by rhs_j as "row C", so the
// LDL^T elimination performs the forward substitution on the fly. acol(j) is
// the start of column j; tab[] maps a packed position to its (row, column).
__host__ __device__ __forceinline__ int acol(int j, int C) { return j * (C + 1) - (j * (j - 1)) / 2; }
}  // namespace mba
#include "mba_ldl.cuh"
namespace mba {

template <typename T, int MAXC>
struct Layout {
  static constexpr int N = MAXC, C = 6 * MAXC + 1, NB = MAXC * (MAXC + 1) / 2;
  static constexpr int CA = C * (C + 3) / 2;                        // augmented packed size
  static constexpr size_t oRc = 0;                                  // double[N][9]
  static constexpr size_t oTc = oRc + 8 * 9 * N;                    // double[N][3]
  static constexpr size_t oRt = oTc + 8 * 3 * N;                    // trial sets [5][N][9]
  static constexpr size_t oTt = oRt + 8 * 9 * N * kBacktrackTries;  // [5][N][3]
  static constexpr size_t oDc = oTt + 8 * 3 * N * kBacktrackTries;  // double[C]
  static constexpr size_t oRed = align16(oDc + 8 * C);              // double[kWarps*4]
  static constexpr size_t oS = oRed + 8 * kWarps * 4;               // T[CA]
  static constexpr size_t oRhs = align16(oS + sizeof(T) * CA);      // T[C] LDL^T pivot reciprocals
  static constexpr size_t oL10 = align16(oRhs + sizeof(T) * C);     // T[C] LDL^T pair multipliers
  static constexpr size_t oTab = align16(oL10 + sizeof(T) * C);     // T[kLdlPanel][ldl_lstr(C)] LDL^T panel L
  static constexpr size_t oUcam = align16(oTab + sizeof(T) * kLdlPanel * ldl_lstr(C));  // T[N][kUcamStride]
  static constexpr size_t oCamPtr = align16(oUcam + sizeof(T) * N * kUcamStride);
  static constexpr size_t oSlot = oCamPtr + 4 * (N + 1);
  static constexpr size_t oCos = oSlot + 4 * N;
  static constexpr size_t oBlkOff = oCos + 4 * N;                   // int[NB+1]
  static constexpr size_t oBlkA = oBlkOff + 4 * (NB + 1);           // uchar[NB]
  static constexpr size_t oBlkB = oBlkA + NB;
  static constexpr size_t kFixed = align16(oBlkB + NB);
};

// ---- vector helpers for the 18-value Y blocks ------------------------------
// Y rows are stored with stride kYStride (20, 16-byte vectors) in global
// scratch and kYStrideRes (18, 8-byte vectors) in shared-memory scratch.
constexpr int kYStrideRes = 18;

template <bool RES> struct YS { static constexpr int v = RES ? kYStrideRes : kYStride; };

__device__ __forceinline__ void load18v2(const float* p, float y[18]) {
  const float2* q = reinterpret_cast<const float2*>(p);
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    float2 v = q[i];
    y[2 * i] = v.x;
    y[2 * i + 1] = v.y;
  }
}
__device__ __forceinline__ void store18v2(float* p, const float y[18]) {
  float2* q = reinterpret_cast<float2*>(p);
#pragma unroll
  for (int i = 0; i < 9; ++i) q[i] = make_float2(y[2 * i], y[2 * i + 1]);
}

__device__ __forceinline__ void load18(const float* p, float y[18]) {
  const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float4 v = q[i];
    y[4 * i] = v.x; y[4 * i + 1] = v.y; y[4 * i + 2] = v.z; y[4 * i + 3] = v.w;
  }
  float2 v = reinterpret_cast<const float2*>(p)[8];
  y[16] = v.x;
  y[17] = v.y;
}
__device__ __forceinline__ void store18(float* p, const float y[18]) {
  float4* q = reinterpret_cast<float4*>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) q[i] = make_float4(y[4 * i], y[4 * i + 1], y[4 * i + 2], y[4 * i + 3]);
  reinterpret_cast<float2*>(p)[8] = make_float2(y[16], y[17]);
}
__device__ __forceinline__ void load18(const double* p, double y[18]) {
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    double2 v = q[i];
    y[2 * i] = v.x;
    y[2 * i + 1] = v.y;
  }
}
__device__ __forceinline__ void store18(double* p, const double y[18]) {
  double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
  for (int i = 0; i < 9; ++i) q[i] = make_double2(y[2 * i], y[2 * i + 1]);
}

struct Obs {
  double u, v;
  int cam, pt;
};

__device__ __forceinline__ Obs load_obs(const MbaObs* __restrict__ obs, const float* __restrict__ lo,
                                        int64_t k) {
  float4 r = __ldg(reinterpret_cast<const float4*>(obs) + k);
  Obs o;
  o.u = (double)r.x;
  o.v = (double)r.y;
  o.cam = __float_as_int(r.z);
  o.pt = __float_as_int(r.w);
  if (lo != nullptr) {
    float2 l = __ldg(reinterpret_cast<const float2*>(lo) + k);
    o.u += (double)l.x;
    o.v += (double)l.y;
  }
  return o;
}

__device__ __forceinline__ int obs_cam(const MbaObs* __restrict__ obs, int64_t k) {
  return __ldg(&obs[k].cam);
}

__device__ __forceinline__ int warp_excl_scan(int v, int lane) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x - v;
}

// Cost pass over all observations with camera set (Rs, ts, f) and points
// X + frac * dp (MBA_GRID_COST_U observations per thread per step).
// Returns (sum rho, sum e, sum e^2) to every thread.
template <typename T>
__device__ void cost_pass(const MbaObs* __restrict__ obs, const float* __restrict__ lo, int K,
                          const double* __restrict__ X, const T* __restrict__ ptw, double frac,
                          bool use_dp, const double* Rs, const double* ts, double f, double cx,
                          double cy, double delta, int loss, double* red, double out[3],
                          int start, int stride) {
#ifndef MBA_GRID_COST_U
#define MBA_GRID_COST_U 1   // config 5: 15.5 ms at 4, 15.4 at 2, 15.1 at 1 (scripts/gpu/grid_cost_u.sh)
#endif
  constexpr int U = MBA_GRID_COST_U;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int k0 = start; k0 < K; k0 += U * stride) {
    Obs o[U];
    double Xp[U][3];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * stride;
      if (k < K) o[u] = load_obs(obs, lo, k);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * stride;
      if (k >= K) continue;
      const double* x = X + 3 * o[u].pt;
      Xp[u][0] = x[0];
      Xp[u][1] = x[1];
      Xp[u][2] = x[2];
      if (use_dp) {
        const T* dp = ptw + (size_t)o[u].pt * kPtStride + 12;
        Xp[u][0] = Xp[u][0] + frac * (double)dp[0];
        Xp[u][1] = Xp[u][1] + frac * (double)dp[1];
        Xp[u][2] = Xp[u][2] + frac * (double)dp[2];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * stride;
      if (k >= K) continue;
      Proj pr = project_residual_fast(Rs + 9 * o[u].cam, ts + 3 * o[u].cam, Xp[u], f, cx, cy, o[u].u, o[u].v);
      double e = sqrt(pr.ru * pr.ru + pr.rv * pr.rv);
      acc[0] += robust_rho(e, delta, loss);
      acc[1] += e;
      acc[2] += e * e;
    }
  }
  block_sum<double, 3>(acc, red);
  out[0] = acc[0];
  out[1] = acc[1];
  out[2] = acc[2];
}

// Per-problem scratch: in shared memory (RES) or in this CTA's global slot.
template <typename T, bool RES>
struct Scratch {
  using Idx = typename std::conditional<RES, unsigned short, int>::type;  // K < 65536 when resident
  Idx* perm;        // camera-major permutation of the observations
  Idx* ptr;         // point CSR
  void* pairs;      // RES: uint32 (i << 16 | j); else int2
  T* Ybuf;          // [K][kYStride]
  T* ptw;           // [P][kPtStride]
  __device__ __forceinline__ int2 pair(int q) const {
    if (RES) {
      const unsigned v = static_cast<const unsigned*>(pairs)[q];
      return make_int2((int)(v >> 16), (int)(v & 0xffffu));
    }
    return static_cast<const int2*>(pairs)[q];
  }
  __device__ __forceinline__ void set_pair(int q, int i, int j) const {
    if (RES) static_cast<unsigned*>(pairs)[q] = ((unsigned)i << 16) | (unsigned)j;
    else static_cast<int2*>(pairs)[q] = make_int2(i, j);
  }
};

template <typename T, bool RES>
__host__ __device__ inline size_t scratch_bytes(int64_t max_obs, int64_t max_points, int64_t max_pairs) {
  return align16((RES ? 2 : 4) * max_obs) + align16((RES ? 2 : 4) * (max_points + 1)) +
         align16((RES ? 4 : 8) * max_pairs) + align16(sizeof(T) * YS<RES>::v * max_obs) +
         align16(sizeof(T) * kPtStride * max_points);
}

template <typename T, bool RES>
__device__ __forceinline__ Scratch<T, RES> scratch_at(unsigned char* base, const MbaBatchDesc& D) {
  using Idx = typename Scratch<T, RES>::Idx;
  Scratch<T, RES> w;
  w.perm = (Idx*)base;
  w.ptr = (Idx*)(base + align16(sizeof(Idx) * D.max_obs));
  unsigned char* q = (unsigned char*)w.ptr + align16(sizeof(Idx) * (D.max_points + 1));
  w.pairs = q;
  q += align16((RES ? 4 : 8) * D.max_pairs);
  w.Ybuf = (T*)q;
  w.ptw = (T*)(q + align16(sizeof(T) * YS<RES>::v * D.max_obs));
  return w;
}

// Cross-CTA buffers of the cooperative mode (one problem spread over the grid).
// Cooperative mode: work chunks of the camera / pair jobs (spread over every
// warp of the grid; a camera job is split into runs of kChunkObs observations,
// a pair block into runs of kChunkPairs co-observation pairs) and their partial
// sums, reduced per job in chunk order (deterministic).
constexpr int kChunkObs = 256;
constexpr int kChunkPairs = 512;

__host__ __device__ inline int64_t grid_max_chunks(int64_t max_obs, int64_t max_pairs, int maxc) {
  return (max_obs + kChunkObs - 1) / kChunkObs + maxc + (max_pairs + kChunkPairs - 1) / kChunkPairs +
         (int64_t)maxc * (maxc + 1) / 2;
}

// Cross-CTA buffers of the cooperative mode (one problem spread over the grid).
template <typename T, int MAXC>
struct GridBufs {
  static constexpr int C = 6 * MAXC + 1, CA = C * (C + 3) / 2, NB = MAXC * (MAXC + 1) / 2;
  static constexpr size_t oS = 0;                                     // T[CA]
  static constexpr size_t oU = align16(oS + sizeof(T) * CA);          // T[MAXC][kUcamStride]
  static constexpr size_t oCnt = align16(oU + sizeof(T) * MAXC * kUcamStride);  // int[MAXC + NB + 2]
  static constexpr size_t oCoff = align16(oCnt + 4 * (MAXC + NB + 2));  // int[MAXC + NB + 1] chunks per job
  static constexpr size_t oJobQ = align16(oCoff + 4 * (MAXC + NB + 1));  // int[2] job-chunk queues (by LM iteration parity)
  static constexpr size_t oRed = align16(oJobQ + 8);                   // double[2][G][4]
  static __host__ __device__ size_t oChunk(int G) { return align16(oRed + 8 * 2 * 4 * (size_t)G); }  // int2[chunks]
  static __host__ __device__ size_t oPart(int G, int64_t chunks) {   // T[chunks][kUcamStride]
    return align16(oChunk(G) + 8 * (size_t)chunks);
  }
  static __host__ __device__ size_t oSeg(int G, int64_t chunks) {   // int[G * warps][MAXC]
    return align16(oPart(G, chunks) + sizeof(T) * kUcamStride * (size_t)chunks);
  }
  static __host__ __device__ size_t bytes(int G, int64_t chunks) {
    return oSeg(G, chunks) + 4 * (size_t)G * (kThreads / 32) * MAXC;
  }
};

// global (L2) -> shared bulk copy on the TMA engine (cp.async.bulk, 1-D): one
// thread arms the CTA's mbarrier with the byte count and issues the copies,
// every thread waits on the barrier's phase. No registers staged (a strided
// load/store loop waited one L2 round trip per element -- ~50k cycles for the
// 142 KB reduced system of a 32-camera problem -- and unrolling it cost the
// grid kernel registers). Sizes are rounded up to 16 bytes: both regions are
// followed by 16-byte alignment slack. `phase` is the caller's parity bit.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__host__ __device__ constexpr unsigned bulk_bytes(size_t b) { return (unsigned)((b + 15u) & ~size_t(15)); }
// arm the barrier for `bytes` (the sum of the bulk_bytes of the copies that follow)
__device__ __forceinline__ void mbar_arm(unsigned long long* mbar, unsigned bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* mbar) {
  const unsigned mb = smem_u32(mbar);
  constexpr unsigned kChunk = 32768;
  for (unsigned off = 0; off < bytes; off += kChunk) {
    const unsigned sz = bytes - off < kChunk ? bytes - off : kChunk;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32((char*)dst + off)),
                 "l"((const char*)src + off), "r"(sz), "r"(mb)
                 : "memory");
  }
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(mbar)),
      "r"(phase)
      : "memory");
}

template <typename T, int MAXC, bool RES, bool GRID = false, int NT = kThreads>
__device__ void solve_one(const SolveParams& P, int b, unsigned char* smem_raw) {
  constexpr int kWarps = NT / 32;
  using L = Layout<T, MAXC>;
  using GB = GridBufs<T, MAXC>;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // work distribution: one CTA (batched mode) or the whole grid (cooperative mode)
  const int rank = GRID ? (int)blockIdx.x : 0, nranks = GRID ? (int)gridDim.x : 1;
  const int gtid = rank * blockDim.x + tid, gthreads = nranks * blockDim.x;
  const int gwid = rank * kWarps + wid, gwarps = nranks * kWarps;
  const bool lead = tid == 0 && rank == 0;    // writes traces and outputs
  auto gsync = [&]() {
    if constexpr (GRID) cooperative_groups::this_grid().sync();
    else __syncthreads();
  };
  int red_epoch = 0;
  __shared__ double s_gsum[4];
  // deterministic cross-CTA sum of N per-CTA values (after a block_sum)
  auto grid_sum = [&](double* v, int N) {
    if constexpr (GRID) {
      double* buf = (double*)(P.grid + GB::oRed) + (size_t)(red_epoch & 1) * nranks * 4;
      ++red_epoch;
      if (tid == 0)
        for (int i = 0; i < N; ++i) buf[rank * 4 + i] = v[i];
      gsync();
      // warp i sums value i over the ranks: lanes load in parallel (one L2
      // round trip instead of one per rank -- the sequential loop cost ~100k
      // cycles per 4-value sum on 148 CTAs), fixed-order lane sums and a
      // fixed xor tree, so every CTA derives bit-identical totals
      if (wid < N) {
        double s_ = 0.0;
        for (int r = lane; r < nranks; r += 32) s_ += __ldcg(buf + r * 4 + wid);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s_ += __shfl_xor_sync(0xffffffffu, s_, o);
        if (lane == 0) s_gsum[wid] = s_;
      }
      __syncthreads();
      for (int i = 0; i < N; ++i) v[i] = s_gsum[i];
      __syncthreads();
    }
  };
  const MbaBatchDesc& D = P.d;
  const MbaLmConfig& cfg = P.cfg;
  const MbaOutputs& O = P.o;
  struct {
    double *Rc, *tc, *Rt, *tt, *dc, *red;
    T *S, *rhs, *ucam;
    int *cam_ptr, *slot, *cam_of_slot, *blk_off;
    unsigned char *blk_a, *blk_b;
  } sm;
  sm.Rc = (double*)(smem_raw + L::oRc);
  sm.tc = (double*)(smem_raw + L::oTc);
  sm.Rt = (double*)(smem_raw + L::oRt);
  sm.tt = (double*)(smem_raw + L::oTt);
  sm.dc = (double*)(smem_raw + L::oDc);
  sm.red = (double*)(smem_raw + L::oRed);
  sm.S = (T*)(smem_raw + L::oS);
  sm.rhs = (T*)(smem_raw + L::oRhs);
  sm.ucam = (T*)(smem_raw + L::oUcam);
  sm.cam_ptr = (int*)(smem_raw + L::oCamPtr);
  sm.slot = (int*)(smem_raw + L::oSlot);
  sm.cam_of_slot = (int*)(smem_raw + L::oCos);
  sm.blk_off = (int*)(smem_raw + L::oBlkOff);
  sm.blk_a = smem_raw + L::oBlkA;
  sm.blk_b = smem_raw + L::oBlkB;
  __shared__ int s_flag;        // setup error
  __shared__ __align__(8) unsigned long long s_mbar;   // GRID: bulk copies of the job totals
  unsigned mbar_phase = 0u;
  if (GRID && tid == 0) mbar_init(&s_mbar);
  __shared__ int s_C, s_nf;
  double* s_red4 = sm.red;

  const int64_t cb = D.cam_off[b], pb = D.pt_off[b], ob = D.obs_off[b];
  const int n = (int)(D.cam_off[b + 1] - cb);
  const int Pn = (int)(D.pt_off[b + 1] - pb);
  const int K = (int)(D.obs_off[b + 1] - ob);
  const uint8_t fl = D.flags[b];
  const bool has_f = fl & 1, opt_pts = (fl >> 1) & 1;
  const double cx = D.cx[b], cy = D.cy[b];
  const double delta = cfg.delta, nu = cfg.nu;
  const int loss = cfg.loss, max_it = cfg.max_iters;
  const MbaObs* __restrict__ obs = D.obs + ob;
  const float* __restrict__ lo = D.obs_lo ? D.obs_lo + 2 * ob : nullptr;
  double* __restrict__ X = O.points_out + 3 * pb;

  const Scratch<T, RES> W = scratch_at<T, RES>(
      RES ? smem_raw + L::kFixed : P.ws + (GRID ? 0 : (size_t)blockIdx.x * P.ws_slot_bytes), D);
  int* gcnt = GRID ? (int*)(P.grid + GB::oCnt) : nullptr;
  int* jobq = GRID ? (int*)(P.grid + GB::oJobQ) : nullptr;
  if (GRID && rank == 0 && tid == 0) jobq[0] = jobq[1] = 0;   // published by the setup's grid syncs
  constexpr int YSTR = YS<RES>::v;
  auto ld18 = [](const T* p, T y[18]) {
    if constexpr (RES && sizeof(T) == 4) load18v2((const float*)p, (float*)y); else load18(p, y);
  };
  auto st18 = [](T* p, const T y[18]) {
    if constexpr (RES && sizeof(T) == 4) store18v2((float*)p, (const float*)y); else store18(p, y);
  };
  typename Scratch<T, RES>::Idx* __restrict__ perm = W.perm;
  typename Scratch<T, RES>::Idx* __restrict__ ptr = W.ptr;
  T* __restrict__ Ybuf = W.Ybuf;
  T* __restrict__ ptw = W.ptw;

  double* costs = O.costs + (size_t)b * (max_it + 1);
  double* lambdas = O.lambdas + (size_t)b * max_it;
  uint8_t* accepted = O.accepted + (size_t)b * max_it;
  uint8_t* evals = O.evals + (size_t)b * max_it;

  PROF_DECL
  // ---------------- setup ----------------
  for (int i = tid; i < n * 9; i += blockDim.x) sm.Rc[i] = O.R_in[cb * 9 + i];
  for (int i = tid; i < n * 3; i += blockDim.x) sm.tc[i] = O.t_in[cb * 3 + i];
  if (O.points_in != O.points_out)
    for (int i = gtid; i < Pn * 3; i += gthreads) X[i] = O.points_in[pb * 3 + i];
  if (tid == 0) {
    int nf = 0;
    for (int c = 0; c < n; ++c) {
      if (D.fixed[cb + c]) {
        sm.slot[c] = -1;
      } else {
        sm.slot[c] = nf;
        sm.cam_of_slot[nf] = c;
        ++nf;
      }
    }
    int q = 0;
    for (int a = 0; a < nf; ++a)
      for (int bb = a; bb < nf; ++bb, ++q) {
        sm.blk_a[q] = (unsigned char)a;
        sm.blk_b[q] = (unsigned char)bb;
      }
    s_nf = nf;
    s_C = 6 * nf + (has_f ? 1 : 0);
    s_flag = 0;
  }
  // point CSR: observations are point-major; ptr[p] = first k with pt >= p
  for (int p = gtid; p <= Pn; p += gthreads) {
    int lo_i = 0, hi_i = K;
    while (lo_i < hi_i) {
      int mid = (lo_i + hi_i) >> 1;
      if (__ldg(&obs[mid].pt) < p) lo_i = mid + 1; else hi_i = mid;
    }
    ptr[p] = lo_i;
  }
  for (int k = gtid; k < K; k += gthreads) {
    int pt = __ldg(&obs[k].pt), c = __ldg(&obs[k].cam);
    bool bad = pt < 0 || pt >= Pn || c < 0 || c >= n || (k > 0 && __ldg(&obs[k - 1].pt) > pt);
    if (bad) s_flag = 1;
  }
  __syncthreads();
  if constexpr (GRID) {
    double fv = s_flag;
    __syncthreads();
    grid_sum(&fv, 1);
    if (tid == 0) s_flag = fv != 0.0;
  }
  // camera-major permutation
  if constexpr (GRID) {
    // cooperative mode: every warp owns a contiguous segment of the
    // observations; per-segment camera counts, a per-camera scan over the
    // segments, then each warp scatters its segment in order (one warp per
    // camera scanning all K observations took ~2 ms at K = 200k)
    int* seg = (int*)(P.grid + GB::oSeg(nranks, P.grid_chunks));
    const int seg_len = (K + gwarps - 1) / gwarps;
    const int s0 = gwid * seg_len, s1 = min(K, s0 + seg_len);
    const unsigned lt = (1u << lane) - 1u;
    int my_cnt = 0;   // lane c: observations of camera c in this segment
    for (int k0 = s0; k0 < s1; k0 += 32) {
      const int k = k0 + lane;
      const int cl = k < s1 ? obs_cam(obs, k) : -1;
      for (int c = 0; c < n; ++c) {
        const unsigned m = __ballot_sync(0xffffffffu, cl == c);
        if (lane == c) my_cnt += __popc(m);
      }
    }
    if (lane < n) seg[gwid * n + lane] = my_cnt;
    gsync();
    for (int c = gwid; c < n; c += gwarps) {   // exclusive scan over segments, per camera
      int carry = 0;
      for (int s_ = 0; s_ < gwarps; s_ += 32) {
        const int v = s_ + lane < gwarps ? seg[(s_ + lane) * n + c] : 0;
        const int inc = warp_excl_scan(v, lane) + v;
        if (s_ + lane < gwarps) seg[(s_ + lane) * n + c] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) gcnt[c + 1] = carry;
    }
    gsync();
    if (tid == 0) {
      sm.cam_ptr[0] = 0;
      for (int c = 0; c < n; ++c) sm.cam_ptr[c + 1] = sm.cam_ptr[c] + gcnt[c + 1];
    }
    __syncthreads();
    int my_base = lane < n ? sm.cam_ptr[lane] + seg[gwid * n + lane] : 0;
    for (int k0 = s0; k0 < s1; k0 += 32) {
      const int k = k0 + lane;
      const int cl = k < s1 ? obs_cam(obs, k) : -1;
      for (int c = 0; c < n; ++c) {
        const unsigned m = __ballot_sync(0xffffffffu, cl == c);
        const int bc = __shfl_sync(0xffffffffu, my_base, c);
        if (cl == c) perm[bc + __popc(m & lt)] = k;
        if (lane == c) my_base += __popc(m);
      }
    }
    gsync();
  } else {
  for (int c = gwid; c < n; c += gwarps) {
    int cnt = 0;
    for (int k0 = 0; k0 < K; k0 += 32) {
      int k = k0 + lane;
      bool hit = k < K && obs_cam(obs, k) == c;
      cnt += __popc(__ballot_sync(0xffffffffu, hit));
    }
    if (lane == 0) {
      if constexpr (GRID) gcnt[c + 1] = cnt; else sm.cam_ptr[c + 1] = cnt;
    }
  }
  gsync();
  if (tid == 0) {
    sm.cam_ptr[0] = 0;
    for (int c = 0; c < n; ++c) sm.cam_ptr[c + 1] = sm.cam_ptr[c] + (GRID ? gcnt[c + 1] : sm.cam_ptr[c + 1]);
  }
  __syncthreads();
  for (int c = gwid; c < n; c += gwarps) {
    int base = sm.cam_ptr[c];
    for (int k0 = 0; k0 < K; k0 += 32) {
      int k = k0 + lane;
      bool hit = k < K && obs_cam(obs, k) == c;
      unsigned m = __ballot_sync(0xffffffffu, hit);
      if (hit) perm[base + __popc(m & ((1u << lane) - 1u))] = k;
      base += __popc(m);
    }
  }
  gsync();
  }
  const int nf = s_nf, C = s_C, FI = C - 1;
  const int nb = opt_pts ? nf * (nf + 1) / 2 : 0;
  // co-observation pair lists per camera block (a <= b): count, scan, fill
  int* blk_cnt = GRID ? gcnt + MAXC + 1 : sm.blk_off;
  for (int pass = 0; pass < 2; ++pass) {
    for (int blk = gwid; blk < nb; blk += gwarps) {
      const int ca = sm.cam_of_slot[sm.blk_a[blk]], cbb = sm.cam_of_slot[sm.blk_b[blk]];
      const int q1 = sm.cam_ptr[ca + 1];
      int base = pass ? sm.blk_off[blk] : 0;
      for (int q0 = sm.cam_ptr[ca]; q0 < q1; q0 += 32) {
        const int q = q0 + lane;
        int i = -1, j0 = 0, j1 = 0, m = 0;
        if (q < q1) {
          i = perm[q];
          const int pt = __ldg(&obs[i].pt);
          j0 = ptr[pt];
          j1 = ptr[pt + 1];
          for (int j = j0; j < j1; ++j) m += obs_cam(obs, j) == cbb;
        }
        if (pass) {
          int pos = base + warp_excl_scan(m, lane);
          for (int j = j0; j < j1 && m; ++j)
            if (obs_cam(obs, j) == cbb) W.set_pair(pos++, i, j);
        }
        base += warp_sum(m);
      }
      if (!pass && lane == 0) blk_cnt[blk + 1] = base;
    }
    gsync();
    if (!pass && tid == 0) {
      sm.blk_off[0] = 0;
      for (int q = 0; q < nb; ++q) sm.blk_off[q + 1] = sm.blk_off[q] + blk_cnt[q + 1];
    }
    __syncthreads();
  }
  const int CA = C * (C + 3) / 2;
  // cooperative mode: the job chunk table (job, first item) and chunks per job
  int* coff = GRID ? (int*)(P.grid + GB::oCoff) : nullptr;
  int2* chunk = GRID ? (int2*)(P.grid + GB::oChunk(nranks)) : nullptr;
  T* cpart = GRID ? (T*)(P.grid + GB::oPart(nranks, P.grid_chunks)) : nullptr;
  if constexpr (GRID) {
    if (rank == 0 && tid == 0) {
      int q = 0;
      coff[0] = 0;
      for (int job = 0; job < nf + nb; ++job) {
        const int len = job < nf ? sm.cam_ptr[sm.cam_of_slot[job] + 1] - sm.cam_ptr[sm.cam_of_slot[job]]
                                 : sm.blk_off[job - nf + 1] - sm.blk_off[job - nf];
        const int ch = job < nf ? kChunkObs : kChunkPairs;
        for (int lo_i = 0; lo_i < len && q < P.grid_chunks; lo_i += ch) chunk[q++] = make_int2(job, lo_i);
        coff[job + 1] = q;
      }
    }
    gsync();
  }
  double f = O.focal_in[b];
  if (s_flag) {  // malformed problem: report and leave parameters untouched
    if (lead) {
      O.n_iters[b] = 0;
      O.status[b] = -1;
      if (O.focal_out) O.focal_out[b] = f;
    }
    if (rank == 0) {
      for (int i = tid; i < n * 9; i += blockDim.x) O.R_out[cb * 9 + i] = sm.Rc[i];
      for (int i = tid; i < n * 3; i += blockDim.x) O.t_out[cb * 3 + i] = sm.tc[i];
    }
    __syncthreads();
    return;
  }

  PROF_MARK(PH_SETUP)
  // initial cost (miniba.py:232-235)
  double st[3];
  cost_pass<T>(obs, lo, K, X, ptw, 0.0, false, sm.Rc, sm.tc, f, cx, cy, delta, loss, sm.red, st,
               gtid, gthreads);
  grid_sum(st, 3);
  PROF_MARK(PH_COST0)
  double cost = st[0], se = st[1], se2 = st[2];
  double lam = cfg.lambda_init;
  if (lead) costs[0] = cost;
  int it = 0, stop_reason = MBA_SOLVE_MAX_ITERS;

  for (; it < max_it;) {
    const T tlam = T(lam);
    // ---------- K1+K2 point pass ----------
    T part[4] = {T(0), T(0), T(0), T(0)};  // U_ff, g_f, sum yf.yf, sum yf.z
    for (int p = gtid; p < Pn; p += gthreads) {
      const double Xp[3] = {X[3 * p], X[3 * p + 1], X[3 * p + 2]};
      const int k0 = ptr[p], k1 = ptr[p + 1];
      T V[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};  // 00 10 11 20 21 22
      T g[3] = {T(0), T(0), T(0)}, wf[3] = {T(0), T(0), T(0)};
      for (int k = k0; k < k1; ++k) {
        Obs o = load_obs(obs, lo, k);
        const double* Rk = sm.Rc + 9 * o.cam;
        Proj pr = project_residual_fast(Rk, sm.tc + 3 * o.cam, Xp, f, cx, cy, o.u, o.v);
        double e = sqrt(pr.ru * pr.ru + pr.rv * pr.rv);
        T w = T(robust_w(e, delta, loss));
        T A[12], Fb[2], Bm[6];
        jac_blocks<T>(pr, Rk, f, A, Fb, Bm);
        T r0 = T(pr.ru), r1 = T(pr.rv);
        T wB[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) wB[i] = w * Bm[i];
        if (has_f) {
          part[0] += w * (Fb[0] * Fb[0] + Fb[1] * Fb[1]);
          part[1] += w * (Fb[0] * r0 + Fb[1] * r1);
        }
        if (opt_pts) {
          V[0] += Bm[0] * wB[0] + Bm[3] * wB[3];
          V[1] += Bm[1] * wB[0] + Bm[4] * wB[3];
          V[2] += Bm[1] * wB[1] + Bm[4] * wB[4];
          V[3] += Bm[2] * wB[0] + Bm[5] * wB[3];
          V[4] += Bm[2] * wB[1] + Bm[5] * wB[4];
          V[5] += Bm[2] * wB[2] + Bm[5] * wB[5];
#pragma unroll
          for (int a = 0; a < 3; ++a) g[a] += wB[a] * r0 + wB[3 + a] * r1;
          if (has_f) {
            T wf0 = w * Fb[0], wf1 = w * Fb[1];
#pragma unroll
            for (int a = 0; a < 3; ++a) wf[a] += wf0 * Bm[a] + wf1 * Bm[3 + a];
          }
          if (sm.slot[o.cam] >= 0) {
            T W[18];
#pragma unroll
            for (int r = 0; r < 6; ++r)
#pragma unroll
              for (int a = 0; a < 3; ++a) W[r * 3 + a] = A[r] * wB[a] + A[6 + r] * wB[3 + a];
            st18(Ybuf + (size_t)k * YSTR, W);
          }
        }
      }
      if (!opt_pts) continue;
      // damping (miniba.py:191-193) and 3x3 Cholesky of Vd
      V[0] += tlam * (V[0] > T(kDiagFloor) ? V[0] : T(kDiagFloor));
      V[2] += tlam * (V[2] > T(kDiagFloor) ? V[2] : T(kDiagFloor));
      V[5] += tlam * (V[5] > T(kDiagFloor) ? V[5] : T(kDiagFloor));
      T L00 = sqrt(V[0]);
      T i00 = T(1) / L00;
      T L10 = V[1] * i00, L20 = V[3] * i00;
      T L11 = sqrt(V[2] - L10 * L10);
      T i11 = T(1) / L11;
      T L21 = (V[4] - L20 * L10) * i11;
      T L22 = sqrt(V[5] - L20 * L20 - L21 * L21);
      T i22 = T(1) / L22;
      for (int k = k0; k < k1; ++k) {
        if (sm.slot[obs_cam(obs, k)] < 0) continue;
        T* Wk = Ybuf + (size_t)k * YSTR;
        T y[18];
        ld18(Wk, y);
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          T y0 = y[r * 3 + 0] * i00;
          T y1 = (y[r * 3 + 1] - L10 * y0) * i11;
          T y2 = (y[r * 3 + 2] - L20 * y0 - L21 * y1) * i22;
          y[r * 3 + 0] = y0;
          y[r * 3 + 1] = y1;
          y[r * 3 + 2] = y2;
        }
        st18(Wk, y);
      }
      T z0 = g[0] * i00, z1 = (g[1] - L10 * z0) * i11, z2 = (g[2] - L20 * z0 - L21 * z1) * i22;
      T f0 = wf[0] * i00, f1 = (wf[1] - L10 * f0) * i11, f2 = (wf[2] - L20 * f0 - L21 * f1) * i22;
      part[2] += f0 * f0 + f1 * f1 + f2 * f2;
      part[3] += f0 * z0 + f1 * z1 + f2 * z2;
      T* pw = ptw + (size_t)p * kPtStride;
      pw[0] = L00; pw[1] = L10; pw[2] = L11; pw[3] = L20; pw[4] = L21; pw[5] = L22;
      pw[6] = z0; pw[7] = z1; pw[8] = z2;
      pw[9] = f0; pw[10] = f1; pw[11] = f2;
    }
    {
      T pf[4] = {part[0], part[1], part[2], part[3]};
      block_sum<T, 4>(pf, (T*)s_red4);
      if constexpr (GRID) {
        double pd[4] = {(double)pf[0], (double)pf[1], (double)pf[2], (double)pf[3]};
        grid_sum(pd, 4);   // also the barrier that publishes Y / point factors
        for (int i = 0; i < 4; ++i) pf[i] = T(pd[i]);
      }
      part[0] = pf[0]; part[1] = pf[1]; part[2] = pf[2]; part[3] = pf[3];
    }
    // (block_sum ended with __syncthreads: point factors are visible)
    PROF_MARK(PH_POINT)

    // ---------- K2 camera jobs + K3 pair jobs ----------
    // batched mode: one warp per job; cooperative mode: one warp per job CHUNK
    // (every warp of the grid busy), partial sums reduced per job afterwards
    T* S_jobs = GRID ? (T*)(P.grid + GB::oS) : sm.S;
    T* U_jobs = GRID ? (T*)(P.grid + GB::oU) : sm.ucam;
    const int n_items = GRID ? coff[nf + nb] : nf + nb;
    // cooperative mode: warps pull chunks from a grid-wide queue (one atomic per
    // chunk; results do not depend on which warp takes which chunk) -- the
    // static round robin left warps with 1 or 2 chunks of unequal cost waiting
    // at the grid barrier
    if (GRID && rank == 0 && tid == 0) jobq[(it + 1) & 1] = 0;   // last used two iterations ago
    for (int item = gwid;; item += gwarps) {
      if constexpr (GRID) {
        int q = 0;
        if (lane == 0) q = atomicAdd(jobq + (it & 1), 1);
        item = __shfl_sync(0xffffffffu, q, 0);
      }
      if (item >= n_items) break;
      // reconverge the warp before the lane-strided loops: without it the lanes
      // that left the previous item's loop at different trip counts stay
      // split and the loop runs with ~2 of 32 lanes active (measured)
      __syncwarp();
      int job = item, q_lo = 0, q_hi = 0;
      if constexpr (GRID) {
        const int2 cj = chunk[item];
        job = cj.x;
        q_lo = cj.y;
      }
#ifdef MBA_PHASE_PROF
      long long t_item;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_item));
#endif
      if (job < nf) {
        const int s = job, c = sm.cam_of_slot[s];
        const double* Rk = sm.Rc + 9 * c;
        T acc[kUcamStride];
#pragma unroll
        for (int i = 0; i < kUcamStride; ++i) acc[i] = T(0);
        int qa = sm.cam_ptr[c], qb = sm.cam_ptr[c + 1];
        if constexpr (GRID) {
          qa += q_lo;
          q_hi = qa + kChunkObs;
          qb = q_hi < qb ? q_hi : qb;
        }
        for (int q0 = qa; q0 < qb; q0 += 32) {
          __syncwarp();
          const int q = q0 + lane;
          if (q >= qb) continue;
          const int k = perm[q];
          Obs o = load_obs(obs, lo, k);
          const double Xp[3] = {X[3 * o.pt], X[3 * o.pt + 1], X[3 * o.pt + 2]};
          Proj pr = project_residual_fast(Rk, sm.tc + 3 * c, Xp, f, cx, cy, o.u, o.v);
          double e = sqrt(pr.ru * pr.ru + pr.rv * pr.rv);
          T w = T(robust_w(e, delta, loss));
          T A[12], Fb[2], Bm[6];
          jac_blocks<T>(pr, Rk, f, A, Fb, Bm);
          T r0 = T(pr.ru), r1 = T(pr.rv);
          int idx = 0;
#pragma unroll
          for (int r = 0; r < 6; ++r) {
            T wa0 = w * A[r], wa1 = w * A[6 + r];
#pragma unroll
            for (int cc = 0; cc <= r; ++cc) acc[idx++] += wa0 * A[cc] + wa1 * A[6 + cc];
            acc[21 + r] += wa0 * Fb[0] + wa1 * Fb[1];
            acc[27 + r] += wa0 * r0 + wa1 * r1;
          }
          if (opt_pts) {
            T y[18];
            ld18(Ybuf + (size_t)k * YSTR, y);
            const T* pw = ptw + (size_t)o.pt * kPtStride;
            const T z0 = pw[6], z1 = pw[7], z2 = pw[8], f0 = pw[9], f1 = pw[10], f2 = pw[11];
#pragma unroll
            for (int r = 0; r < 6; ++r) {
              acc[33 + r] += y[r * 3] * f0 + y[r * 3 + 1] * f1 + y[r * 3 + 2] * f2;
              acc[39 + r] += y[r * 3] * z0 + y[r * 3 + 1] * z1 + y[r * 3 + 2] * z2;
            }
          }
        }
        // transposed warp reduction (halving butterflies, ~N shuffles instead
        // of 5N); one lane writes each total
        T* dst = GRID ? cpart + (size_t)item * kUcamStride : U_jobs + s * kUcamStride;
        warp_reduce_to<T, kUcamStride>(acc, dst, lane);
      } else {
        const int blk = job - nf;
        const int sa = sm.blk_a[blk], sb = sm.blk_b[blk];
        T acc[36];
#pragma unroll
        for (int i = 0; i < 36; ++i) acc[i] = T(0);
        int qa = sm.blk_off[blk], q1 = sm.blk_off[blk + 1];
        if constexpr (GRID) {
          qa += q_lo;
          q_hi = qa + kChunkPairs;
          q1 = q_hi < q1 ? q_hi : q1;
        }
        for (int q0 = qa; q0 < q1; q0 += 32) {
          __syncwarp();
          const int q = q0 + lane;
          if (q >= q1) continue;
#ifdef MBA_PHASE_PROF
          {
            const unsigned am = __activemask();
            if (tid == 0) {
              s_prof[PH_NCAM] += __popc(am);
              s_prof[PH_NPAIR] += 1;
            }
          }
#endif
          const int2 pr = W.pair(q);
          T yi[18], yj[18];
          ld18(Ybuf + (size_t)pr.x * YSTR, yi);
          ld18(Ybuf + (size_t)pr.y * YSTR, yj);
#pragma unroll
          for (int r = 0; r < 6; ++r)
#pragma unroll
            for (int cc = 0; cc < 6; ++cc)
              acc[r * 6 + cc] += yi[r * 3] * yj[cc * 3] + yi[r * 3 + 1] * yj[cc * 3 + 1] +
                                 yi[r * 3 + 2] * yj[cc * 3 + 2];
        }
        if constexpr (GRID) {
          warp_reduce_to<T, 36>(acc, cpart + (size_t)item * kUcamStride, lane);
        } else {
          // acc[r][cc] = S(6sa + r, 6sb + cc); stored in the lower triangle
          warp_reduce_apply(acc, lane, [&](int i, T v) {
            const int r = i / 6, cc = i % 6;
            if (sa == sb) {
              if (cc <= r) S_jobs[acol(6 * sa + cc, C) + r - cc] = -v;
            } else {
              const int row = 6 * sb + cc, col = 6 * sa + r;
              S_jobs[acol(col, C) + row - col] = -v;
            }
          });
        }
      }
#ifdef MBA_PHASE_PROF
      if (tid == 0) {
        long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        s_prof[job < nf ? PH_ITEMS : PH_ITEMS2] += t_end - t_item;
        (void)0;
      }
#endif
    }
    PROF_MARK(PH_JOBS)
    gsync();
    PROF_MARK(PH_JWAIT)
    if constexpr (GRID) {
      // per-job totals of the chunk partials, in chunk order
      const int nu = nf * kUcamStride;
      for (int it2 = gtid; it2 < nu + nb * 36; it2 += gthreads) {
        const int job = it2 < nu ? it2 / kUcamStride : nf + (it2 - nu) / 36;
        const int i = it2 < nu ? it2 % kUcamStride : (it2 - nu) % 36;
        // the chunk partials in chunk order; eight loads in flight per step
        // (a job has up to ~25 chunks and each is an L2 round trip)
        T v = T(0);
        const int q1 = coff[job + 1];
        for (int q0 = coff[job]; q0 < q1; q0 += 8) {
          T pv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) pv[u] = q0 + u < q1 ? cpart[(size_t)(q0 + u) * kUcamStride + i] : T(0);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (q0 + u < q1) v += pv[u];
        }
        if (job < nf) {
          U_jobs[job * kUcamStride + i] = v;
        } else {
          const int blk = job - nf, sa = sm.blk_a[blk], sb = sm.blk_b[blk], r = i / 6, cc = i % 6;
          if (sa == sb) {
            if (cc <= r) S_jobs[acol(6 * sa + cc, C) + r - cc] = -v;
          } else {
            const int row = 6 * sb + cc, col = 6 * sa + r;
            S_jobs[acol(col, C) + row - col] = -v;
          }
        }
      }
      PROF_MARK(PH_JRED)
      gsync();
      PROF_MARK(PH_JSYNC)
      // both jobs' totals into shared memory on the TMA engine (one mbarrier
      // completion covers both copies)
      if (tid == 0) {
        const unsigned bS = bulk_bytes(CA * sizeof(T)), bU = bulk_bytes(nf * kUcamStride * sizeof(T));
        mbar_arm(&s_mbar, bS + bU);
        bulk_g2s(sm.S, S_jobs, bS, &s_mbar);
        bulk_g2s(sm.ucam, U_jobs, bU, &s_mbar);
      }
      mbar_wait(&s_mbar, mbar_phase);
      mbar_phase ^= 1u;
      __syncthreads();
    }
    PROF_MARK(PH_JRED)

    // ---------- assemble damped S and rhs (miniba.py:188-213) ----------
    if (!opt_pts) {
      for (int i = tid; i < CA; i += blockDim.x) sm.S[i] = T(0);
      __syncthreads();
    }
    for (int s = tid; s < nf; s += blockDim.x) {
      const T* u = sm.ucam + s * kUcamStride;
      int idx = 0;
      for (int r = 0; r < 6; ++r) {
        for (int cc = 0; cc <= r; ++cc, ++idx) {
          T ud = u[idx];
          if (r == cc) ud += tlam * (ud > T(kDiagFloor) ? ud : T(kDiagFloor));
          sm.S[acol(6 * s + cc, C) + r - cc] += ud;
        }
        const int col = 6 * s + r;
        if (has_f) sm.S[acol(col, C) + FI - col] = u[21 + r] - (opt_pts ? u[33 + r] : T(0));
        sm.S[acol(col, C) + C - col] = -u[27 + r] + (opt_pts ? u[39 + r] : T(0));  // rhs row
      }
    }
    if (has_f && tid == 0) {
      T uff = part[0];
      T ud = uff + tlam * (uff > T(kDiagFloor) ? uff : T(kDiagFloor));
      sm.S[acol(FI, C)] = ud - part[2];
      sm.S[acol(FI, C) + 1] = -part[1] + part[3];
    }
    __syncthreads();
    PROF_MARK(PH_ASM)

    // ---------- K4 LDL^T of the augmented system (mba_ldl.cuh) ----------
    bool chol_fail;
    {
      __shared__ T s_ltop[kLdlPanel * kLdlPanel];
      __shared__ int s_bad;
      chol_fail = ldl_blocked<T, NT>(sm.S, C, sm.rhs, (T*)(smem_raw + L::oTab), s_ltop, &s_bad);
    }
    if (it < 64 && ((cfg.fail_iters_mask >> it) & 1ull)) chol_fail = true;
    PROF_MARK(PH_CHOL)

    if (!chol_fail) {
      // back substitution D L^T x = y for the cameras (mba_ldl.cuh)
      ldl_backsub<T, NT>(sm.S, C, sm.rhs, (T*)(smem_raw + L::oTab), sm.dc);
      __syncthreads();
      PROF_MARK(PH_BSUB)
      // back substitution for the points (miniba.py:217)
      if (opt_pts) {
        const T df = has_f ? T(sm.dc[FI]) : T(0);
        for (int p = gtid; p < Pn; p += gthreads) {
          T* pw = ptw + (size_t)p * kPtStride;
          T u0 = pw[6] + pw[9] * df, u1 = pw[7] + pw[10] * df, u2 = pw[8] + pw[11] * df;
          for (int k = ptr[p]; k < ptr[p + 1]; ++k) {
            const int s = sm.slot[obs_cam(obs, k)];
            if (s < 0) continue;
            T y[18];
            ld18(Ybuf + (size_t)k * YSTR, y);
#pragma unroll
            for (int r = 0; r < 6; ++r) {
              const T dd = T(sm.dc[6 * s + r]);
              u0 += y[r * 3 + 0] * dd;
              u1 += y[r * 3 + 1] * dd;
              u2 += y[r * 3 + 2] * dd;
            }
          }
          const T L00 = pw[0], L10 = pw[1], L11 = pw[2], L20 = pw[3], L21 = pw[4], L22 = pw[5];
          T x2 = u2 / L22;
          T x1 = (u1 - L21 * x2) / L11;
          T x0 = (u0 - L10 * x1 - L20 * x2) / L00;
          pw[12] = -x0;
          pw[13] = -x1;
          pw[14] = -x2;
        }
      }
      gsync();
    }
    PROF_MARK(PH_SOLVE)

    // ---------- K5 trials, accept / reject, lambda (miniba.py:244-293) ----------
    if (lead) lambdas[it] = lam;
    int tries = 0, took = -1;
    double tc_[3] = {0, 0, 0};
    double ft = f;
    if (!chol_fail) {
      // all five trial camera sets at once (one thread per (try, camera))
      for (int q = tid; q < kBacktrackTries * n; q += blockDim.x) {
        const int bt = q / n, c = q % n, s = sm.slot[c];
        const double frac = ldexp(1.0, -bt);
        double* Rq = sm.Rt + (size_t)(bt * n + c) * 9;
        double* tq = sm.tt + (size_t)(bt * n + c) * 3;
        if (s < 0) {
          for (int i = 0; i < 9; ++i) Rq[i] = sm.Rc[9 * c + i];
          for (int i = 0; i < 3; ++i) tq[i] = sm.tc[3 * c + i];
        } else {
          double w[3] = {frac * sm.dc[6 * s], frac * sm.dc[6 * s + 1], frac * sm.dc[6 * s + 2]};
          double E[9];
          exp_so3(w, E);
          matmul33(E, sm.Rc + 9 * c, Rq);
          for (int i = 0; i < 3; ++i) tq[i] = sm.tc[3 * c + i] + frac * sm.dc[6 * s + 3 + i];
        }
      }
      __syncthreads();
      for (int bt = 0; bt < kBacktrackTries; ++bt) {
        const double frac = ldexp(1.0, -bt);
        ft = has_f ? f + frac * sm.dc[FI] : f;
        cost_pass<T>(obs, lo, K, X, ptw, frac, opt_pts, sm.Rt + (size_t)bt * n * 9,
                     sm.tt + (size_t)bt * n * 3, ft, cx, cy, delta, loss, sm.red, tc_, gtid, gthreads);
        grid_sum(tc_, 3);
        ++tries;
        if (tc_[0] < cost && isfinite(tc_[0])) {
          took = bt;
          break;
        }
      }
    }
    PROF_MARK(PH_TRIAL)
    if (lead) evals[it] = (uint8_t)tries;
    bool stop = false;
    if (took >= 0) {
      const double frac = ldexp(1.0, -took);
      for (int i = tid; i < n * 9; i += blockDim.x) sm.Rc[i] = sm.Rt[(size_t)took * n * 9 + i];
      for (int i = tid; i < n * 3; i += blockDim.x) sm.tc[i] = sm.tt[(size_t)took * n * 3 + i];
      if (opt_pts)
        for (int p = gtid; p < Pn; p += gthreads) {
          const T* dp = ptw + (size_t)p * kPtStride + 12;
          X[3 * p + 0] = X[3 * p + 0] + frac * (double)dp[0];
          X[3 * p + 1] = X[3 * p + 1] + frac * (double)dp[1];
          X[3 * p + 2] = X[3 * p + 2] + frac * (double)dp[2];
        }
      f = ft;
      lam = took == 0 ? fmax(lam / nu, 1e-15) : fmin(lam * nu, kLambdaMax);
      const double improve = cost - tc_[0];
      cost = tc_[0];
      se = tc_[1];
      se2 = tc_[2];
      if (lead) accepted[it] = 1;
      if (improve <= 1e-15 * fmax(cost, 1.0)) {
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
    if (lead) costs[it + 1] = cost;
    ++it;
    gsync();
    PROF_MARK(PH_COMMIT)
    if (stop) break;
  }

  // ---------------- outputs ----------------
  if (rank == 0) {
    for (int i = tid; i < n * 9; i += blockDim.x) O.R_out[cb * 9 + i] = sm.Rc[i];
    for (int i = tid; i < n * 3; i += blockDim.x) O.t_out[cb * 3 + i] = sm.tc[i];
  }
  if (lead) {
    O.focal_out[b] = f;
    O.n_iters[b] = it;
    O.status[b] = stop_reason;
    O.final_stats[4 * b + 0] = cost;
    O.final_stats[4 * b + 1] = se;
    O.final_stats[4 * b + 2] = se2;
    O.final_stats[4 * b + 3] = (double)K;
  }
  PROF_FLUSH
  __syncthreads();
}

template <typename T, int MAXC, bool RES, int NT = kThreads, int MINB = (sizeof(T) == 4 && !RES) ? 2 : 1>
__global__ void __launch_bounds__(NT, MINB) solve_kernel(SolveParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_prob;
  for (;;) {
    if (threadIdx.x == 0) s_prob = atomicAdd(P.counter, 1);
    __syncthreads();
    const int b = s_prob;
    __syncthreads();
    if (b >= P.d.n_problems) return;
    if (P.only_flagged && P.o.status[b] != v4::kStatusPlanOverflow) continue;
    solve_one<T, MAXC, RES, false, NT>(P, b, smem_raw);
  }
}

constexpr size_t kSmemLimit = 227 * 1024;

// Cooperative mode: every CTA of the grid works on the same problem (points,
// observations and Schur jobs are split across the grid; the small reduced
// camera system is factorised redundantly in every CTA, so no broadcast is
// needed). Problems of the batch are processed one after another.
template <typename T, int MAXC>
__global__ void __launch_bounds__(kThreads, 1) solve_grid_kernel(SolveParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  for (int b = 0; b < P.d.n_problems; ++b) {
    solve_one<T, MAXC, false, true>(P, b, smem_raw);
    cooperative_groups::this_grid().sync();
  }
}

template <typename T, int MAXC>
static int launch_grid(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const size_t scratch = scratch_bytes<T, false>(d->max_obs, d->max_points, d->max_pairs);
  const size_t smem = Layout<T, MAXC>::kFixed;
  if (smem > kSmemLimit) return MBA_ERR_TOO_LARGE;
  cudaFuncSetAttribute(solve_grid_kernel<T, MAXC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_grid_kernel<T, MAXC>, kThreads, smem);
  if (per_sm < 1) return MBA_ERR_TOO_LARGE;
  int grid = n_sm;  // one CTA per SM
  // enough observations per CTA to amortise the grid barriers
  const int64_t want = (d->max_obs + 511) / 512;
  if (want < grid) grid = (int)(want < 1 ? 1 : want);
  if (const char* e = getenv("MBA_GRID_CTAS")) {   // experiments: fewer CTAs
    const int v = atoi(e);
    if (v > 0 && v < grid) grid = v;
  }
  const int64_t chunks = grid_max_chunks(d->max_obs, d->max_pairs, MAXC);
  const size_t gbytes = align16(GridBufs<T, MAXC>::bytes(grid, chunks));
  if (ws_bytes < 256 + scratch + gbytes) return MBA_ERR_INVALID;
  SolveParams P;
  P.d = *d;
  P.cfg = *cfg;
  P.o = *o;
  P.counter = (int*)ws;
  P.ws = (unsigned char*)ws + 256;
  P.ws_slot_bytes = scratch;
  P.max_cams = d->max_cams;
  P.grid = P.ws + align16(scratch);
  P.grid_chunks = chunks;
  void* args[] = {&P};
  cudaLaunchCooperativeKernel((void*)solve_grid_kernel<T, MAXC>, dim3(grid), dim3(kThreads), args, smem, st);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}

template <typename T, int MAXC, bool RES, int NT = kThreads, int MINB = (sizeof(T) == 4 && !RES) ? 2 : 1>
static int launch_cfg(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o, void* ws,
                      size_t ws_bytes, cudaStream_t st, int only_flagged = 0) {
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const size_t scratch = scratch_bytes<T, RES>(d->max_obs, d->max_points, d->max_pairs);
  const size_t smem = Layout<T, MAXC>::kFixed + (RES ? scratch : 0);
  if (smem > kSmemLimit) return MBA_ERR_TOO_LARGE;
  cudaFuncSetAttribute(solve_kernel<T, MAXC, RES, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_kernel<T, MAXC, RES, NT, MINB>, NT, smem);
  if (const char* e = getenv("MBA_PER_SM")) { int v = atoi(e); if (v > 0 && v < per_sm) per_sm = v; }
  if (per_sm < 1) return MBA_ERR_TOO_LARGE;
  int grid = n_sm * per_sm;
  if (grid > d->n_problems) grid = d->n_problems;
  if (!RES && ws_bytes < 256 + scratch * (size_t)grid) return MBA_ERR_INVALID;
  SolveParams P;
  P.d = *d;
  P.cfg = *cfg;
  P.o = *o;
  P.counter = (int*)ws;
  P.ws = (unsigned char*)ws + 256;
  P.ws_slot_bytes = scratch;
  P.max_cams = d->max_cams;
  P.only_flagged = only_flagged;
  cudaMemsetAsync(ws, 0, sizeof(int), st);
  // (no persisting-L2 window: a process-wide carve-out would outlive this
  // call and shrink L2 for the caller's own kernels; the scratch slots are
  // L2-resident at the sizes this path serves anyway)
  solve_kernel<T, MAXC, RES, NT, MINB><<<grid, NT, smem, st>>>(P);
  return cudaGetLastError() == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}

// Shared-memory-resident scratch when the largest problem of the batch fits,
// else scratch in a per-CTA global slot (L2-resident for moderate sizes).
template <typename T, int MAXC>
static bool resident_fits(const MbaBatchDesc* d) {
  return d->max_obs < 65536 &&
         Layout<T, MAXC>::kFixed + scratch_bytes<T, true>(d->max_obs, d->max_points, d->max_pairs) <= kSmemLimit;
}

// Kernel choice: many small problems -> one warp per problem; otherwise one
// CTA per problem (scratch in shared memory when it fits).
static int choose_mode(const MbaBatchDesc* d, const MbaLmConfig* cfg) {
  // forced (tests, experiments): 2 CTA kernel, 4 cooperative grid, 9 cluster kernel
  if (cfg->ctas_per_problem < 0) return -cfg->ctas_per_problem;
  // the cluster-resident kernel whenever its shared-memory plan fits (<= 8
  // cameras): config 4 f64 250k problems/s vs 78k for the CTA kernel; a single
  // config-2 problem (K = 20k) in 0.44 ms on a 16-CTA cluster vs 2.43 ms for
  // the whole-GPU cooperative kernel. Plan overflows are re-solved by the CTA
  // kernel.
  if (v4::plan_cluster(d, cfg) > 0) return 0;
  // otherwise a few large problems spread over the whole GPU (cooperative grid)
  if (d->n_problems <= 8 && d->max_obs >= 4096) return 4;
  return 2;
}

template <typename T>
static int launch(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o, void* ws,
                  size_t ws_bytes, cudaStream_t st) {
  int mode = choose_mode(d, cfg);
  if (mode != 0 && mode != 2 && mode != 4 && mode != 9) return MBA_ERR_INVALID;
  if (mode == 0 && v4::plan_cluster(d, cfg) == 0) mode = 2;   // outside the cluster kernel's envelope
  if (mode == 9 || mode == 0) {
    // cluster-resident kernel; problems whose slices overflow its shared-memory
    // plan are re-solved by the CTA kernel (restricted to flagged problems)
    const int R = v4::plan_cluster(d, cfg);
    if (R > 0) {
      int rc = v4::launch(d, cfg, o, st, R, ws, ws_bytes);
      if (rc != MBA_OK || !v4::may_overflow(d, cfg)) return rc;
      return launch_cfg<T, 8, false>(d, cfg, o, ws, ws_bytes, st, 1);
    }
    if (mode == 9) return MBA_ERR_TOO_LARGE;
  }
  if (mode == 4) {
    if (d->max_cams <= 8) return launch_grid<T, 8>(d, cfg, o, ws, ws_bytes, st);
    if (d->max_cams <= 16) return launch_grid<T, 16>(d, cfg, o, ws, ws_bytes, st);
    if (d->max_cams <= 32) return launch_grid<T, 32>(d, cfg, o, ws, ws_bytes, st);
    return MBA_ERR_TOO_LARGE;
  }
  if (d->max_cams <= 8) {
    if (resident_fits<T, 8>(d)) return launch_cfg<T, 8, true>(d, cfg, o, ws, ws_bytes, st);
    return launch_cfg<T, 8, false>(d, cfg, o, ws, ws_bytes, st);
  }
  if (d->max_cams <= 16) {
    if (resident_fits<T, 16>(d)) return launch_cfg<T, 16, true>(d, cfg, o, ws, ws_bytes, st);
    return launch_cfg<T, 16, false>(d, cfg, o, ws, ws_bytes, st);
  }
  if (d->max_cams <= 32) return launch_cfg<T, 32, false>(d, cfg, o, ws, ws_bytes, st);
  return MBA_ERR_TOO_LARGE;
}

}  // namespace mba

extern "C" {

int32_t mba_abi_version(void) { return MBA_ABI_VERSION; }

#ifdef MBA_PHASE_PROF
int32_t mba_debug_set_phase_buffer(unsigned long long* dev_buf) {
  mba::v4::set_prof(dev_buf);
  return cudaMemcpyToSymbol(mba::g_prof, &dev_buf, sizeof(dev_buf)) == cudaSuccess ? MBA_OK : MBA_ERR_CUDA;
}
#endif

size_t mba_workspace_bytes(const MbaBatchDesc* d, const MbaLmConfig* cfg) {
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n_sm = 148;
  const bool f64 = cfg->precision == MBA_LIN_F64;
  const size_t slot = f64 ? mba::scratch_bytes<double, false>(d->max_obs, d->max_points, d->max_pairs)
                          : mba::scratch_bytes<float, false>(d->max_obs, d->max_points, d->max_pairs);
  const size_t gextra =
      mba::align16(mba::GridBufs<double, 32>::bytes(n_sm, mba::grid_max_chunks(d->max_obs, d->max_pairs, 32))) + 256;
  // one scratch slot per resident CTA of the CTA kernel (bounded by the batch)
  // plus the cooperative grid mode's cross-CTA buffers
  size_t grid = (size_t)n_sm * 16;
  if (grid > (size_t)d->n_problems) grid = (size_t)d->n_problems;
  return 256 + slot * grid + gextra;
}

int32_t mba_solve_plan(const MbaBatchDesc* d, const MbaLmConfig* cfg) {
  if (!d || !cfg || d->n_problems < 1 || d->max_cams < 1 || d->max_obs < 1) return 0;
  int mode = mba::choose_mode(d, cfg);
  if (mode == 0 || mode == 9) {
    const int R = mba::v4::plan_cluster(d, cfg);
    if (R > 0) return R;
    if (mode == 9) return 0;
    mode = 2;
  }
  return -mode;
}

int32_t mba_solve_launches(const MbaBatchDesc* d, const MbaLmConfig* cfg) {
  const int32_t p = mba_solve_plan(d, cfg);
  if (p == 0) return 0;
  if (p > 0) return mba::v4::may_overflow(d, cfg) ? 2 : 1;
  return 1;
}

int32_t mba_solve(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o,
                  void* ws, size_t ws_bytes, void* stream) {
  if (!d || !cfg || !o || d->n_problems < 0 || cfg->max_iters < 0) return MBA_ERR_INVALID;
  if (d->n_problems == 0) return MBA_OK;
  if (d->max_cams < 1 || d->max_obs < 1) return MBA_ERR_EMPTY;
  if (d->max_obs > 0x7fffffff || d->max_points > 0x7ffffffe || d->max_pairs > 0x7fffffff)
    return MBA_ERR_TOO_LARGE;
  cudaStream_t st = (cudaStream_t)stream;
  if (cfg->precision == MBA_LIN_F64) return mba::launch<double>(d, cfg, o, ws, ws_bytes, st);
  return mba::launch<float>(d, cfg, o, ws, ws_bytes, st);
}

}  // extern "C"
