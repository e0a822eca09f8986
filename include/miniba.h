/*
 * miniba.h -- C ABI of the B200-native mini bundle adjustment (libminiba.so).
 *
 * The reference (`/root/reference/pkg/src/gsrecon/miniba.py`) is a pure
 * Python/numpy package with no FFI layer; its drop-in boundary is the Python
 * surface of `gsrecon.miniba` that `pkg/smoke_miniba.py` imports. The Python
 * host package `src/gsrecon` keeps that surface and binds these entry points
 * with ctypes. Each entry point names the reference
 * function it replaces.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller (torch
 *    tensors on the Python side); the library never allocates on the hot path.
 *  - float64 parameter state; int32 local indices; 16-byte observation records.
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*).
 *  - Return value: MBA_OK or a negative MbaStatus; per-problem solver
 *    outcomes are data (MbaOutputs.status), not errors.
 */
#ifndef MINIBA_H_
#define MINIBA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MBA_ABI_VERSION 1

enum MbaStatus {
  MBA_OK = 0,
  MBA_ERR_INVALID = -1,     /* bad descriptor / argument (-> ValueError)          */
  MBA_ERR_TOO_LARGE = -2,   /* problem exceeds the shared-memory plan             */
  MBA_ERR_CUDA = -3,        /* CUDA launch / runtime failure                      */
  MBA_ERR_EMPTY = -4,       /* a problem has no residuals (miniba.py:229-230)     */
  MBA_ERR_NOT_PD = -5       /* stage solve: reduced system not PD (LinAlgError)   */
};

enum MbaLoss { MBA_LOSS_HUBER = 0, MBA_LOSS_CAUCHY = 1 };

/* arithmetic of the linearise / Schur / Cholesky stages; state and the
 * residual / cost passes are always float64 */
enum MbaPrecision { MBA_LIN_F32 = 0, MBA_LIN_F64 = 1 };

/* per-problem solver outcome (MbaOutputs.status) */
enum MbaSolveStatus {
  MBA_SOLVE_MAX_ITERS = 0,   /* ran max_iters iterations                        */
  MBA_SOLVE_CONVERGED = 1,   /* improve <= 1e-15 max(cost,1)  (miniba.py:285)   */
  MBA_SOLVE_LAMBDA_CAP = 2   /* rejected with lambda >= 1e10  (miniba.py:292)   */
};

/* One observation: pixel (u, v) rounded to float, local camera and point index.
 * Within a problem the records are sorted point-major (all observations of
 * point 0, then point 1, ...). */
typedef struct {
  float u, v;
  int32_t cam;
  int32_t pt;
} MbaObs;

/* A batch of independent problems, packed back to back (BaProblem,
 * miniba.py:65-83). Offsets are int64 arrays of length n_problems + 1. */
typedef struct {
  int32_t n_problems;
  int32_t max_cams;          /* max cameras in any problem            */
  int64_t max_obs;           /* max observations in any problem       */
  int64_t max_points;        /* max points in any problem             */
  int64_t max_pairs;         /* max over problems of sum_p m_p (m_p + 1) / 2, m_p =
                                observations of point p (co-observation pairs)  */
  int32_t max_track;         /* max observations of any single point           */
  int32_t reserved;
  const int64_t* cam_off;    /* camera rows of problem b: [cam_off[b], cam_off[b+1]) */
  const int64_t* pt_off;
  const int64_t* obs_off;
  const MbaObs* obs;         /* [total_obs]                                      */
  const float* obs_lo;       /* [total_obs][2] uv - float(uv) (exact fp64 uv), or NULL */
  const uint8_t* fixed;      /* [total_cams] 1 = fixed camera (miniba.py:78)     */
  const double* cx;          /* [n_problems]                                      */
  const double* cy;          /* [n_problems]                                      */
  const uint8_t* flags;      /* [n_problems] bit0 optimize_focal, bit1 optimize_points */
} MbaBatchDesc;

/* LmConfig (config.py:9-17) plus the loss / precision extensions */
typedef struct {
  double lambda_init;
  double nu;
  double delta;              /* Huber delta / Cauchy scale, px            */
  int32_t max_iters;
  int32_t loss;              /* MbaLoss                                   */
  int32_t precision;         /* MbaPrecision                              */
  int32_t ctas_per_problem;  /* 0 = auto; >1 = thread-block cluster per problem */
  uint64_t fail_iters_mask;  /* fault injection (tests): bit i forces the solve of
                                iteration i to fail like a LinAlgError (miniba.py:247-251) */
} MbaLmConfig;

/* Parameter state in / out and the LM traces (lm_solve return dict,
 * miniba.py:294-296). *_in may alias *_out. */
typedef struct {
  const double* R_in;        /* [total_cams][3][3] */
  const double* t_in;        /* [total_cams][3]    */
  const double* focal_in;    /* [n_problems]       */
  const double* points_in;   /* [total_points][3]  */
  double* R_out;
  double* t_out;
  double* focal_out;
  double* points_out;
  double* costs;             /* [n_problems][max_iters+1] robust cost trace      */
  double* lambdas;           /* [n_problems][max_iters]                          */
  uint8_t* accepted;         /* [n_problems][max_iters]                          */
  uint8_t* evals;            /* [n_problems][max_iters] trial passes executed    */
  int32_t* n_iters;          /* [n_problems]                                     */
  int32_t* status;           /* [n_problems] MbaSolveStatus                      */
  double* final_stats;       /* [n_problems][4]: cost, sum e, sum e^2, K         */
} MbaOutputs;

/* Device-side packing of raw per-problem observation arrays (BaProblem
 * cam_idx / pt_idx / uv, miniba.py:65-83, uploaded back to back per problem as
 * int32 / int32 / uv rounded to float32, plus -- only when some pixel is not
 * fp32-representable -- the low-order float32 residual uv_lo = uv - float(uv))
 * into the MbaObs records mba_solve consumes: stable point-major order within
 * each problem (numpy argsort(kind="stable") of pt_idx) and, when out_lo and
 * uv_lo are not NULL, the low-order stream in the same order. Replaces the
 * host-side sort of the producers' track-major (miniba.py:762-770) or
 * camera-major (smoke_miniba.py:50-55) arrays. Problems with an out-of-range
 * index are written unsorted; mba_solve then reports them malformed
 * (status -1). workspace: >= mba_pack_obs_workspace_bytes(total points) bytes. */
size_t mba_pack_obs_workspace_bytes(int64_t total_points);
int32_t mba_pack_obs(int32_t n_problems, const int64_t* obs_off, const int64_t* pt_off,
                     const int64_t* cam_off, const int32_t* cam, const int32_t* pt, const float* uv,
                     const float* uv_lo, MbaObs* out, float* out_lo, void* workspace,
                     size_t workspace_bytes, void* stream);

/* The bootstrap schedule around lm_solve (miniba.py:782-805, run_schedule) as
 * one device sequence over a batch of independent problems, no host round
 * trip: mba_solve with cfg1 (first half of the iterations, out1) -> residual
 * norms of that state and the robust filter e <= median + mad_factor * MAD
 * (miniba.py:57-62), observations of points left with < 2 survivors dropped
 * -> stable compaction into obs2 / obs_lo2 with offsets obs_off2 (n_kept per
 * problem; 0 means the filter removed everything: BootstrapFailure) ->
 * mba_solve with cfg2 continuing from out1's state (out2->*_in must equal
 * out1->*_out) -> gauge: t and points scaled by 1 / mean pairwise camera
 * distance (gauge_scale receives that distance; may be NULL). pt_alive[p] = 1
 * for points that keep observations (the reference's surviving tracks). */
size_t mba_bootstrap_workspace_bytes(const MbaBatchDesc* desc, const MbaLmConfig* cfg1);
int32_t mba_bootstrap_schedule(const MbaBatchDesc* desc, const MbaLmConfig* cfg1,
                               const MbaLmConfig* cfg2, double mad_factor, const MbaOutputs* out1,
                               const MbaOutputs* out2, MbaObs* obs2, float* obs_lo2,
                               int64_t* obs_off2, int64_t* n_kept, uint8_t* pt_alive,
                               double* gauge_scale, void* workspace, size_t workspace_bytes,
                               void* stream);

/* Packs the per-problem LM traces of an mba_solve (MbaOutputs costs /
 * lambdas / accepted / evals, max_iters wide) back to back before a read-back:
 * trace_off[b] = sum of n_iters over problems before b (n_problems + 1
 * entries); problem b's n_iters lambdas / accepted / evals land at
 * trace_off[b] and its n_iters + 1 costs at trace_off[b] + b. Output buffers
 * are sized for the worst case (n_problems * max_iters, costs + n_problems). */
int32_t mba_compact_traces(int32_t n_problems, int32_t max_iters, const int32_t* n_iters,
                           const double* costs, const double* lambdas, const uint8_t* accepted,
                           const uint8_t* evals, int64_t* trace_off, double* costs_out,
                           double* lambdas_out, uint8_t* accepted_out, uint8_t* evals_out,
                           void* stream);

int32_t mba_abi_version(void);

/* Bytes of device workspace mba_solve needs for this batch and config (scratch
 * of the CTA kernel and the cooperative grid buffers; the cluster kernel also
 * keeps per-SM linearisation caches in it when it is large enough). */
size_t mba_workspace_bytes(const MbaBatchDesc* desc, const MbaLmConfig* cfg);

/* Full Levenberg-Marquardt mini-BA on every problem of the batch: replaces
 * lm_solve (miniba.py:223-296) with its helpers residuals (85-98),
 * huber_cost/weights (46-54), _build_blocks (101-132), _assemble (135-177)
 * and solve_step(method="schur") (180-220). The whole LM loop runs on device;
 * no host round trip per iteration. */
int32_t mba_solve(const MbaBatchDesc* desc, const MbaLmConfig* cfg, const MbaOutputs* out,
                  void* workspace, size_t workspace_bytes, void* stream);

/* Which device path mba_solve takes for this batch and config: the cluster
 * size R > 0 of the cluster-resident kernel (R CTAs per problem, all scratch in
 * shared memory; fused backtracking tries 1-4), or -2 CTA per problem (9-32
 * cameras, overflow re-solves), -4 whole-GPU cooperative (a few large
 * problems); 0 = not solvable (more than 32 cameras: the stage kernels). */
int32_t mba_solve_plan(const MbaBatchDesc* desc, const MbaLmConfig* cfg);

/* Number of kernel launches one mba_solve call issues for this batch and config
 * (the cluster-resident kernel plus, when some problem may exceed its plan, the
 * CTA kernel restricted to those problems). */
int32_t mba_solve_launches(const MbaBatchDesc* desc, const MbaLmConfig* cfg);

/* ---- stage entry points (float64), for the reference's internal API ---- */

/* BaProblem.residuals (miniba.py:85-98): r [K][2], p_cam [K][3], bad [K] */
int32_t mba_residuals(int64_t K, const double* R, const double* t, double focal, double cx,
                      double cy, const double* points, const int64_t* cam_idx,
                      const int64_t* pt_idx, const double* uv, double* r, double* p_cam,
                      uint8_t* bad, void* stream);

/* huber_cost / huber_weights (miniba.py:46-54) and the Cauchy extension:
 * w [n] (may be NULL) and the summed cost into cost[0] (may be NULL). */
int32_t mba_robust(int64_t n, const double* e, double delta, int32_t loss, double* w,
                   double* cost, void* stream);

/* _build_blocks (miniba.py:101-132): A [K][2][6], F [K][2], B [K][2][3] */
int32_t mba_blocks(int64_t K, const double* R, const double* t, double focal,
                   const int64_t* cam_idx, const double* p_cam, const uint8_t* bad, double* A,
                   double* F, double* B, void* stream);

/* _assemble (miniba.py:135-177). Observation orders are supplied by the
 * caller: pt_order/pt_ptr (observations grouped by point, P+1 offsets) and
 * cam_order/cam_ptr (grouped by camera, n+1 offsets); slot[n_cams] maps a
 * camera to its free-camera slot (-1 = fixed), cam_of_slot[n_free] inverts it.
 * Outputs dense U [C][C], g_c [C], V [P][3][3], g_p [P][3], Wf [P][C][3]
 * (zeroed by the call). */
int32_t mba_assemble(int64_t K, int32_t n_cams, int32_t n_free, int64_t P, const int32_t* slot,
                     const int32_t* cam_of_slot, int32_t optimize_focal, int32_t optimize_points,
                     const int64_t* cam_idx, const double* w, const double* r, const double* A,
                     const double* F, const double* B, const int64_t* pt_order,
                     const int64_t* pt_ptr, const int64_t* cam_order, const int64_t* cam_ptr,
                     double* U, double* g_c, double* V, double* g_p, double* Wf, void* stream);

/* solve_step (miniba.py:180-220); method 0 = schur, 1 = dense. Writes dc [C],
 * dp [P][3]. `scratch` must hold mba_solve_step_scratch_bytes(C, P, method).
 * Returns MBA_ERR_NOT_PD when the factorisation fails (np.linalg.LinAlgError). */
size_t mba_solve_step_scratch_bytes(int32_t C, int64_t P, int32_t method);
int32_t mba_solve_step(int32_t C, int64_t P, const double* U, const double* g_c,
                       const double* V, const double* g_p, const double* Wf, double lam,
                       int32_t method, double* dc, double* dp, void* scratch, void* stream);

/* Batched pose-only LM (pose_lm, miniba.py:334-389): nb problems of m
 * correspondences each, `iters` single-trial iterations. R/t updated in
 * place; cost [nb]. If X_all/uv_all are given, also scores every refined
 * hypothesis on the full correspondence set (estimate_pose_ransac,
 * miniba.py:418-431): inlier count [nb] and inlier sum of squared errors [nb]. */
int32_t mba_pose_lm(int32_t nb, int32_t m, const double* X, const double* uv, double focal,
                    double cx, double cy, int32_t iters, double lambda_init, double nu,
                    double delta, double* R, double* t, double* cost, int32_t m_all,
                    const double* X_all, const double* uv_all, double inlier_px,
                    int32_t* inliers, double* inlier_sse, void* stream);

/* Batched triangulation (triangulate, miniba.py:458-530), one
 * track per thread: track k's observations are [obs_off[k], obs_off[k+1]) with
 * camera index cam[] into R [n_cams][3][3] / t [n_cams][3] and pixel uv[][2].
 * Widest-angle ray pair midpoint, gn_steps Gauss-Newton steps, mean
 * reprojection check. Outputs X [n_tracks][3] (NaN on failure), status
 * [n_tracks] (0 ok, 1 fewer than two views, 2 baseline angle <= min_angle_deg,
 * 3 parallel rays, 4 point behind a camera, 5 mean reprojection > max_reproj_px
 * -- the reference's TriangulationFailure cases), mean_err [n_tracks] (may be NULL). */
int32_t mba_triangulate(int32_t n_tracks, const int64_t* obs_off, const int32_t* cam, const double* uv,
                        int32_t n_cams, const double* R, const double* t, double focal, double cx,
                        double cy, double max_reproj_px, double min_angle_deg, int32_t gn_steps,
                        double* X, int32_t* status, double* mean_err, void* stream);

/* Batched descriptor matching (frontend.match, frontend.py:220-250; the
 * exhaustive pairwise matching of build_tracks, miniba.py:555-591; SURVEY
 * 8(f)-3). desc: n_frames' 256-bit descriptors, 32 bytes each, frame f's rows
 * [desc_off[f], desc_off[f+1]). pairs: n_pairs (frame_a, frame_b). row_off_a /
 * row_off_b [n_pairs]: where pair p's per-row outputs start for the rows of
 * frame_a / frame_b; max_rows >= the largest frame. Per row of frame_a:
 * match_b (index in frame_b of the mutual ratio-tested nearest neighbour, or -1)
 * and dist (its Hamming distance); nn_ab/ok_a/best_ab/nn_ba/ok_b are the
 * per-direction scratch results (caller-sized like the row offsets: rows_a /
 * rows_b entries). Every distance is computed once (64 x 64 tiles with row and
 * column partial minima); workspace >= mba_match_workspace_bytes(rows_a,
 * rows_b, max_rows) bytes holds the partials. */
size_t mba_match_workspace_bytes(int64_t rows_a, int64_t rows_b, int64_t max_rows);
int32_t mba_match_pairs(int32_t n_frames, const uint8_t* desc, const int64_t* desc_off, int32_t n_pairs,
                        const int32_t* pairs, const int64_t* row_off_a, const int64_t* row_off_b,
                        int64_t max_rows, double ratio_max, int32_t* nn_ab, uint8_t* ok_a, int32_t* best_ab,
                        int32_t* nn_ba, uint8_t* ok_b, int32_t* match_b, int32_t* dist, int64_t rows_a,
                        int64_t rows_b, void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MINIBA_H_ */
