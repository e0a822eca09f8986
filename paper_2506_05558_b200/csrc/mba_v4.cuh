// mba_v4.cuh -- internal interface of the cluster-resident mini-BA solver
// (mba_v4.cu), used by the mba_solve dispatcher in mba_solve.cu.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/miniba.h"

namespace mba {
namespace v4 {

// Per-problem status written when a problem does not fit the shared-memory
// plan of the cluster-resident kernel; the dispatcher re-solves exactly those
// problems with the CTA kernel (MBA_SOLVE_* codes are >= 0).
constexpr int kStatusPlanOverflow = -2;

// The kernel is compiled once per arithmetic type (mba_v4.cu built with and
// without -DMBA_V4_F32: two translation units, compiled in parallel); these
// are the per-type entry points, dispatched below on cfg->precision.
int plan_cluster_f64(const MbaBatchDesc* d);
int plan_cluster_f32(const MbaBatchDesc* d);
int launch_f64(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o, cudaStream_t st, int R,
               void* ws, size_t ws_bytes);
int launch_f32(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o, cudaStream_t st, int R,
               void* ws, size_t ws_bytes);
int may_overflow_f64(const MbaBatchDesc* d);
int may_overflow_f32(const MbaBatchDesc* d);
#ifdef MBA_PHASE_PROF
void set_prof_f64(unsigned long long* p);
void set_prof_f32(unsigned long long* p);
#endif

constexpr int kMaxCams = 8;   // cameras per problem the kernel's layout holds

// Cluster size (CTAs per problem) the kernel would use, or 0 if the batch is
// outside its envelope (more than 8 cameras, too large for a 16-CTA cluster).
inline int plan_cluster(const MbaBatchDesc* d, const MbaLmConfig* cfg) {
  if (d->max_cams > kMaxCams || d->max_cams < 1 || d->max_obs >= 65535 * 16) return 0;
  return cfg->precision == MBA_LIN_F64 ? plan_cluster_f64(d) : plan_cluster_f32(d);
}

// Launch the solver; returns MBA_OK / negative MbaStatus. Problems that do not
// fit report kStatusPlanOverflow (the caller then runs the CTA kernel
// restricted to those problems). `ws` (optional, the mba_solve workspace)
// holds the per-SM linearisation caches of plans whose shared memory has no
// room for them.
inline int launch(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o, cudaStream_t st,
                  int cluster, void* ws = nullptr, size_t ws_bytes = 0) {
  if (plan_cluster(d, cfg) != cluster || cluster == 0) return MBA_ERR_TOO_LARGE;
  return cfg->precision == MBA_LIN_F64 ? launch_f64(d, cfg, o, st, cluster, ws, ws_bytes)
                                       : launch_f32(d, cfg, o, st, cluster, ws, ws_bytes);
}

// 0 when no problem of the batch can exceed the plan (one CTA per problem and
// the descriptor maxima fit), so the overflow re-solve launch can be skipped.
inline int may_overflow(const MbaBatchDesc* d, const MbaLmConfig* cfg) {
  if (plan_cluster(d, cfg) == 0) return 1;
  return cfg->precision == MBA_LIN_F64 ? may_overflow_f64(d) : may_overflow_f32(d);
}

#ifdef MBA_PHASE_PROF
inline void set_prof(unsigned long long* p) {
  set_prof_f64(p);
  set_prof_f32(p);
}
#endif

}  // namespace v4
}  // namespace mba
