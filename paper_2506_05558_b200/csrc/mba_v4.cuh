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

// Cluster size (CTAs per problem) the kernel would use, or 0 if the batch is
// outside its envelope (more than 8 cameras, too large for a 16-CTA cluster).
int plan_cluster(const MbaBatchDesc* d, const MbaLmConfig* cfg);

// Launch the solver; returns MBA_OK / negative MbaStatus. Problems that do not
// fit report kStatusPlanOverflow (the caller then runs the CTA kernel
// restricted to those problems).
int launch(const MbaBatchDesc* d, const MbaLmConfig* cfg, const MbaOutputs* o, cudaStream_t st,
           int cluster);

// 0 when no problem of the batch can exceed the plan (one CTA per problem and
// the descriptor maxima fit), so the overflow re-solve launch can be skipped.
int may_overflow(const MbaBatchDesc* d, const MbaLmConfig* cfg);

#ifdef MBA_PHASE_PROF
void set_prof(unsigned long long* p);
#endif

}  // namespace v4
}  // namespace mba
