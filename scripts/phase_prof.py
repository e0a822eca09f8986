"""Per-phase cycle breakdown of the solver kernels (profiling build of
libminiba, -DMBA_PHASE_PROF; rebuilt here when a source is newer).

    python scripts/phase_prof.py --config 4 --problems 8192 [--precision mixed]
"""
import argparse
import ctypes as ct
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "src")]
_PROF = os.path.join(REPO, "paper_2506_05558_b200", "libminiba_prof.so")
os.environ["MBA_LIB"] = os.environ.get("MBA_PROF_LIB") or _PROF


def _ensure_prof_lib():
    """Rebuild the profiling library when any CUDA source is newer (a stale
    one silently reports the previous code's phases)."""
    if os.environ.get("MBA_PROF_LIB"):
        return
    csrc = os.path.join(REPO, "paper_2506_05558_b200", "csrc")
    srcs = [os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith((".cu", ".cuh"))]
    if os.path.exists(_PROF) and all(os.path.getmtime(f) <= os.path.getmtime(_PROF) for f in srcs):
        return
    from paper_2506_05558_b200 import build
    build.build(prof=True)

# index -> phase; the cluster kernel (mba_v4.cu) and the CTA / grid kernels
# (mba_solve.cu) share 0-8; 9-10 are ldl-core / unused (v4) and
# jobs-barrier-wait / job-reduction (grid mode)
PHASES = ["setup", "cost0", "point", "jobs", "assemble", "cholesky", "solve+backsub", "trials", "commit",
          "ldl|jobs_wait", "camera_backsub(v4)|jobs_reduce", "setup_stage_validate|cam_chunks_cyc", "setup_slots_X|pair_chunks_cyc",
          "setup_perm|n_cam_chunks", "setup_pairs|n_pair_chunks", "camera_backsub", "jobs_reduce_sync"]   # the last: CTA / grid kernels


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--problems", type=int, default=8192)
    ap.add_argument("--precision", default="mixed")
    ap.add_argument("--kernel", default="auto")
    a = ap.parse_args()
    _ensure_prof_lib()
    import torch
    from paper_2506_05558_b200 import _lib, solver
    from paper_2506_05558_b200.synth import CONFIGS, make_batch
    c = CONFIGS[a.config]
    n = min(a.problems, c["n_problems"])
    b = make_batch(n, n_cams=c["n_cams"], K=c["K"], outlier_frac=c.get("outlier_frac", 0.0),
                   workers=os.cpu_count())
    db = solver.to_device(solver.pack_synth(b))
    prm = solver.LmParams(max_iters=c["max_iters"], loss=c["loss"], precision=a.precision,
                          kernel=a.kernel)
    L = _lib.lib()
    buf = torch.zeros(32, dtype=torch.int64, device="cuda")
    L.mba_debug_set_phase_buffer.argtypes = [ct.c_void_p]
    sol = solver.solve(db, prm)
    torch.cuda.synchronize()
    L.mba_debug_set_phase_buffer(ct.c_void_p(buf.data_ptr()))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    solver.solve(db, prm, sol)
    ev[1].record()
    torch.cuda.synchronize()
    cyc = buf.cpu().numpy()[:len(PHASES)].astype(float)
    tot = cyc.sum()
    iters = float(sol.n_iters.sum().item())
    out = {"config": a.config, "problems": n, "precision": a.precision, "kernel": a.kernel,
           "cluster_env": os.environ.get("MBA_V4_R"), "note": "cycles summed over every CTA of a cluster", "ms": ev[0].elapsed_time(ev[1]),
           "lm_iters": iters,
           "phases": {p: {"frac": c_ / tot, "cycles_per_problem_iter": c_ / iters} for p, c_ in zip(PHASES, cyc)}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
