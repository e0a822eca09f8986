"""Time gsrecon.miniba.lm_solve_batch end to end on a list of BaProblem
objects (host arrays in, solved host arrays out): config 4 by default.

    python scripts/bench_e2e_api.py [--problems 65536] [--steps 3] [--precision f64]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "src")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--precision", default="f64")
    ap.add_argument("--chunks", type=int, default=16)
    ap.add_argument("--ring", type=int, default=4)
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    import torch
    from gsrecon.config import LmConfig
    from gsrecon.miniba import BaProblem, lm_solve_batch, _SOLVERS
    from paper_2506_05558_b200.batch import BatchSolver
    from paper_2506_05558_b200.synth import make_batch
    t0 = time.perf_counter()
    b = make_batch(a.problems, n_cams=8, K=2000, seed=0, workers=len(os.sched_getaffinity(0)))
    probs = []
    for i in range(a.problems):
        p = b.problem(i)
        p["cam_idx"] = p["cam_idx"].astype(np.int64)
        p["pt_idx"] = p["pt_idx"].astype(np.int64)
        probs.append(BaProblem(**p))
    init = [(p.R.copy(), p.t.copy(), p.focal, p.points.copy()) for p in probs]
    gen = time.perf_counter() - t0
    bs = BatchSolver(None, n_chunks=a.chunks, threads=a.threads or None, ring=a.ring)
    _SOLVERS[torch.cuda.current_device()] = bs
    cfg = LmConfig(max_iters=200)
    times = []
    for s in range(a.steps + 1):
        for p, (R, t, f, X) in zip(probs, init):
            p.R[...] = R
            p.t[...] = t
            p.focal = f
            p.points[...] = X
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        infos = lm_solve_batch(probs, cfg, precision=a.precision)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t1
        if s:
            times.append(dt)
    st = np.asarray(infos.status)
    print(json.dumps({"problems": a.problems, "precision": a.precision, "chunks": a.chunks,
                      "threads": bs.threads, "s_per_call": times,
                      "problems_per_s": a.problems / float(np.median(times)),
                      "h2d_bytes": bs.h2d_bytes, "d2h_bytes": bs.d2h_bytes,
                      "mean_iters": float(np.mean(infos.n_iters)), "status_ok": int(np.sum(st >= 0)),
                      "host_s_last_call": bs.host_s,
                      "gen_s": gen}))


if __name__ == "__main__":
    main()
