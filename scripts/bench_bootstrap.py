"""Measurement of the SURVEY 8(f)-2 row: the bootstrap schedule around
lm_solve (miniba.py:729-854: track building, 100 LM iterations, median + 4 MAD
filter and track compaction, 100 more LM iterations, gauge normalisation), on
the reference's own bootstrap oracle problems (tests/golden/bootstrap_seed*.npz,
8 cameras, 300 points, 0.5 px noise).

    python scripts/bench_bootstrap.py            # this package (device lm_solve), GPU box
    python scripts/bench_bootstrap.py --ref      # the unmodified reference, CPU (needs
                                                 # /root/reference; this container only)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")


def _inputs(seed):
    z = np.load(f"{GOLDEN}/bootstrap_seed{seed}.npz")
    feats, o = [], 0
    for c in z["counts"]:
        feats.append((z["keypoints"][o:o + c], z["ids"][o:o + c]))
        o += c
    return z, feats


def _matcher(fa, fb):
    ida, idb = fa[1], fb[1]
    pos = {int(v): j for j, v in enumerate(idb)}
    ia, ib = [], []
    for i, v in enumerate(ida):
        j = pos.get(int(v))
        if j is not None:
            ia.append(i)
            ib.append(j)
    return np.array(ia, dtype=np.int64), np.array(ib, dtype=np.int64), np.zeros(len(ia))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    if a.ref:
        os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
        sys.path.insert(0, "/root/reference/pkg/src")
    else:
        sys.path[:0] = [REPO, os.path.join(REPO, "src")]
    from gsrecon import miniba as M
    from gsrecon.config import CaptureConfig
    from gsrecon.scene import CameraIntrinsics
    sync = (lambda: None)
    if not a.ref:
        import torch
        sync = torch.cuda.synchronize
    out = []
    for seed in (0, 1):
        z, feats = _inputs(seed)
        intr = CameraIntrinsics(float(z["focal"]), float(z["cx"]), float(z["cy"]), int(z["width"]),
                                int(z["height"]))
        M.bootstrap(feats, intr, CaptureConfig(), matcher=_matcher)   # warm-up (imports, JIT, context)
        sync()
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            poses, intr_out, table, info = M.bootstrap(feats, intr, CaptureConfig(), matcher=_matcher)
            sync()
            ts.append(time.perf_counter() - t0)
        err = max(np.abs(p.R - R).max() for p, R in zip(poses, z["out_R"]))
        out.append({"seed": seed, "median_s": float(np.median(ts)), "focal": float(intr_out.focal),
                    "ref_focal": float(z["out_focal"]), "max_R_diff_vs_reference_output": float(err)})
    batched = None
    if not a.ref:
        # many windows through ONE device schedule (bootstrap_batch): the 20
        # acceptance windows (tests/golden/bootstrap20.npz) replicated
        z20 = np.load(f"{GOLDEN}/bootstrap20.npz")
        wins, o = [], 0
        counts = z20["counts"].reshape(20, -1)
        for s_ in range(20):
            w = []
            for c in counts[s_]:
                w.append((z20["kp"][o:o + c], z20["ids"][o:o + c]))
                o += c
            wins.append(w)
        intrs = [CameraIntrinsics(float(z20["focal"][s_]), float(z20["cx"][s_]), float(z20["cy"][s_]),
                                  int(z20["width"][s_]), int(z20["height"][s_])) for s_ in range(20)]
        reps = 8
        W, I = wins * reps, intrs * reps
        M.bootstrap_batch(W, I, CaptureConfig(), matcher=_matcher)
        sync()
        from gsrecon import _bootstrap as B_
        sched_s = []
        orig = B_.schedule_batch

        def timed(*args, **kw):
            t = time.perf_counter()
            out = orig(*args, **kw)
            sched_s.append(time.perf_counter() - t)
            return out
        B_.schedule_batch = timed
        t0 = time.perf_counter()
        res = M.bootstrap_batch(W, I, CaptureConfig(), matcher=_matcher)
        sync()
        dt = time.perf_counter() - t0
        B_.schedule_batch = orig
        batched = {"windows": len(W), "seconds": dt, "bootstraps_per_s": len(W) / dt,
                   "device_schedule_seconds": sched_s,
                   "schedule_bootstraps_per_s": len(W) / sched_s[0] if sched_s else None,
                   "failures": sum(isinstance(r, Exception) for r in res),
                   "note": "host track building (exact matcher) + one device schedule + the rescue schedule"}
    print(json.dumps({"metric": "bootstrap wall time (SURVEY 8(f)-2)", "batched": batched,
                      "impl": "reference (CPU, numpy/scipy)" if a.ref else "this package (device lm_solve)",
                      "cores": len(os.sched_getaffinity(0)), "runs": out}))


if __name__ == "__main__":
    main()
