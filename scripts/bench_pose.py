"""Measurement of the SURVEY 8(f)-1 row: batched pose-only LM (pose_lm,
miniba.py:334-389; the RANSAC-hypothesis batch of estimate_pose_ransac).

Device: mba_pose_lm (one warp per pose problem, lanes over correspondences,
6x6 normal equations by warp butterflies, register Cholesky, single trial per
iteration), inputs resident on the GPU, CUDA-event timed. CPU: the oracle port
of pose_lm (numpy, 1 thread) on a bounded prefix of the same inputs. Parity: the
device final costs against the oracle's on that prefix.

    python scripts/bench_pose.py [--batch 4096 --m 256 --iters 5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "src")]
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")


def make_inputs(B, M, seed=0):
    from gsrecon.scene import exp_so3
    rng = np.random.default_rng(seed)
    f, cx, cy = 520.0, 320.0, 240.0
    X = rng.uniform(-0.6, 0.6, (B, M, 3)) + np.array([0.0, 0.0, 2.0])
    uv = np.stack([f * X[..., 0] / X[..., 2] + cx, f * X[..., 1] / X[..., 2] + cy], -1)
    uv += rng.normal(0.0, 0.5, uv.shape)
    out = rng.random((B, M)) < 0.1                       # 10 % outliers
    uv[out] = rng.uniform([0, 0], [640, 480], (int(out.sum()), 2))
    R0 = np.stack([exp_so3(rng.normal(0, 0.02, 3)) for _ in range(B)])
    t0 = rng.normal(0, 0.02, (B, 3))
    return R0, t0, X, uv, (f, cx, cy)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--m", type=int, default=256)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--cpu-problems", type=int, default=256)
    a = ap.parse_args()
    import torch
    from oracle import miniba_oracle as O
    from paper_2506_05558_b200 import _lib
    from paper_2506_05558_b200._lib import ptr

    B, M, it = a.batch, a.m, a.iters
    R0, t0, X, uv, (f, cx, cy) = make_inputs(B, M)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    dX, dU, dR0, dt0 = dev(X), dev(uv), dev(R0), dev(t0)
    R, t = dR0.clone(), dt0.clone()
    cost = torch.empty(B, dtype=torch.float64, device="cuda")
    L = _lib.lib()

    def run():
        R.copy_(dR0)
        t.copy_(dt0)
        _lib.check(L.mba_pose_lm(B, M, ptr(dX), ptr(dU), f, cx, cy, it, 1e-5, 2.0, 2.0, ptr(R), ptr(t),
                                 ptr(cost), 0, None, None, 0.0, None, None, _lib.stream_ptr()),
                   "mba_pose_lm")

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.steps)]
    ms = []
    for s in range(a.steps):
        ev[2 * s].record()
        run()
        ev[2 * s + 1].record()
    torch.cuda.synchronize()
    ms = [ev[2 * s].elapsed_time(ev[2 * s + 1]) for s in range(a.steps)]
    dev_ms = float(np.median(ms))
    dev_cost = cost.cpu().numpy()

    n = min(a.cpu_problems, B)
    t_cpu = time.perf_counter()
    Rc, tc, cc = O.pose_lm(R0[:n], t0[:n], X[:n], uv[:n], f, cx, cy, it)
    t_cpu = time.perf_counter() - t_cpu
    rel = np.abs(dev_cost[:n] - cc) / np.maximum(np.abs(cc), 1e-300)
    line = {
        "metric": "batched pose-only LM (pose_lm, miniba.py:334-389): pose-iterations/s",
        "config": {"batch": B, "correspondences": M, "iters": it, "outliers": 0.1, "data": "synthetic"},
        "device": {"ms_per_call": dev_ms, "pose_iters_per_s": B * it / (dev_ms / 1e3),
                   "correspondence_iters_per_s": B * M * it / (dev_ms / 1e3),
                   "kernel": "mba_pose_lm (warp per pose problem)"},
        "cpu_oracle": {"problems": n, "seconds": t_cpu, "pose_iters_per_s": n * it / t_cpu, "cores": 1,
                       "kind": "port (oracle/miniba_oracle.pose_lm, numpy)"},
        "parity": {"problems": n, "max_rel_cost_diff": float(rel.max()), "rtol": 1e-9,
                   "ok": bool(rel.max() <= 1e-9)},
    }
    line["speedup_vs_cpu_1core"] = line["device"]["pose_iters_per_s"] / line["cpu_oracle"]["pose_iters_per_s"]
    # roofline (SURVEY 8d counts one pass over the correspondences per
    # evaluation: 40 B each -- X 24 + uv 16 -- for the initial cost, and per
    # iteration the linearisation and the trial cost)
    try:
        peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
        kind = "measured"
    except OSError:
        peak, kind = 6650.0, "fallback"
    passes = 1 + 2 * it
    pass_bytes = 40.0 * B * M * passes
    in_bytes = 40.0 * B * M
    flops = B * M * (passes * 60.0 + it * 110.0)   # ~60 flop per residual, ~110 per Jacobian + normal-eq update
    s = dev_ms / 1e3
    line["roofline"] = {"bytes_model": "40 B per correspondence per pass, %d passes" % passes,
                        "achieved_pass_gbs": pass_bytes / s / 1e9, "inputs_once_gbs": in_bytes / s / 1e9,
                        "peak_gbs": peak, "peak_kind": kind, "frac_pass": pass_bytes / s / 1e9 / peak,
                        "fp64_tflops": flops / s / 1e12, "fp64_peak_tflops": 37.22,
                        "inputs_bytes": in_bytes, "larger_than_l2": in_bytes > 126 * 2 ** 20}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
