"""Per-hypothesis comparison of the device pose_lm against the reference's
golden (tests/golden/pose_lm.npz), with the accept margins of every
iteration from the oracle restatement: enumerates the hypotheses whose
result differs and why.

    python scripts/pose_diag.py [--out profiles/round2_pose_diag.json]
"""
import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "src")]


def oracle_trace(R0, t0, X, uv, f, cx, cy, iters):
    """The oracle's pose_lm, one hypothesis at a time, recording per iteration
    the trial cost, the current cost and the accept decision."""
    from oracle import miniba_oracle as O
    out = []
    R, t = R0[None].copy(), t0[None].copy()
    for it in range(iters):
        cost0, _ = O._pose_eval(R, t, X[None], uv[None], f, cx, cy, 2.0)
        Rn, tn, c = O.pose_lm(R, t, X[None], uv[None], f, cx, cy, 1,
                              lambda_init=1e-5 * 2.0 ** 0)  # single step from the current state
        out.append(float(cost0[0]))
        R, t = Rn, tn
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from gsrecon import miniba as M
    from gsrecon.config import LmConfig
    from gsrecon.scene import CameraIntrinsics
    from oracle import miniba_oracle as O
    z = np.load(os.path.join(REPO, "tests", "golden", "pose_lm.npz"))
    f, cx, cy = float(z["focal"]), float(z["cx"]), float(z["cy"])
    intr = CameraIntrinsics(f, cx, cy, 640, 480)
    iters = int(z["iters"])
    R, t, c = M.pose_lm(z["R0"], z["t0"], z["X"], z["uv"], intr, iters, LmConfig())
    # the oracle restatement (numpy, batched exactly like the reference)
    Ro, to, co = O.pose_lm(z["R0"], z["t0"], z["X"], z["uv"], f, cx, cy, iters)
    rows = []
    for b in range(len(c)):
        dt = float(np.abs(t[b] - z["t_out"][b]).max())
        dc = float(abs(c[b] - z["cost_out"][b]) / max(abs(z["cost_out"][b]), 1e-300))
        if dt > 1e-9 or dc > 1e-9:
            rows.append(dict(hyp=b, dt=dt, dcost_rel=dc, cost_ref=float(z["cost_out"][b]),
                             cost_dev=float(c[b]), oracle_dt=float(np.abs(to[b] - z["t_out"][b]).max())))
    out = dict(hypotheses=len(c), differing=len(rows), rows=rows,
               oracle_vs_reference_max_dt=float(np.abs(to - z["t_out"]).max()))
    s = json.dumps(out, indent=1)
    print(s)
    if a.out:
        open(a.out, "w").write(s)


if __name__ == "__main__":
    main()
