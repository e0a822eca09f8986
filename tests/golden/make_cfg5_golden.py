"""Config-5 stress golden from the UNMODIFIED reference (SURVEY.md 8c stress row).

BASELINE config 5 is 32 frames, K = 200k observations, 20 % outliers, 50 LM
iterations. The reference has only the Huber loss (miniba.py:46-54), so this
fixture pins the Huber variant of that workload to the reference itself:
`lm_solve` (miniba.py:223-296) with `CaptureConfig().lm(50)`. It takes about
20-25 min on one CPU core; run once in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cfg5_golden.py

Inputs are the seeded synth workload (paper_2506_05558_b200/synth.py, config 5
shape), stored compactly (fp32-representable values as float32, int32
indices) so the GPU box never needs /root/reference. The evals trace is
recovered by the same non-invasive huber_cost/huber_weights counter as
make_golden.py.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import M, CaptureConfig, run_ref  # noqa: E402  (reference, read-only)
from paper_2506_05558_b200.synth import make_batch  # noqa: E402

SEED = 5
N_CAMS, K, OUTLIERS, ITERS = 32, 200_000, 0.2, 50


def main(out=os.path.join(HERE, "stress_cfg5_huber.npz")):
    b = make_batch(1, n_cams=N_CAMS, K=K, seed=SEED, outlier_frac=OUTLIERS)
    p = b.problem(0)
    cfg = CaptureConfig().lm(ITERS)
    t0 = time.time()
    prob, info, ev = run_ref(p, cfg)
    dt = time.time() - t0
    f32 = lambda a: np.asarray(a, dtype=np.float32)
    assert np.array_equal(f32(p["uv"]).astype(np.float64), p["uv"])
    np.savez_compressed(
        out, seed=SEED, n_cams=N_CAMS, K=K, outlier_frac=OUTLIERS,
        R=f32(p["R"]), t=f32(p["t"]), focal=p["focal"], cx=p["cx"], cy=p["cy"],
        points=f32(p["points"]), cam_idx=p["cam_idx"].astype(np.int32),
        pt_idx=p["pt_idx"].astype(np.int32), uv=f32(p["uv"]), fixed_cams=p["fixed_cams"],
        optimize_focal=True, optimize_points=True, lambda_init=cfg.lambda_init, nu=cfg.nu,
        delta=cfg.huber_delta, max_iters=cfg.max_iters, loss="huber",
        out_costs=info["costs"], out_accepted=info["accepted"], out_lambdas=info["lambdas"],
        out_evals=ev, out_final_rms=info["final_rms"], out_mean_err=info["mean_err"],
        out_R=prob.R, out_t=prob.t, out_focal=prob.focal, out_points=prob.points,
        ref_seconds=dt)
    print(f"cfg5 huber: iters={len(info['accepted'])} acc={int(info['accepted'].sum())} "
          f"evals={ev.tolist()} cost {info['costs'][0]:.6g} -> {info['costs'][-1]:.6g} "
          f"({dt:.0f} s)")


if __name__ == "__main__":
    main()
