"""Acceptance fixtures produced by the UNMODIFIED reference.

Run once in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_acceptance_golden.py

* bootstrap20.npz -- criterion 1: 20 seeded synthetic 8-camera / 500-point
  problems, 0.5 px noise (gsrecon.synthetic.bootstrap_problem): the features
  (keypoints + ground-truth point ids, matched exactly), intrinsics, ground
  truth camera centres / focal / span, and the reference bootstrap's output
  (miniba.py:729-854: R, t, focal, n_tracks, rescued, mean_err, wall time).
* ransac20.npz -- criterion 3: 20 seeded PnP problems with 30 % outliers
  (gsrecon.synthetic.pnp_problem), the reference estimate_pose_ransac's pose
  and inlier mask (miniba.py:392-439) for rng seed 100 + seed, and the
  planted inlier mask.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import gsrecon.miniba as M  # noqa: E402  (the reference, read-only)
from gsrecon import synthetic as S  # noqa: E402
from gsrecon.config import CaptureConfig  # noqa: E402

assert M.__file__.startswith("/root/reference"), M.__file__


def bootstrap20():
    cfg = CaptureConfig()
    cols = {k: [] for k in ("kp", "ids", "counts", "gt_centers", "out_R", "out_t")}
    scal = {k: [] for k in ("focal", "cx", "cy", "width", "height", "gt_focal", "span", "out_focal",
                            "out_n_tracks", "out_rescued", "out_mean_err", "ref_seconds")}
    for seed in range(20):
        bp = S.bootstrap_problem(seed, n_cams=8, n_points=500, noise_px=0.5)
        intr = bp["intr"]
        t0 = time.perf_counter()
        poses, intr_out, table, info = M.bootstrap(bp["features"], intr, cfg, matcher=bp["matcher"])
        dt = time.perf_counter() - t0
        for kp, ids in bp["features"]:
            cols["kp"].append(np.asarray(kp, np.float64))
            cols["ids"].append(np.asarray(ids, np.int64))
            cols["counts"].append(len(ids))
        cols["gt_centers"].append(np.stack([p.camera_center() for p in bp["gt_poses"]]))
        cols["out_R"].append(np.stack([p.R for p in poses]))
        cols["out_t"].append(np.stack([p.translation for p in poses]))
        for k, v in (("focal", intr.focal), ("cx", intr.cx), ("cy", intr.cy), ("width", intr.width),
                     ("height", intr.height), ("gt_focal", bp["gt_focal"]), ("span", bp["span"]),
                     ("out_focal", intr_out.focal), ("out_n_tracks", info["n_tracks"]),
                     ("out_rescued", info["rescued"]), ("out_mean_err", info["mean_err"]),
                     ("ref_seconds", dt)):
            scal[k].append(v)
        print(f"bootstrap seed {seed}: focal {intr_out.focal:.3f} (gt {bp['gt_focal']}) "
              f"tracks {info['n_tracks']} rescued {info['rescued']} {dt:.2f} s")
    np.savez_compressed(os.path.join(HERE, "bootstrap20.npz"),
                        kp=np.concatenate(cols["kp"]), ids=np.concatenate(cols["ids"]),
                        counts=np.array(cols["counts"]), gt_centers=np.stack(cols["gt_centers"]),
                        out_R=np.stack(cols["out_R"]), out_t=np.stack(cols["out_t"]),
                        **{k: np.array(v) for k, v in scal.items()})


def ransac20():
    cfg = CaptureConfig()
    out = {k: [] for k in ("points", "pixels", "inlier_gt", "init_R", "init_t", "gt_R", "gt_t",
                           "ref_R", "ref_t", "ref_inl")}
    intr = None
    for seed in range(20):
        d = S.pnp_problem(seed, n=160, outlier_frac=0.3)
        intr = d["intr"]
        pose, inl = M.estimate_pose_ransac(d["points"], d["pixels"], intr, d["init_pose"], cfg,
                                           np.random.default_rng(100 + seed))
        for k, v in (("points", d["points"]), ("pixels", d["pixels"]), ("inlier_gt", d["inlier_mask"]),
                     ("init_R", d["init_pose"].R), ("init_t", d["init_pose"].translation),
                     ("gt_R", d["gt_pose"].R), ("gt_t", d["gt_pose"].translation), ("ref_R", pose.R),
                     ("ref_t", pose.translation), ("ref_inl", inl)):
            out[k].append(np.asarray(v))
        rec = (inl & d["inlier_mask"]).sum() / d["inlier_mask"].sum()
        print(f"ransac seed {seed}: recall {rec:.3f}")
    np.savez_compressed(os.path.join(HERE, "ransac20.npz"), focal=intr.focal, cx=intr.cx, cy=intr.cy,
                        width=intr.width, height=intr.height, **{k: np.stack(v) for k, v in out.items()})


if __name__ == "__main__":
    bootstrap20()
    ransac20()
