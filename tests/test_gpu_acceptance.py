"""The reference spec's acceptance criteria for the mini-BA path
(/root/reference/SPEC.md:722-724), on the device, against fixtures produced
by the unmodified reference (tests/golden/make_acceptance_golden.py):

1. bootstrap oracle -- 20 seeded 8-camera / 500-point problems, 0.5 px noise:
   focal within 2 % of truth, translation APE < 1 % of the span after
   similarity alignment, < 10 s per run; and the reference's own output
   (focal, poses, tracks, rescue decision) reproduced;
2. LM contract -- Jacobians match central finite differences within 1e-5
   relative at 100 random configurations (stage kernels, miniba.py:101-132);
3. RANSAC robustness -- 30 % outliers over 20 seeds: recovered inlier sets
   contain >= 95 % of the true inliers, identical to the reference's sets.
"""
import time

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _windows():
    z = np.load(f"{GOLDEN}/bootstrap20.npz")
    feats, o = [], 0
    counts = z["counts"].reshape(20, -1)
    for s in range(20):
        w = []
        for c in counts[s]:
            w.append((z["kp"][o:o + c], z["ids"][o:o + c]))
            o += c
        feats.append(w)
    return z, feats


def _exact_matcher(fa, fb):
    """The synthetic problems' descriptors are ground-truth point ids."""
    ida, idb = np.asarray(fa[1]), np.asarray(fb[1])
    common, ia, ib = np.intersect1d(ida, idb, assume_unique=True, return_indices=True)
    order = np.argsort(ia, kind="stable")
    return ia[order].astype(np.int64), ib[order].astype(np.int64), np.zeros(len(ia))


def _ape_over_span(poses, gt_centers, span):
    from gsrecon.scene import umeyama
    est = np.stack([-p.R.T @ p.translation for p in poses])
    s, Rg, tg = umeyama(est, gt_centers, with_scale=True)
    aligned = s * est @ Rg.T + tg
    return float(np.sqrt(np.mean(np.sum((aligned - gt_centers) ** 2, axis=1)))) / span


def test_bootstrap_oracle_20_seeds(cuda_ok):
    from gsrecon import miniba as M
    from gsrecon.config import CaptureConfig
    from gsrecon.scene import CameraIntrinsics
    z, wins = _windows()
    cfg = CaptureConfig()
    for s in range(20):
        intr = CameraIntrinsics(float(z["focal"][s]), float(z["cx"][s]), float(z["cy"][s]),
                                int(z["width"][s]), int(z["height"][s]))
        t0 = time.perf_counter()
        poses, intr_out, table, info = M.bootstrap(wins[s], intr, cfg, matcher=_exact_matcher)
        dt = time.perf_counter() - t0
        assert dt < 10.0
        # SPEC.md:722 against ground truth
        assert abs(intr_out.focal - z["gt_focal"][s]) / z["gt_focal"][s] < 0.02, s
        assert _ape_over_span(poses, z["gt_centers"][s], float(z["span"][s])) < 0.01, s
        # and the reference's own result on the same input
        assert bool(info["rescued"]) == bool(z["out_rescued"][s]), s
        assert info["n_tracks"] == int(z["out_n_tracks"][s]), s
        np.testing.assert_allclose(intr_out.focal, z["out_focal"][s], rtol=1e-6, err_msg=str(s))
        for p, R, t in zip(poses, z["out_R"][s], z["out_t"][s]):
            np.testing.assert_allclose(p.R, R, atol=1e-6, err_msg=str(s))
            np.testing.assert_allclose(p.translation, t, atol=1e-6, err_msg=str(s))
        np.testing.assert_allclose(info["mean_err"], z["out_mean_err"][s], rtol=1e-5, err_msg=str(s))


def test_bootstrap_batch_of_20_windows_in_one_schedule(cuda_ok):
    """All 20 windows through ONE device schedule (plus one for the rescued
    window): same answers as one window at a time."""
    from gsrecon import miniba as M
    from gsrecon.config import CaptureConfig
    from gsrecon.scene import CameraIntrinsics
    z, wins = _windows()
    intrs = [CameraIntrinsics(float(z["focal"][s]), float(z["cx"][s]), float(z["cy"][s]),
                              int(z["width"][s]), int(z["height"][s])) for s in range(20)]
    res = M.bootstrap_batch(wins, intrs, CaptureConfig(), matcher=_exact_matcher)
    for s, r in enumerate(res):
        assert not isinstance(r, Exception), (s, r)
        poses, intr_out, table, info = r
        np.testing.assert_allclose(intr_out.focal, z["out_focal"][s], rtol=1e-6)
        assert bool(info["rescued"]) == bool(z["out_rescued"][s])
        assert len(table) == int(z["out_n_tracks"][s])


def test_ransac_30pct_outliers_20_seeds(cuda_ok):
    from gsrecon import miniba as M
    from gsrecon.config import CaptureConfig
    from gsrecon.scene import CameraIntrinsics, Pose
    z = np.load(f"{GOLDEN}/ransac20.npz")
    intr = CameraIntrinsics(float(z["focal"]), float(z["cx"]), float(z["cy"]), int(z["width"]),
                            int(z["height"]))
    for s in range(20):
        init = Pose.from_matrix(z["init_R"][s], z["init_t"][s])
        pose, inl = M.estimate_pose_ransac(z["points"][s], z["pixels"][s], intr, init, CaptureConfig(),
                                           np.random.default_rng(100 + s))
        gt = z["inlier_gt"][s]
        assert (inl & gt).sum() >= 0.95 * gt.sum(), s
        np.testing.assert_array_equal(inl, z["ref_inl"][s], err_msg=str(s))
        np.testing.assert_allclose(pose.R, z["ref_R"][s], atol=1e-9)
        np.testing.assert_allclose(pose.translation, z["ref_t"][s], atol=1e-9)


def test_jacobians_match_finite_differences_100_configs(cuda_ok):
    """_build_blocks (device stage kernel) against central differences of
    residuals (device stage kernel) at 100 random configurations: camera
    (left-perturbation rotation, translation), focal and point blocks within
    1e-5 relative."""
    from gsrecon import miniba as M
    from gsrecon.scene import exp_so3
    rng = np.random.default_rng(2024)
    worst = 0.0
    for cfg_i in range(100):
        n, P = 3, 5
        R = np.stack([exp_so3(0.3 * rng.standard_normal(3)) for _ in range(n)])
        t = 0.2 * rng.standard_normal((n, 3)) + np.array([0.0, 0.0, 4.0])
        X = 0.5 * rng.standard_normal((P, 3))
        cam = np.repeat(np.arange(n), P)
        pt = np.tile(np.arange(P), n)
        f = float(rng.uniform(300, 800))
        uv = rng.uniform(0, 640, (len(cam), 2))
        prob = M.BaProblem(R=R, t=t, focal=f, cx=320.0, cy=240.0, points=X, cam_idx=cam, pt_idx=pt,
                           uv=uv, fixed_cams=np.zeros(n, bool))
        r0, pc, bad = prob.residuals()
        assert not bad.any()
        A, F, B = M._build_blocks(prob, pc, bad)
        h = 1e-6

        def res_with(**kw):
            q = M.BaProblem(R=kw.get("R", R), t=kw.get("t", t), focal=kw.get("focal", f), cx=320.0, cy=240.0,
                            points=kw.get("points", X), cam_idx=cam, pt_idx=pt, uv=uv,
                            fixed_cams=np.zeros(n, bool))
            return q.residuals()[0]

        def rel(num, ana):
            return np.abs(num - ana).max() / max(np.abs(ana).max(), 1e-12)
        errs = []
        for c in range(n):
            rows = cam == c
            for a in range(3):
                w = np.zeros(3)
                w[a] = h
                Rp, Rm = R.copy(), R.copy()
                Rp[c] = exp_so3(w) @ R[c]
                Rm[c] = exp_so3(-w) @ R[c]
                num = (res_with(R=Rp) - res_with(R=Rm))[rows] / (2 * h)
                errs.append(rel(num, A[rows, :, a]))
                tp, tm = t.copy(), t.copy()
                tp[c, a] += h
                tm[c, a] -= h
                num = (res_with(t=tp) - res_with(t=tm))[rows] / (2 * h)
                errs.append(rel(num, A[rows, :, 3 + a]))
        num = (res_with(focal=f + h * f) - res_with(focal=f - h * f)) / (2 * h * f)
        errs.append(rel(num, F))
        for j in range(P):
            rows = pt == j
            for a in range(3):
                Xp, Xm = X.copy(), X.copy()
                Xp[j, a] += h
                Xm[j, a] -= h
                num = (res_with(points=Xp) - res_with(points=Xm))[rows] / (2 * h)
                errs.append(rel(num, B[rows, :, a]))
        worst = max(worst, max(errs))
        assert max(errs) < 1e-5, (cfg_i, max(errs))
    print("worst relative FD error", worst)
