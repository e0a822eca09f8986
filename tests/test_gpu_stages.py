"""Device stage kernels behind the reference's internal API, against the
reference's own outputs (tests/golden/stages_smoke.npz, pose_lm.npz)."""
import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _prob(M, z):
    return M.BaProblem(R=z["R"].copy(), t=z["t"].copy(), focal=float(z["focal"]), cx=float(z["cx"]),
                       cy=float(z["cy"]), points=z["points"].copy(), cam_idx=z["cam_idx"].copy(),
                       pt_idx=z["pt_idx"].copy(), uv=z["uv"].copy(), fixed_cams=z["fixed_cams"].copy(),
                       optimize_focal=True)


def test_stage_kernels_match_reference(cuda_ok):
    from gsrecon import miniba as M
    z = np.load(f"{GOLDEN}/stages_smoke.npz")
    prob = _prob(M, z)
    r, pc, bad = prob.residuals()
    np.testing.assert_allclose(r, z["r"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(pc, z["p_cam"], rtol=1e-13, atol=1e-13)
    assert np.array_equal(bad, z["bad"])
    e = np.linalg.norm(r, axis=1)
    w = M.huber_weights(e, 2.0)
    np.testing.assert_allclose(w, z["w"], rtol=1e-12)
    np.testing.assert_allclose(M.huber_cost(e, 2.0), float(z["huber_cost"]), rtol=1e-12)
    A, F, B = M._build_blocks(prob, pc, bad)
    np.testing.assert_allclose(A, z["A"], rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(F, z["F"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(B, z["B"], rtol=1e-12, atol=1e-9)
    blocks = M._assemble(prob, z["w"], z["r"], z["A"], z["F"], z["B"])
    for got, name in zip(blocks, ("U", "g_c", "V", "g_p", "Wf")):
        np.testing.assert_allclose(got, z[name], rtol=1e-11, atol=1e-7, err_msg=name)
    gold = [z[k] for k in ("U", "g_c", "V", "g_p", "Wf")]
    lam = float(z["lam"])
    dc1, dp1 = M.solve_step(*gold, lam, "schur")
    dc2, dp2 = M.solve_step(*gold, lam, "dense")
    np.testing.assert_allclose(dc1, z["dc_schur"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(dp1, z["dp_schur"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(dc2, z["dc_dense"], rtol=1e-8, atol=1e-12)
    rel = max(np.abs(dc1 - dc2).max() / np.abs(dc2).max(), np.abs(dp1 - dp2).max() / np.abs(dp2).max())
    assert rel < 1e-8  # smoke_miniba.py:96


def test_solve_step_not_pd_raises(cuda_ok):
    from gsrecon import miniba as M
    C, P = 7, 2
    U = -np.eye(C)
    with pytest.raises(np.linalg.LinAlgError):
        M.solve_step(U, np.zeros(C), np.tile(np.eye(3), (P, 1, 1)), np.zeros((P, 3)),
                     np.zeros((P, C, 3)), 1e-5, "schur")


def test_pose_lm_matches_reference(cuda_ok):
    from gsrecon import miniba as M
    from gsrecon.config import LmConfig
    from gsrecon.scene import CameraIntrinsics
    z = np.load(f"{GOLDEN}/pose_lm.npz")
    intr = CameraIntrinsics(float(z["focal"]), float(z["cx"]), float(z["cy"]), 640, 480)
    R, t, c = M.pose_lm(z["R0"], z["t0"], z["X"], z["uv"], intr, int(z["iters"]), LmConfig())
    # Every hypothesis: same accept decisions (no accept margin in this batch is
    # below 2.8e-4 relative), final cost to 1e-12. Poses agree to 1e-9 except
    # the two hypotheses enumerated below, whose last accepted step solves a
    # normal matrix with cond(H) = 4.1e6 (hyp 3) / 1.7e7 (hyp 140): Huber
    # outliers leave a flat valley, the fp64 step along it depends on the
    # summation order, and t lands 1.3e-6 / 2.0e-5 apart at costs equal to
    # 1e-14 (scripts/pose_diag.py, profiles/round2_pose_diag.json).
    ILL_CONDITIONED = {3: 1e-5, 140: 1e-4}
    np.testing.assert_allclose(c, z["cost_out"], rtol=1e-12)
    dt = np.abs(t - z["t_out"]).max(axis=1)
    for b in range(len(dt)):
        assert dt[b] <= ILL_CONDITIONED.get(b, 1e-9), (b, dt[b])
    R, t, c = M.pose_lm(z["Rf0"], z["tf0"], z["Xf"], z["uvf"], intr, int(z["iters_f"]), LmConfig())
    np.testing.assert_allclose(c, z["costf_out"], rtol=1e-9)
    np.testing.assert_allclose(t, z["tf_out"], rtol=1e-7, atol=1e-10)


def test_dense_lm_solve_path(cuda_ok):
    """lm_solve(method='dense') (the verification path) against the golden."""
    from gsrecon import miniba as M
    from gsrecon.config import LmConfig
    z = np.load(f"{GOLDEN}/lm_cfg1_5cam.npz")
    prob = M.BaProblem(R=z["R"].copy(), t=z["t"].copy(), focal=float(z["focal"]), cx=float(z["cx"]),
                       cy=float(z["cy"]), points=z["points"].copy(), cam_idx=z["cam_idx"],
                       pt_idx=z["pt_idx"], uv=z["uv"], fixed_cams=z["fixed_cams"])
    info = M.lm_solve(prob, LmConfig(max_iters=int(z["max_iters"])), method="dense")
    np.testing.assert_allclose(info["costs"][-1], z["out_costs"][-1], rtol=1e-8)
    assert info["accepted"][:5].tolist() == z["out_accepted"][:5].tolist()


def _exact_matcher(feat_a, feat_b):
    """Fake matcher of the reference's oracle (synthetic.py:313-327): the
    'descriptors' are ground-truth point ids."""
    pos_b = {int(v): j for j, v in enumerate(feat_b[1])}
    ia, ib = [], []
    for i, v in enumerate(feat_a[1]):
        j = pos_b.get(int(v))
        if j is not None:
            ia.append(i)
            ib.append(j)
    return np.array(ia, dtype=np.int64), np.array(ib, dtype=np.int64), np.zeros(len(ia))


@pytest.mark.parametrize("seed", [0, 1])
def test_bootstrap_matches_reference(seed, cuda_ok):
    """Bootstrap (miniba.py:729-854: tracks, 100 + 100 LM iterations with the
    median + 4 MAD filter between, gauge normalisation) on the reference's own
    bootstrap oracle problem, against the reference's output."""
    from gsrecon import miniba as M
    from gsrecon.config import CaptureConfig
    from gsrecon.scene import CameraIntrinsics
    z = np.load(f"{GOLDEN}/bootstrap_seed{seed}.npz")
    feats, o = [], 0
    for c in z["counts"]:
        feats.append((z["keypoints"][o:o + c], z["ids"][o:o + c]))
        o += c
    intr = CameraIntrinsics(float(z["focal"]), float(z["cx"]), float(z["cy"]), int(z["width"]),
                            int(z["height"]))
    poses, intr_out, table, info = M.bootstrap(feats, intr, CaptureConfig(), matcher=_exact_matcher)
    assert info["n_tracks"] == int(z["out_n_tracks"])
    assert bool(info["rescued"]) == bool(z["out_rescued"])
    np.testing.assert_allclose(intr_out.focal, float(z["out_focal"]), rtol=1e-6)
    for p, R, t in zip(poses, z["out_R"], z["out_t"]):
        np.testing.assert_allclose(p.R, R, atol=1e-6)
        np.testing.assert_allclose(p.translation, t, atol=1e-6)
    np.testing.assert_allclose(info["mean_err"], float(z["out_mean_err"]), rtol=1e-6)


def test_triangulate_batch_matches_reference(cuda_ok):
    """mba_triangulate (one thread per track) against the unmodified
    reference's triangulate on 600 tracks of 2..8 views, including tiny
    baselines, outliers and points behind the cameras: identical
    success/failure classification, points to 1e-10."""
    from gsrecon import miniba as M
    from gsrecon.scene import CameraIntrinsics
    z = np.load(f"{GOLDEN}/triangulate.npz")
    intr = CameraIntrinsics(float(z["focal"]), float(z["cx"]), float(z["cy"]), 640, 480)
    X, st, err = M.triangulate_batch(z["R"], z["t"], z["cam"], z["uv"], z["obs_off"], intr)
    np.testing.assert_array_equal(st, z["status"])
    ok = st == 0
    np.testing.assert_allclose(X[ok], z["X"][ok], rtol=0, atol=1e-10)
    assert np.all(np.isnan(X[~ok]))
    assert np.all(err[ok] <= 8.0)


def test_match_batch_matches_reference(cuda_ok):
    """mba_match_pairs for all 28 frame pairs of 8 frames against the
    unmodified reference's frontend.match on the same descriptors (planted
    correspondences with flipped bits, distractors, exact duplicates that
    exercise the ratio test): identical indices and scores."""
    from gsrecon import miniba as M
    z = np.load(f"{GOLDEN}/match.npz")
    off = z["desc_off"]
    descs = [z["desc"][off[f]:off[f + 1]] for f in range(len(off) - 1)]
    res = M.match_batch(descs, z["pairs"])
    po = z["pair_off"]
    assert sum(len(r[0]) for r in res) == po[-1]
    for p, (ia, ib, sc) in enumerate(res):
        np.testing.assert_array_equal(ia, z["idx_a"][po[p]:po[p + 1]])
        np.testing.assert_array_equal(ib, z["idx_b"][po[p]:po[p + 1]])
        np.testing.assert_array_equal(sc, z["score"][po[p]:po[p + 1]])


def test_build_tracks_device_matches_reference(cuda_ok):
    """build_tracks_device (all 28 frame pairs matched in one device call, host
    flow filter + union-find) against the reference's build_tracks(features,
    default_matcher) on an 8-frame synthetic window: identical tracks."""
    from gsrecon._bootstrap import build_tracks_device
    z = np.load(f"{GOLDEN}/tracks.npz")
    off = z["off"]
    feats = [(z["kp"][off[f]:off[f + 1]], z["desc"][off[f]:off[f + 1]]) for f in range(len(off) - 1)]
    tracks = build_tracks_device(feats)
    flat = np.array([(ti, fr, k, x, y) for ti, tr in enumerate(tracks) for (fr, k, x, y) in tr])
    np.testing.assert_array_equal(flat, z["tracks"])


def test_triangulate_batch_rejects_bad_camera_index(cuda_ok):
    from gsrecon import miniba as M
    from gsrecon.scene import CameraIntrinsics
    z = np.load(f"{GOLDEN}/triangulate.npz")
    intr = CameraIntrinsics(float(z["focal"]), float(z["cx"]), float(z["cy"]), 640, 480)
    cam = z["cam"].copy()
    cam[3] = len(z["R"])
    with pytest.raises(IndexError):
        M.triangulate_batch(z["R"], z["t"], cam, z["uv"], z["obs_off"], intr)
