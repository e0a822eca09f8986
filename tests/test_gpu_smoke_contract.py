"""The acceptance checks of the reference's pkg/smoke_miniba.py, restated as
tests against this package (same scene recipe, same thresholds), plus the
unchanged script itself when a copy is present in oracle/_ref/ (placed there
by build() from /root/reference; git-ignored, travels to the GPU box)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def _arc_scene(rng):
    from gsrecon.scene import CameraIntrinsics, Pose, project
    W, H = 640, 480
    intr = CameraIntrinsics(520.0, (W - 1) / 2, (H - 1) / 2, W, H)
    poses = []
    for a in np.linspace(-0.35, 0.35, 8):
        c = np.array([2.5 * np.sin(a), 0.15 * np.sin(2 * a), -2.5 * np.cos(a)])
        fwd = -c / np.linalg.norm(c)
        right = np.cross([0.0, -1.0, 0.0], fwd)
        right /= np.linalg.norm(right)
        Rwc = np.stack([right, np.cross(fwd, right), fwd])
        poses.append(Pose.from_matrix(Rwc, -Rwc @ c))
    pts = rng.uniform([-0.8, -0.6, -0.5], [0.8, 0.6, 0.5], (160, 3))
    uv = np.stack([project(intr, p, pts)[0] for p in poses])
    return intr, poses, pts, uv


def test_smoke_contract(cuda_ok):
    from gsrecon.config import CaptureConfig
    from gsrecon.miniba import (BaProblem, EstimationFailure, TriangulationFailure, _assemble,
                                _build_blocks, estimate_pose_ransac, huber_weights, lm_solve,
                                refine_pose, robust_filter, solve_step, triangulate)
    from gsrecon.scene import project, umeyama
    rng = np.random.default_rng(7)
    cfg = CaptureConfig()
    intr, poses, pts, obs_uv = _arc_scene(rng)
    n_cam, n_pts = 8, 160
    cam_idx = np.repeat(np.arange(n_cam), n_pts)
    pt_idx = np.tile(np.arange(n_pts), n_cam)
    uv = obs_uv.reshape(-1, 2)
    d = np.stack([(uv[:n_pts, 0] - intr.cx) / 448.0, (uv[:n_pts, 1] - intr.cy) / 448.0,
                  np.ones(n_pts)], axis=-1)
    prob = BaProblem(R=np.stack([np.eye(3)] * n_cam), t=np.zeros((n_cam, 3)), focal=448.0,
                     cx=intr.cx, cy=intr.cy, points=d.copy(), cam_idx=cam_idx, pt_idx=pt_idx,
                     uv=uv.copy(), fixed_cams=np.arange(n_cam) == 0, optimize_focal=True)
    info = lm_solve(prob, cfg.lm(200))
    assert info["mean_err"] < 1e-6, info["mean_err"]
    ce = np.stack([np.linalg.solve(prob.R[i], -prob.t[i]) for i in range(n_cam)])
    cg = np.stack([p.camera_center() for p in poses])
    s, Rg, tg = umeyama(ce, cg, with_scale=True)
    ape = np.sqrt(np.mean(np.sum(((s * (Rg @ ce.T)).T + tg - cg) ** 2, axis=1)))
    span = np.linalg.norm(cg.max(0) - cg.min(0))
    assert ape / span < 0.01
    assert abs(prob.focal - 520.0) / 520.0 < 0.02
    assert np.all(np.diff(info["costs"]) <= 1e-12)
    # schur vs dense through the stage API
    r, pc, bad = prob.residuals()
    w = huber_weights(np.linalg.norm(r, axis=1), 2.0)
    A, F, B = _build_blocks(prob, pc, bad)
    blocks = _assemble(prob, w, r, A, F, B)
    dc1, dp1 = solve_step(*blocks, 1e-5, "schur")
    dc2, dp2 = solve_step(*blocks, 1e-5, "dense")
    rel = max(np.abs(dc1 - dc2).max() / max(np.abs(dc2).max(), 1e-300),
              np.abs(dp1 - dp2).max() / max(np.abs(dp2).max(), 1e-300))
    assert rel < 1e-8, rel
    # noisy arc
    prob2 = BaProblem(R=np.stack([np.eye(3)] * n_cam), t=np.zeros((n_cam, 3)), focal=448.0,
                      cx=intr.cx, cy=intr.cy, points=d.copy(), cam_idx=cam_idx, pt_idx=pt_idx,
                      uv=uv + rng.normal(0, 0.5, uv.shape), fixed_cams=np.arange(n_cam) == 0,
                      optimize_focal=True)
    lm_solve(prob2, cfg.lm(200))
    ce2 = np.stack([np.linalg.solve(prob2.R[i], -prob2.t[i]) for i in range(n_cam)])
    s2, Rg2, tg2 = umeyama(ce2, cg, with_scale=True)
    ape2 = np.sqrt(np.mean(np.sum(((s2 * (Rg2 @ ce2.T)).T + tg2 - cg) ** 2, axis=1)))
    assert ape2 / span < 0.01 and abs(prob2.focal - 520.0) / 520.0 < 0.02
    assert robust_filter(np.array([1.0, 1.0, 1.0, 100.0])).tolist() == [True, True, True, False]
    assert robust_filter(np.array([1.0, 2.0, 3.0, 4.0, 5.0])).all()
    # RANSAC + refine
    uv_q, _ = project(intr, poses[4], pts)
    uv_n = uv_q + rng.normal(0, 0.3, uv_q.shape)
    out = rng.choice(n_pts, 30, replace=False)
    uv_n[out] += rng.uniform(30, 120, (30, 2)) * rng.choice([-1, 1], (30, 2))
    pose_est, inl = estimate_pose_ransac(pts, uv_n, intr, poses[3].copy(), cfg, np.random.default_rng(3))
    assert inl.sum() >= n_pts - 35
    ref = refine_pose(pose_est, pts[inl], uv_n[inl], intr, cfg)
    assert np.linalg.norm(ref.camera_center() - poses[4].camera_center()) < 0.01
    with pytest.raises(EstimationFailure):
        estimate_pose_ransac(pts, uv_q + rng.uniform(50, 300, uv_q.shape), intr, poses[3].copy(), cfg,
                             np.random.default_rng(0))
    Xg = np.array([0.2, -0.1, 0.3])
    px = np.stack([project(intr, p, Xg[None])[0][0] for p in poses[:4]])
    assert np.linalg.norm(triangulate(poses[:4], px, intr) - Xg) < 1e-9
    with pytest.raises(TriangulationFailure):
        triangulate([poses[0], poses[0]], np.stack([px[0], px[0]]), intr)


SMOKE = os.path.join(REPO, "oracle", "_ref", "smoke_miniba.py")


@pytest.mark.skipif(not os.path.exists(SMOKE), reason="no copy of the reference smoke script")
def test_reference_smoke_script_runs_unchanged(cuda_ok):
    """Runs pkg/smoke_miniba.py byte-for-byte from the repo root: its
    sys.path.insert(0, "src") picks up this package's src/gsrecon."""
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    code = ("import runpy, sys; sys.argv = [%r]; runpy.run_path(%r, run_name='__main__'); "
            "import gsrecon.miniba as m; print('GSRECON_FROM', m.__file__)" % (SMOKE, SMOKE))
    r = subprocess.run([sys.executable, "-c", code], cwd=REPO, capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL MINIBA SMOKE CHECKS PASSED" in r.stdout
    # it must have exercised this package, not the reference
    assert f"GSRECON_FROM {os.path.join(REPO, 'src', 'gsrecon', 'miniba.py')}" in r.stdout


@pytest.mark.gpu
def test_bench_two_ranks_on_one_gpu(tmp_path):
    """The N-rank bench flow (torchrun, contiguous shards, max-over-ranks
    timing, final gather) end to end with 2 ranks; on this one-GPU box both
    ranks share GPU 0 and the collectives go over gloo (MBA_BENCH_ONE_GPU)."""
    import json
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MBA_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
           "--problems", "512", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=repo, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]   # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["n_problems"] == 512
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] >= 1
    os.makedirs(os.path.join(repo, "gpurun_out"), exist_ok=True)
    with open(os.path.join(repo, "gpurun_out", "bench_two_ranks.json"), "w") as fh:
        fh.write(lines[0] + "\n")
