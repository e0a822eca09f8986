"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `gsrecon` read-only from /root/reference/pkg/src, builds the
fixture problems, runs the reference `lm_solve` / `pose_lm` / stage functions
on them and writes inputs + outputs to tests/golden/*.npz. The per-iteration
trial-count trace `evals` is recovered non-invasively by wrapping the module's
`huber_cost` / `huber_weights` globals and counting cost calls between weight
calls. Fault injection wraps `solve_step` to raise LinAlgError at
chosen iterations (exercises miniba.py:247-251, which never fires naturally).

Nothing here is imported by the product or by the GPU box at run time; the
.npz files are the committed artefacts.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, REPO)

import gsrecon.miniba as M  # noqa: E402  (the reference, read-only)
from gsrecon.config import CaptureConfig, LmConfig  # noqa: E402
from gsrecon.scene import CameraIntrinsics, Pose, project  # noqa: E402
from gsrecon import synthetic as S  # noqa: E402

from paper_2506_05558_b200.synth import make_batch  # noqa: E402

assert M.__file__.startswith("/root/reference"), M.__file__

PROB_KEYS = ("R", "t", "points", "cam_idx", "pt_idx", "uv", "fixed_cams")


class _Counter:
    def __init__(self):
        self.evals = []
        self.cur = None
        self._cost = M.huber_cost
        self._w = M.huber_weights

    def install(self):
        def cost(e, d):
            if self.cur is not None:
                self.cur += 1
            return self._cost(e, d)

        def weights(e, d):
            if self.cur is not None:
                self.evals.append(self.cur)
            self.cur = 0
            return self._w(e, d)
        M.huber_cost = cost
        M.huber_weights = weights

    def uninstall(self):
        M.huber_cost = self._cost
        M.huber_weights = self._w

    def finish(self, n_iters):
        if self.cur is not None:
            self.evals.append(self.cur)
        ev = self.evals[:n_iters]
        return np.array(ev, dtype=np.int32)


def run_ref(p, cfg, fail_at=()):
    prob = M.BaProblem(R=p["R"].copy(), t=p["t"].copy(), focal=float(p["focal"]),
                       cx=float(p["cx"]), cy=float(p["cy"]), points=p["points"].copy(),
                       cam_idx=p["cam_idx"].copy(), pt_idx=p["pt_idx"].copy(),
                       uv=p["uv"].copy(), fixed_cams=p["fixed_cams"].copy(),
                       optimize_focal=bool(p["optimize_focal"]),
                       optimize_points=bool(p.get("optimize_points", True)))
    cnt = _Counter()
    cnt.install()
    orig_solve = M.solve_step
    calls = {"n": 0}
    if fail_at:
        def failing(*a, **k):
            i = calls["n"]
            calls["n"] += 1
            if i in fail_at:
                raise np.linalg.LinAlgError("injected")
            return orig_solve(*a, **k)
        M.solve_step = failing
    try:
        info = M.lm_solve(prob, cfg)
    finally:
        cnt.uninstall()
        M.solve_step = orig_solve
    n_it = len(info["accepted"])
    ev = cnt.finish(n_it)
    # a Cholesky failure skips the trial loop: huber_cost is not called
    return prob, info, ev


def save_case(name, p, cfg, prob, info, ev, fail_at=(), loss="huber"):
    out = {k: np.asarray(p[k]) for k in PROB_KEYS}
    out.update(focal=p["focal"], cx=p["cx"], cy=p["cy"],
               optimize_focal=bool(p["optimize_focal"]),
               optimize_points=bool(p.get("optimize_points", True)),
               lambda_init=cfg.lambda_init, nu=cfg.nu, delta=cfg.huber_delta,
               max_iters=cfg.max_iters, loss=loss, fail_at=np.array(sorted(fail_at), dtype=np.int64),
               out_costs=info["costs"], out_accepted=info["accepted"],
               out_lambdas=info["lambdas"], out_evals=ev,
               out_final_rms=info["final_rms"], out_mean_err=info["mean_err"],
               out_R=prob.R, out_t=prob.t, out_focal=prob.focal, out_points=prob.points)
    np.savez_compressed(os.path.join(HERE, f"lm_{name}.npz"), **out)
    print(f"{name:24s} K={len(p['uv']):6d} iters={len(info['accepted']):3d} "
          f"acc={int(info['accepted'].sum()):3d} evals={ev.tolist()[:12]} cost={info['costs'][-1]:.6g}")


def smoke_scene(noisy):
    """The smoke_miniba.py:12-60 scene, built with the reference's own helpers."""
    rng = np.random.default_rng(7)
    W, H = 640, 480
    intr = CameraIntrinsics(520.0, (W - 1) / 2, (H - 1) / 2, W, H)
    n_cam, n_pts = 8, 160
    poses = []
    for a in np.linspace(-0.35, 0.35, n_cam):
        c = np.array([2.5 * np.sin(a), 0.15 * np.sin(2 * a), -2.5 * np.cos(a)])
        fwd = -c / np.linalg.norm(c)
        right = np.cross(np.array([0.0, -1.0, 0.0]), fwd)
        right /= np.linalg.norm(right)
        Rwc = np.stack([right, np.cross(fwd, right), fwd])
        poses.append(Pose.from_matrix(Rwc, -Rwc @ c))
    pts = rng.uniform([-0.8, -0.6, -0.5], [0.8, 0.6, 0.5], (n_pts, 3))
    uv = np.concatenate([project(intr, p, pts)[0] for p in poses])
    d = np.stack([(uv[:n_pts, 0] - intr.cx) / (0.7 * W), (uv[:n_pts, 1] - intr.cy) / (0.7 * W),
                  np.ones(n_pts)], axis=-1)
    if noisy:
        # smoke draws the noise after consuming the noise-free solve's rng state;
        # we draw from a fresh stream (the exact values do not matter here).
        uv = uv + np.random.default_rng(77).normal(0, 0.5, uv.shape)
    return dict(R=np.stack([np.eye(3)] * n_cam), t=np.zeros((n_cam, 3)), focal=0.7 * W,
                cx=intr.cx, cy=intr.cy, points=d, cam_idx=np.repeat(np.arange(n_cam), n_pts),
                pt_idx=np.tile(np.arange(n_pts), n_cam), uv=uv,
                fixed_cams=np.arange(n_cam) == 0, optimize_focal=True, optimize_points=True)


def perturbed_ba(seed, n_cams=8, n_points=160, noise=0.5):
    """synthetic.ba_problem (all-visible) with SPEC.md:207 style perturbation."""
    d = S.ba_problem(seed, n_cams=n_cams, n_points=n_points, noise_px=noise)
    rng = np.random.default_rng(1000 + seed)
    R = np.stack([p.R for p in d["gt_poses"]])
    t = np.stack([p.translation for p in d["gt_poses"]])
    for c in range(1, n_cams):
        R[c] = M.exp_so3(np.deg2rad(1.0) * rng.standard_normal(3)) @ R[c]
        t[c] = t[c] + 0.01 * np.linalg.norm(t[c]) * rng.standard_normal(3)
    return dict(R=R, t=t, focal=d["gt_focal"] * 1.02, cx=d["intr"].cx, cy=d["intr"].cy,
                points=d["gt_points"] + 0.01 * rng.standard_normal(d["gt_points"].shape),
                cam_idx=d["cam_idx"], pt_idx=d["pt_idx"], uv=d["uv"],
                fixed_cams=np.arange(n_cams) == 0, optimize_focal=True, optimize_points=True)


def main():
    cfg = CaptureConfig()
    cases = []
    cases.append(("smoke_noisefree", smoke_scene(False), cfg.lm(200), ()))
    cases.append(("smoke_noisy", smoke_scene(True), cfg.lm(200), ()))
    b = make_batch(6, n_cams=8, K=2000, seed=0)
    for i in (0, 3, 5):
        cases.append((f"cfg4_seed0_p{i}", b.problem(i), cfg.lm(200), ()))
    b1 = make_batch(1, n_cams=5, K=1000, seed=1)
    cases.append(("cfg1_5cam", b1.problem(0), cfg.lm(20), ()))
    cases.append(("ba_all_visible", perturbed_ba(3), cfg.lm(200), ()))
    # no focal, two fixed cameras, camera-major order
    p = perturbed_ba(4, n_points=120)
    p["optimize_focal"] = False
    p["fixed_cams"] = np.isin(np.arange(8), [0, 5])
    cases.append(("nofocal_2fixed", p, cfg.lm(200), ()))
    # points held fixed (optimize_points=False): pose+focal only
    p = perturbed_ba(5, n_points=100)
    p["optimize_points"] = False
    cases.append(("fixed_points", p, cfg.lm(50), ()))
    # behind-camera observations: push some points behind camera 2
    p = perturbed_ba(6, n_points=120)
    Rc, tc = p["R"][2], p["t"][2]
    sel = np.nonzero(p["cam_idx"] == 2)[0][:6]
    for k in sel:
        j = p["pt_idx"][k]
        pc = Rc @ p["points"][j] + tc
        pc[2] = -abs(pc[2])
        p["points"][j] = Rc.T @ (pc - tc)
    cases.append(("behind_camera", p, cfg.lm(60), ()))
    # outliers (Huber regime) -- pnp-style uniform replacement on a tracked problem
    b2 = make_batch(1, n_cams=8, K=2000, seed=7, outlier_frac=0.2)
    cases.append(("outliers20", b2.problem(0), cfg.lm(40), ()))
    # fault injection on the Cholesky path
    cases.append(("fault_inject", b.problem(1), cfg.lm(200), (0, 2, 3)))
    # shuffled observation order (camera-major input, unsorted)
    p = b.problem(2)
    perm = np.random.default_rng(11).permutation(len(p["uv"]))
    for k in ("cam_idx", "pt_idx", "uv"):
        p[k] = p[k][perm]
    cases.append(("shuffled_obs", p, cfg.lm(200), ()))

    for name, p, lmcfg, fail in cases:
        prob, info, ev = run_ref(p, lmcfg, fail)
        save_case(name, p, lmcfg, prob, info, ev, fail)

    # ---- stage-level goldens on the smoke scene at its solution ----------
    p = smoke_scene(True)
    prob, info, ev = run_ref(p, cfg.lm(5))
    r, pc, bad = prob.residuals()
    e = np.linalg.norm(r, axis=1)
    w = M.huber_weights(e, 2.0)
    A, F, B = M._build_blocks(prob, pc, bad)
    U, g_c, V, g_p, Wf = M._assemble(prob, w, r, A, F, B)
    dc_s, dp_s = M.solve_step(U, g_c, V, g_p, Wf, 1e-3, "schur")
    dc_d, dp_d = M.solve_step(U, g_c, V, g_p, Wf, 1e-3, "dense")
    np.savez_compressed(os.path.join(HERE, "stages_smoke.npz"),
                        R=prob.R, t=prob.t, focal=prob.focal, cx=prob.cx, cy=prob.cy,
                        points=prob.points, cam_idx=prob.cam_idx, pt_idx=prob.pt_idx,
                        uv=prob.uv, fixed_cams=prob.fixed_cams, r=r, p_cam=pc, bad=bad,
                        e=e, w=w, A=A, F=F, B=B, U=U, g_c=g_c, V=V, g_p=g_p, Wf=Wf,
                        lam=1e-3, dc_schur=dc_s, dp_schur=dp_s, dc_dense=dc_d, dp_dense=dp_d,
                        huber_cost=M.huber_cost(e, 2.0))
    print("stages_smoke written")

    # ---- pose_lm golden: RANSAC-shaped batch and a refine ------------------
    d = S.pnp_problem(3, n=160, outlier_frac=0.3)
    intr = d["intr"]
    rng = np.random.default_rng(5)
    Bh, Ms = 256, 4
    samples = np.argsort(rng.random((Bh, len(d["points"]))), axis=1)[:, :Ms]
    R0 = np.broadcast_to(d["init_pose"].R, (Bh, 3, 3)).copy()
    t0 = np.broadcast_to(d["init_pose"].translation, (Bh, 3)).copy()
    lmc = LmConfig()
    Rr, tr, cr = M.pose_lm(R0, t0, d["points"][samples], d["pixels"][samples], intr, 5, lmc)
    inl = d["inlier_mask"]
    Rf, tf, cf = M.pose_lm(d["init_pose"].R[None], d["init_pose"].translation[None],
                           d["points"][inl][None], d["pixels"][inl][None], intr, 20, lmc)
    np.savez_compressed(os.path.join(HERE, "pose_lm.npz"),
                        focal=intr.focal, cx=intr.cx, cy=intr.cy,
                        R0=R0, t0=t0, X=d["points"][samples], uv=d["pixels"][samples],
                        iters=5, R_out=Rr, t_out=tr, cost_out=cr,
                        Rf0=d["init_pose"].R[None], tf0=d["init_pose"].translation[None],
                        Xf=d["points"][inl][None], uvf=d["pixels"][inl][None], iters_f=20,
                        Rf_out=Rf, tf_out=tf, costf_out=cf)
    print("pose_lm written")

    # ---- bootstrap (the production caller of lm_solve, miniba.py:729-854) ----
    for seed in (0, 1):
        bp = S.bootstrap_problem(seed, n_cams=8, n_points=300, noise_px=0.5)
        poses, intr_out, table, info = M.bootstrap(bp["features"], bp["intr"], cfg,
                                                   matcher=bp["matcher"])
        kp = np.concatenate([f[0] for f in bp["features"]])
        ids = np.concatenate([f[1] for f in bp["features"]])
        counts = np.array([len(f[1]) for f in bp["features"]])
        np.savez_compressed(os.path.join(HERE, f"bootstrap_seed{seed}.npz"),
                            keypoints=kp, ids=ids, counts=counts, focal=bp["intr"].focal,
                            cx=bp["intr"].cx, cy=bp["intr"].cy, width=bp["intr"].width,
                            height=bp["intr"].height,
                            out_R=np.stack([p.R for p in poses]),
                            out_t=np.stack([p.translation for p in poses]),
                            out_focal=intr_out.focal, out_n_tracks=info["n_tracks"],
                            out_mean_err=info["mean_err"], out_rescued=info["rescued"],
                            out_costs=info["costs"])
        print(f"bootstrap seed {seed}: focal {intr_out.focal:.3f} tracks {info['n_tracks']} "
              f"rescued {info['rescued']}")


if __name__ == "__main__":
    main()
