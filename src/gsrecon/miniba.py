"""Mini bundle adjustment -- B200-native drop-in for the reference's
`gsrecon.miniba` (/root/reference/pkg/src/gsrecon/miniba.py).

Same names, argument layouts, return layouts and error behaviour as the
reference; the numerical work runs in libminiba.so (sm_100a):

* `lm_solve` (miniba.py:223-296) -> one `mba_solve` launch: the entire LM loop
  (linearise, normal equations, Schur, Cholesky, backtracking trials, lambda
  schedule, termination) runs on device; one upload, one download.
* `lm_solve_batch` -> many independent problems in one launch (extension).
* `BaProblem.residuals`, `huber_cost`, `huber_weights`, `_build_blocks`,
  `_assemble`, `solve_step` -> the float64 stage kernels (mba_stages.cu),
  kept for callers of the reference's internal API (smoke_miniba.py:85-96).
* `pose_lm`, `estimate_pose_ransac`, `refine_pose` -> the batched pose-only LM
  kernel (mba_pose.cu) with on-device hypothesis scoring.

Host-side helpers that are not LM (triangulation, robust filter, restart and
alignment checks, bootstrap orchestration) are small numpy code written for
this package. There is no CPU fallback for any LM path: without the library
or a CUDA device the calls raise.
"""
from __future__ import annotations

import os
import sys
from dataclasses import dataclass

import numpy as np

_REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _REPO not in sys.path:
    sys.path.insert(0, _REPO)

from paper_2506_05558_b200 import _lib, solver  # noqa: E402
from paper_2506_05558_b200._lib import ptr  # noqa: E402

from .config import CaptureConfig, LmConfig  # noqa: E402
from .scene import (CameraIntrinsics, Pose, TrackTable, exp_so3, project,  # noqa: E402,F401
                    umeyama, unproject)

MIN_BOOTSTRAP_TRACKS = 100
MIN_PNP_CORRESPONDENCES = 8
LAMBDA_MAX = 1e10
DIAG_FLOOR = 1e-12
BACKTRACK_TRIES = 5
ESSENTIAL_MIN_SHARED = 30
FOCAL_BOUNDS = (0.25, 3.0)


class BootstrapFailure(RuntimeError):
    pass


class EstimationFailure(RuntimeError):
    pass


class TriangulationFailure(RuntimeError):
    pass


class AlignmentRejected(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# device helpers

def _torch():
    return _lib.torch_cuda()


def _dev(a, dtype=None):
    torch = _torch()
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    if not arr.flags.writeable:
        arr = arr.copy()
    return torch.from_numpy(arr).to("cuda", non_blocking=False)


def _empty(shape, dtype):
    torch = _torch()
    return torch.empty(shape, dtype=dtype, device="cuda")


def _host(t):
    return t.cpu().numpy()


def _loss_of(cfg):
    return getattr(cfg, "loss", "huber")


# ---------------------------------------------------------------------------
# robust loss (miniba.py:46-62)

def _robust(e, delta, loss, want_w):
    torch = _torch()
    e = np.asarray(e, dtype=np.float64).reshape(-1)
    de = _dev(e)
    w = _empty(e.shape, torch.float64) if want_w else None
    cost = _empty((1,), torch.float64)
    _lib.check(_lib.lib().mba_robust(len(e), ptr(de), float(delta), _lib.LOSS[loss], ptr(w), ptr(cost),
                                     _lib.stream_ptr()), "mba_robust")
    return (_host(w) if want_w else None), float(cost.item())


def huber_cost(e: np.ndarray, delta: float) -> float:
    return _robust(e, delta, "huber", False)[1]


def huber_weights(e: np.ndarray, delta: float) -> np.ndarray:
    shape = np.shape(e)
    return _robust(e, delta, "huber", True)[0].reshape(shape)


def cauchy_cost(e: np.ndarray, delta: float) -> float:
    return _robust(e, delta, "cauchy", False)[1]


def cauchy_weights(e: np.ndarray, delta: float) -> np.ndarray:
    shape = np.shape(e)
    return _robust(e, delta, "cauchy", True)[0].reshape(shape)


def robust_filter(residual_norms: np.ndarray, factor: float = 4.0) -> np.ndarray:
    """Keep residual norms <= median + factor * MAD (miniba.py:57-62)."""
    e = np.asarray(residual_norms, dtype=np.float64)
    m = np.median(e)
    return e <= m + factor * np.median(np.abs(e - m))


# ---------------------------------------------------------------------------
# problem container (miniba.py:65-98)

@dataclass
class BaProblem:
    R: np.ndarray
    t: np.ndarray
    focal: float
    cx: float
    cy: float
    points: np.ndarray
    cam_idx: np.ndarray
    pt_idx: np.ndarray
    uv: np.ndarray
    fixed_cams: np.ndarray
    optimize_focal: bool = True
    optimize_points: bool = True

    def n_cam_params(self) -> int:
        return 6 * int(np.count_nonzero(~np.asarray(self.fixed_cams, dtype=bool))) + int(bool(self.optimize_focal))

    def residuals(self):
        """(K,2) residuals, (K,3) camera-frame points, (K,) behind-camera mask."""
        torch = _torch()
        K = len(self.uv)
        R, t, X = _dev(self.R, np.float64), _dev(self.t, np.float64), _dev(self.points, np.float64)
        cam, pt, uv = _dev(self.cam_idx, np.int64), _dev(self.pt_idx, np.int64), _dev(self.uv, np.float64)
        r = _empty((K, 2), torch.float64)
        pc = _empty((K, 3), torch.float64)
        bad = _empty((K,), torch.uint8)
        _lib.check(_lib.lib().mba_residuals(K, ptr(R), ptr(t), float(self.focal), float(self.cx),
                                            float(self.cy), ptr(X), ptr(cam), ptr(pt), ptr(uv), ptr(r),
                                            ptr(pc), ptr(bad), _lib.stream_ptr()), "mba_residuals")
        return _host(r), _host(pc), _host(bad).astype(bool)


# ---------------------------------------------------------------------------
# stage API (miniba.py:101-220)

def _build_blocks(prob: BaProblem, p_cam: np.ndarray, bad: np.ndarray):
    torch = _torch()
    K = len(prob.uv)
    R, t = _dev(prob.R, np.float64), _dev(prob.t, np.float64)
    cam, pc, bd = _dev(prob.cam_idx, np.int64), _dev(p_cam, np.float64), _dev(bad, np.uint8)
    A = _empty((K, 2, 6), torch.float64)
    F = _empty((K, 2), torch.float64)
    B = _empty((K, 2, 3), torch.float64)
    _lib.check(_lib.lib().mba_blocks(K, ptr(R), ptr(t), float(prob.focal), ptr(cam), ptr(pc), ptr(bd),
                                     ptr(A), ptr(F), ptr(B), _lib.stream_ptr()), "mba_blocks")
    return _host(A), _host(F), _host(B)


def _slots(fixed):
    fixed = np.asarray(fixed, dtype=bool)
    free = np.flatnonzero(~fixed)
    slot = np.full(len(fixed), -1, dtype=np.int32)
    slot[free] = np.arange(len(free), dtype=np.int32)
    return slot, free.astype(np.int32)


def _assemble(prob: BaProblem, w: np.ndarray, r: np.ndarray, A: np.ndarray, F: np.ndarray,
              B: np.ndarray):
    """U (C,C), g_c (C,), V (P,3,3), g_p (P,3), Wf (P,C,3) (miniba.py:135-177)."""
    torch = _torch()
    K = len(prob.uv)
    n = len(prob.R)
    P = len(prob.points)
    slot, free = _slots(prob.fixed_cams)
    C = prob.n_cam_params()
    cam = np.asarray(prob.cam_idx, dtype=np.int64)
    pt = np.asarray(prob.pt_idx, dtype=np.int64)
    pt_order = np.argsort(pt, kind="stable")
    pt_ptr = np.searchsorted(pt[pt_order], np.arange(P + 1)).astype(np.int64)
    cam_order = np.argsort(cam, kind="stable")
    cam_ptr = np.searchsorted(cam[cam_order], np.arange(n + 1)).astype(np.int64)
    d = [_dev(x) for x in (slot, free if len(free) else np.zeros(1, np.int32), cam,
                           np.asarray(w, np.float64), np.asarray(r, np.float64),
                           np.asarray(A, np.float64), np.asarray(F, np.float64),
                           np.asarray(B, np.float64), pt_order, pt_ptr, cam_order, cam_ptr)]
    U = _empty((C, C), torch.float64)
    g_c = _empty((C,), torch.float64)
    V = _empty((P, 3, 3), torch.float64)
    g_p = _empty((P, 3), torch.float64)
    Wf = _empty((P, C, 3), torch.float64)
    _lib.check(_lib.lib().mba_assemble(K, n, len(free), P, *[ptr(x) for x in d[:2]],
                                       int(bool(prob.optimize_focal)), int(bool(prob.optimize_points)),
                                       *[ptr(x) for x in d[2:]], ptr(U), ptr(g_c), ptr(V), ptr(g_p),
                                       ptr(Wf), _lib.stream_ptr()), "mba_assemble")
    return _host(U), _host(g_c), _host(V), _host(g_p), _host(Wf)


def solve_step(U, g_c, V, g_p, Wf, lam: float, method: str = "schur"):
    """Damped solve for (delta_cam, delta_pts) (miniba.py:180-220).

    Raises np.linalg.LinAlgError when the system is not positive definite."""
    torch = _torch()
    if method not in ("schur", "dense"):
        raise ValueError(f"unknown method {method!r}")
    C = len(g_c)
    P = len(g_p)
    L = _lib.lib()
    m = 0 if method == "schur" else 1
    args = [_dev(np.asarray(a, np.float64)) for a in (U, g_c, V, g_p, Wf)]
    dc = _empty((C,), torch.float64)
    dp = _empty((P, 3), torch.float64)
    scratch = _empty((int(L.mba_solve_step_scratch_bytes(C, P, m)),), torch.uint8)
    _lib.check(L.mba_solve_step(C, P, *[ptr(a) for a in args], float(lam), m, ptr(dc), ptr(dp),
                                ptr(scratch), _lib.stream_ptr()), "mba_solve_step")
    return _host(dc), _host(dp)


# ---------------------------------------------------------------------------
# LM driver (miniba.py:223-296)

_SOLVERS = {}


def lm_solve_batch(problems, cfg: LmConfig, precision: str | None = None):
    """Solve many independent problems (extension of lm_solve): each problem
    is mutated exactly as lm_solve would mutate it (miniba.py:264-270, 288) and
    the per-problem info dicts are returned as a lazy sequence
    (paper_2506_05558_b200.batch.BatchResult).

    The list is walked and copied by native code, the observations are sorted
    point-major and packed on the device, and chunks of the batch flow through
    upload -> pack -> solve -> read-back -> write-back with host and device
    work overlapped (paper_2506_05558_b200/batch.py)."""
    from paper_2506_05558_b200.batch import BatchSolver
    prm = solver.LmParams.from_cfg(cfg)
    if precision is not None:
        prm.precision = precision
    torch = _torch()
    key = torch.cuda.current_device()
    bs = _SOLVERS.get(key)
    if bs is None:
        bs = _SOLVERS[key] = BatchSolver(prm)
    bs.prm = prm
    # more cameras than the fused kernel holds: the stage-kernel loop
    bs.oversize = lambda p: _lm_stages(p, cfg, "schur")
    bs.max_cams = MAX_FUSED_CAMS
    res = bs.solve(problems)
    torch.cuda.current_stream().wait_stream(bs.back)
    return res


MAX_FUSED_CAMS = 32   # cameras per problem the fused on-device LM loop holds (mba_solve)


def _lm_stages(prob: BaProblem, cfg: LmConfig, method: str = "schur") -> dict:
    """The reference loop (miniba.py:223-296) driven from the host with every
    numerical stage on the device stage kernels (residuals, robust weights,
    blocks, assembly, solve_step). Serves method="dense" (the reference's
    verification path) and problems with more cameras than the fused kernel
    holds (MAX_FUSED_CAMS); one host round trip per stage, so it is the slow
    path."""
    loss = _loss_of(cfg)
    cost_fn = huber_cost if loss == "huber" else cauchy_cost
    w_fn = huber_weights if loss == "huber" else cauchy_weights
    lam = cfg.lambda_init
    r, p_cam, bad = prob.residuals()
    e = np.linalg.norm(r, axis=1)
    cost = cost_fn(e, cfg.huber_delta)
    costs, accepted, lambdas, evals = [cost], [], [], []
    status = 0   # MBA_SOLVE_MAX_ITERS / 1 converged / 2 lambda cap, as mba_solve reports
    free = np.flatnonzero(~np.asarray(prob.fixed_cams, dtype=bool))
    for _ in range(cfg.max_iters):
        w = w_fn(e, cfg.huber_delta)
        A, F, B = _build_blocks(prob, p_cam, bad)
        blocks = _assemble(prob, w, r, A, F, B)
        lambdas.append(lam)
        try:
            dc, dp = solve_step(*blocks, lam, method)
        except np.linalg.LinAlgError:
            lam = min(lam * cfg.nu, LAMBDA_MAX)
            accepted.append(False)
            evals.append(0)
            costs.append(cost)
            continue
        R0, t0, f0, X0 = prob.R.copy(), prob.t.copy(), prob.focal, prob.points.copy()
        took, tries = None, 0
        for bt in range(BACKTRACK_TRIES):
            frac = 0.5 ** bt
            for s, c in enumerate(free):
                prob.R[c] = exp_so3(frac * dc[6 * s:6 * s + 3]) @ R0[c]
                prob.t[c] = t0[c] + frac * dc[6 * s + 3:6 * s + 6]
            if prob.optimize_focal:
                prob.focal = f0 + frac * dc[-1]
            if prob.optimize_points:
                prob.points = X0 + frac * dp
            r_new, p_new, bad_new = prob.residuals()
            e_new = np.linalg.norm(r_new, axis=1)
            c_new = cost_fn(e_new, cfg.huber_delta)
            tries += 1
            if c_new < cost and np.isfinite(c_new):
                took = frac
                break
        evals.append(tries)
        if took is None:
            prob.R, prob.t, prob.focal, prob.points = R0, t0, f0, X0
            lam = min(lam * cfg.nu, LAMBDA_MAX)
            accepted.append(False)
            costs.append(cost)
            if lam >= LAMBDA_MAX:
                status = 2
                break
            continue
        lam = max(lam / cfg.nu, 1e-15) if took == 1.0 else min(lam * cfg.nu, LAMBDA_MAX)
        gain = cost - c_new
        cost, r, e, p_cam, bad = c_new, r_new, e_new, p_new, bad_new
        accepted.append(True)
        costs.append(cost)
        if gain <= 1e-15 * max(cost, 1.0):
            status = 1
            break
    return dict(costs=np.array(costs), accepted=np.array(accepted, dtype=bool),
                lambdas=np.array(lambdas), final_rms=float(np.sqrt(np.mean(e ** 2))),
                mean_err=float(np.mean(e)), evals=np.array(evals, dtype=np.int32), status=status)


def lm_solve(prob: BaProblem, cfg: LmConfig, method: str = "schur") -> dict:
    """Levenberg-Marquardt with multiplicative damping, 5-try backtracking and
    rollback (miniba.py:223-296). Mutates prob; returns the info dict
    (costs, accepted, lambdas, final_rms, mean_err; plus evals, status)."""
    if len(prob.uv) == 0:
        raise ValueError("problem has no residuals")
    if method == "dense":
        return _lm_stages(prob, cfg, "dense")
    if method != "schur":
        raise ValueError(f"unknown method {method!r}")
    return lm_solve_batch([prob], cfg)[0]


# ---------------------------------------------------------------------------
# batched pose-only LM (miniba.py:303-451)

def _pose_call(R0, t0, pts, uv, intr, iters, cfg, X_all=None, uv_all=None, thr=0.0):
    torch = _torch()
    R = _dev(np.asarray(R0, np.float64).reshape(-1, 3, 3))
    t = _dev(np.asarray(t0, np.float64).reshape(-1, 3))
    nb = R.shape[0]
    pts = np.asarray(pts, np.float64)
    uv = np.asarray(uv, np.float64)
    m = pts.shape[-2]
    X = _dev(np.broadcast_to(pts.reshape(-1, m, 3), (nb, m, 3)))
    U = _dev(np.broadcast_to(uv.reshape(-1, m, 2), (nb, m, 2)))
    cost = _empty((nb,), torch.float64)
    inl = sse = Xa = Ua = None
    m_all = 0
    if X_all is not None:
        m_all = len(X_all)
        Xa, Ua = _dev(np.asarray(X_all, np.float64)), _dev(np.asarray(uv_all, np.float64))
        inl = _empty((nb,), torch.int32)
        sse = _empty((nb,), torch.float64)
    _lib.check(_lib.lib().mba_pose_lm(nb, m, ptr(X), ptr(U), float(intr.focal), float(intr.cx),
                                      float(intr.cy), int(iters), float(cfg.lambda_init), float(cfg.nu),
                                      float(cfg.huber_delta), ptr(R), ptr(t), ptr(cost), m_all, ptr(Xa),
                                      ptr(Ua), float(thr), ptr(inl), ptr(sse), _lib.stream_ptr()),
               "mba_pose_lm")
    out = (_host(R), _host(t), _host(cost))
    if X_all is not None:
        out = out + (_host(inl), _host(sse))
    return out


def pose_lm(R0: np.ndarray, t0: np.ndarray, pts: np.ndarray, uv: np.ndarray,
            intr: CameraIntrinsics, iters: int, cfg: LmConfig):
    """Batched pose-only LM. R0 (B,3,3), t0 (B,3), pts (B,M,3), uv (B,M,2).
    Returns refined (R, t) and the final per-problem robust cost."""
    R, t, c = _pose_call(R0, t0, pts, uv, intr, iters, cfg)
    return R, t, c


def _reproj_err(R, t, pts, px, intr):
    """Per-correspondence pixel error of one pose (inf behind the camera)."""
    prob = BaProblem(R=np.asarray(R, np.float64)[None], t=np.asarray(t, np.float64)[None],
                     focal=intr.focal, cx=intr.cx, cy=intr.cy, points=np.asarray(pts, np.float64),
                     cam_idx=np.zeros(len(pts), np.int64), pt_idx=np.arange(len(pts)),
                     uv=np.asarray(px, np.float64), fixed_cams=np.array([True]))
    r, _, bad = prob.residuals()
    return np.where(bad, np.inf, np.hypot(r[:, 0], r[:, 1]))


def estimate_pose_ransac(points3d: np.ndarray, pixels: np.ndarray, intr: CameraIntrinsics,
                         init_pose: Pose, cfg: CaptureConfig, rng: np.random.Generator):
    """256 minimal-sample hypotheses, each LM-refined and scored on device
    (miniba.py:392-439). Returns (pose, inlier_mask)."""
    M = len(points3d)
    if M < MIN_PNP_CORRESPONDENCES:
        raise EstimationFailure(f"{M} correspondences < {MIN_PNP_CORRESPONDENCES}")
    B = cfg.ransac_hypotheses
    samples = np.argsort(rng.random((B, M)), axis=1)[:, :cfg.ransac_sample]
    lmc = LmConfig(lambda_init=cfg.lm_lambda_init, nu=cfg.lm_nu, huber_delta=cfg.lm_huber_delta,
                   max_iters=cfg.ransac_lm_iters)
    pts = np.asarray(points3d, np.float64)
    px = np.asarray(pixels, np.float64)
    R0 = np.broadcast_to(init_pose.R, (B, 3, 3))
    t0 = np.broadcast_to(init_pose.translation, (B, 3))
    R, t, _, counts, sse = _pose_call(R0, t0, pts[samples], px[samples], intr, cfg.ransac_lm_iters,
                                      lmc, X_all=pts, uv_all=px, thr=cfg.ransac_inlier_px)
    best_count = int(counts.max())
    if best_count > 0:
        cands = np.flatnonzero(counts == best_count)
        best = int(cands[np.argmin(np.sqrt(sse[cands] / best_count))])
    else:
        best = 0
    if best_count < cfg.ransac_min_inlier_ratio * M:
        raise EstimationFailure(f"inlier ratio {best_count / M:.3f} below {cfg.ransac_min_inlier_ratio}")
    inl = _reproj_err(R[best], t[best], pts, px, intr) < cfg.ransac_inlier_px
    return Pose.from_matrix(R[best], t[best]), inl


def refine_pose(pose: Pose, points3d: np.ndarray, pixels: np.ndarray, intr: CameraIntrinsics,
                cfg: CaptureConfig) -> Pose:
    """Pose-only LM over the given (inlier) correspondences (miniba.py:442-451)."""
    lmc = LmConfig(lambda_init=cfg.lm_lambda_init, nu=cfg.lm_nu, huber_delta=cfg.lm_huber_delta,
                   max_iters=cfg.refine_iters)
    R, t, _ = _pose_call(pose.R[None], pose.translation[None], np.asarray(points3d)[None],
                         np.asarray(pixels)[None], intr, cfg.refine_iters, lmc)
    return Pose.from_matrix(R[0], t[0])


# ---------------------------------------------------------------------------
# host geometry around the solver (not LM; miniba.py:458-530, 861-908)

def triangulate(poses: list, pixels: np.ndarray, intr: CameraIntrinsics, max_reproj_px: float = 8.0,
                min_angle_deg: float = 0.5, gn_steps: int = 3) -> np.ndarray:
    """Widest-angle ray pair midpoint, then Gauss-Newton on reprojection error.
    Raises TriangulationFailure on a degenerate baseline, parallel rays, a point
    behind a camera, or a mean reprojection error above max_reproj_px."""
    n = len(poses)
    if n < 2:
        raise TriangulationFailure("need at least two observations")
    px = np.asarray(pixels, dtype=np.float64).reshape(n, 2)
    Rs = np.stack([p.R for p in poses])
    ts = np.stack([p.translation for p in poses])
    centers = -np.einsum("nji,nj->ni", Rs, ts)
    rays = np.stack([(px[:, 0] - intr.cx) / intr.focal, (px[:, 1] - intr.cy) / intr.focal,
                     np.ones(n)], axis=1)
    rays = np.einsum("nji,nj->ni", Rs, rays)
    rays /= np.linalg.norm(rays, axis=1, keepdims=True)
    cosines = np.clip(np.abs(rays @ rays.T), -1.0, 1.0)
    iu, ju = np.triu_indices(n, 1)
    angles = np.degrees(np.arccos(cosines[iu, ju]))
    k = int(np.argmax(angles))
    if angles[k] <= min_angle_deg:
        raise TriangulationFailure(f"baseline angle {angles[k]:.3f} deg too small")
    i, j = iu[k], ju[k]
    d1, d2, o1, o2 = rays[i], rays[j], centers[i], centers[j]
    a, b, c = d1 @ d1, d1 @ d2, d2 @ d2
    w0 = o2 - o1
    den = a * c - b * b
    if den < 1e-18:
        raise TriangulationFailure("parallel rays")
    s1 = (c * (d1 @ w0) - b * (d2 @ w0)) / den
    s2 = (b * (d1 @ w0) - a * (d2 @ w0)) / den
    X = 0.5 * (o1 + s1 * d1 + o2 + s2 * d2)
    f = intr.focal
    for _ in range(gn_steps):
        pc = np.einsum("nij,j->ni", Rs, X) + ts
        if np.any(pc[:, 2] <= 1e-12):
            raise TriangulationFailure("point behind a camera")
        z = pc[:, 2]
        res = np.stack([f * pc[:, 0] / z + intr.cx - px[:, 0], f * pc[:, 1] / z + intr.cy - px[:, 1]],
                       axis=1).reshape(-1)
        Jp = np.zeros((n, 2, 3))
        Jp[:, 0, 0] = Jp[:, 1, 1] = f / z
        Jp[:, 0, 2] = -f * pc[:, 0] / z ** 2
        Jp[:, 1, 2] = -f * pc[:, 1] / z ** 2
        J = (Jp @ Rs).reshape(-1, 3)
        X = X - np.linalg.solve(J.T @ J + 1e-12 * np.eye(3), J.T @ res)
    pc = np.einsum("nij,j->ni", Rs, X) + ts
    if np.any(pc[:, 2] <= 1e-12):
        raise TriangulationFailure("point behind a camera")
    uvp = np.stack([f * pc[:, 0] / pc[:, 2] + intr.cx, f * pc[:, 1] / pc[:, 2] + intr.cy], axis=1)
    err = float(np.linalg.norm(uvp - px, axis=1).mean())
    if err > max_reproj_px:
        raise TriangulationFailure(f"mean reprojection {err:.2f} px")
    return X


def match_batch(descriptors: list, pairs, ratio_max: float = 0.95) -> list:
    """`frontend.match` (frontend.py:220-250) for every (i, j) in `pairs` in
    one device call (mba_match_pairs): mutual nearest neighbours in Hamming
    distance over 256-bit packed descriptors with the best/second ratio test.
    descriptors: per frame (N_f, 32) uint8. Returns [(idx_a, idx_b, scores)]
    per pair, sorted by idx_a, identical to the reference's."""
    torch = _torch()
    pairs = np.asarray(pairs, np.int32).reshape(-1, 2)
    if len(pairs) == 0:
        return []
    sizes = np.array([len(d) for d in descriptors], np.int64)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    desc = np.concatenate([np.asarray(d, np.uint8).reshape(-1, 32) for d in descriptors]) \
        if off[-1] else np.zeros((1, 32), np.uint8)
    na, nb = sizes[pairs[:, 0]], sizes[pairs[:, 1]]
    row_a = np.concatenate([[0], np.cumsum(na)]).astype(np.int64)
    row_b = np.concatenate([[0], np.cumsum(nb)]).astype(np.int64)
    ra, rb = max(int(row_a[-1]), 1), max(int(row_b[-1]), 1)
    i32 = lambda n: _empty((n,), torch.int32)
    u8 = lambda n: _empty((n,), torch.uint8)
    nn_ab, ok_a, best_ab, match_b, dist = i32(ra), u8(ra), i32(ra), i32(ra), i32(ra)
    nn_ba, ok_b = i32(rb), u8(rb)
    d_desc, d_off, d_pairs = _dev(desc), _dev(off), _dev(pairs)
    d_ra, d_rb = _dev(row_a[:-1]), _dev(row_b[:-1])
    L = _lib.lib()
    max_rows = int(max(sizes.max(), 1))
    nws = int(L.mba_match_workspace_bytes(ra, rb, max_rows))
    ws = _empty((max(nws, 16),), torch.uint8)
    _lib.check(L.mba_match_pairs(len(descriptors), ptr(d_desc), ptr(d_off), len(pairs), ptr(d_pairs),
                                 ptr(d_ra), ptr(d_rb), max_rows, float(ratio_max), ptr(nn_ab), ptr(ok_a),
                                 ptr(best_ab), ptr(nn_ba), ptr(ok_b), ptr(match_b), ptr(dist), ra, rb, ptr(ws),
                                 ws.numel(), _lib.stream_ptr()),
               "mba_match_pairs")
    mb, dd = _host(match_b), _host(dist)
    out = []
    for p in range(len(pairs)):
        m = mb[row_a[p]:row_a[p + 1]]
        ia = np.flatnonzero(m >= 0).astype(np.int64)
        ib = m[ia].astype(np.int64)
        out.append((ia, ib, 1.0 - dd[row_a[p]:row_a[p + 1]][ia] / 256.0))
    return out


TRIANGULATION_FAILURES = {1: "need at least two observations", 2: "baseline angle too small",
                          3: "parallel rays", 4: "point behind a camera", 5: "mean reprojection too large",
                          6: "camera index out of range"}


def triangulate_batch(R: np.ndarray, t: np.ndarray, cam: np.ndarray, pixels: np.ndarray,
                      obs_off: np.ndarray, intr: CameraIntrinsics, max_reproj_px: float = 8.0,
                      min_angle_deg: float = 0.5, gn_steps: int = 3):
    """`triangulate` (miniba.py:458-530) for many tracks in one device call
    (mba_triangulate, one thread per track). Track k observes camera cam[j]
    (rows of R (n,3,3) / t (n,3)) at pixels[j] for j in [obs_off[k],
    obs_off[k+1]). Returns (X (T,3), status (T,), mean_err (T,)): status 0 is a
    triangulated point; otherwise X is NaN and the status names the reference's
    TriangulationFailure (TRIANGULATION_FAILURES)."""
    torch = _torch()
    off = np.asarray(obs_off, np.int64)
    T = len(off) - 1
    if T <= 0:
        return np.zeros((0, 3)), np.zeros(0, np.int32), np.zeros(0)
    n_cams = len(np.asarray(R).reshape(-1, 9))
    cam_arr = np.asarray(cam)
    if len(cam_arr) and (cam_arr.min() < 0 or cam_arr.max() >= n_cams):
        raise IndexError("camera index out of range")
    dR = _dev(np.asarray(R, np.float64).reshape(-1, 3, 3))
    dt = _dev(np.asarray(t, np.float64).reshape(-1, 3))
    dcam = _dev(np.asarray(cam, np.int32))
    duv = _dev(np.asarray(pixels, np.float64).reshape(-1, 2))
    doff = _dev(off)
    X = _empty((T, 3), torch.float64)
    st = _empty((T,), torch.int32)
    err = _empty((T,), torch.float64)
    _lib.check(_lib.lib().mba_triangulate(T, ptr(doff), ptr(dcam), ptr(duv), int(dR.shape[0]), ptr(dR), ptr(dt),
                                          float(intr.focal), float(intr.cx), float(intr.cy),
                                          float(max_reproj_px), float(min_angle_deg), int(gn_steps),
                                          ptr(X), ptr(st), ptr(err), _lib.stream_ptr()),
               "mba_triangulate")
    return _host(X), _host(st), _host(err)


def rebootstrap_check(centers: np.ndarray, window: int = 20, min_dist: float = 0.1 / 3.0) -> bool:
    """True when the mean consecutive camera-centre distance over the last
    `window` centres is below min_dist (miniba.py:861-873)."""
    c = np.asarray(centers, dtype=np.float64)
    if len(c) < window:
        return False
    return bool(np.linalg.norm(np.diff(c[-window:], axis=0), axis=1).mean() < min_dist)


def align_bootstrap(new_poses: list, old_poses: list, new_points: np.ndarray, obs: list,
                    intr: CameraIntrinsics, max_px: float = 1.0):
    """Similarity-align a new bootstrap onto the old poses; gate by projecting
    the aligned points through the OLD poses (miniba.py:876-908)."""
    s, Rg, tg = umeyama(np.stack([p.camera_center() for p in new_poses]),
                        np.stack([p.camera_center() for p in old_poses]), with_scale=True)
    pts = s * np.asarray(new_points, dtype=np.float64) @ Rg.T + tg
    aligned = []
    for p in new_poses:
        Ra = p.R @ Rg.T
        aligned.append(Pose.from_matrix(Ra, s * p.translation - Ra @ tg))
    errs = []
    for ci, pi, u, v in obs:
        px, ok = project(intr, old_poses[ci], pts[pi][None])
        errs.append(float(np.hypot(px[0, 0] - u, px[0, 1] - v)) if ok[0] else float(intr.width))
    mean_err = float(np.mean(errs)) if errs else float("inf")
    if mean_err >= max_px:
        raise AlignmentRejected(f"mean projection error {mean_err:.2f} px")
    return aligned, pts, mean_err


from ._bootstrap import (bootstrap, bootstrap_batch, build_tracks, build_tracks_device,  # noqa: E402,F401
                         default_matcher, filter_matches_flow)
