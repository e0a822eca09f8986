"""Bootstrap orchestration around the device LM (reference miniba.py:537-854).

This is the production caller of `lm_solve`: exhaustive pairwise matching into
tracks (union-find), the paper's initialisation (identity poses, depth-1
points, focal = 0.7 x width), the 100 + 100 iteration schedule with a
median + 4 MAD residual filter in between, gauge normalisation, and the
two-view rescue when self-calibration collapses. Host orchestration only;
both solves run through the device `lm_solve`. Feature extraction / matching
(the reference's `frontend`) is out of scope: pass a `matcher`.
"""
from __future__ import annotations

import numpy as np

from .config import CaptureConfig
from .scene import CameraIntrinsics, Pose, TrackTable, unproject


def _find(parent, x):
    root = parent.setdefault(x, x)
    while root != parent[root]:
        parent[root] = parent[parent[root]]
        root = parent[root]
    parent[x] = root
    return root


def filter_matches_flow(kps_a, kps_b, idx_a, idx_b, k: int = 6, base_tol: float = 3.0,
                        rel_tol: float = 0.5) -> np.ndarray:
    """Keep matches whose displacement agrees with the median displacement of
    their k nearest matched neighbours (frontend.py:188-207): deviation <=
    max(base_tol, rel_tol * |median|). Returns a keep mask."""
    from scipy.spatial import cKDTree
    if len(idx_a) < k + 1:
        return np.ones(len(idx_a), dtype=bool)
    pa = np.asarray(kps_a)[idx_a]
    disp = np.asarray(kps_b)[idx_b] - pa
    _, nb = cKDTree(pa).query(pa, k=k + 1)
    med = np.median(disp[nb[:, 1:]], axis=1)
    dev = np.linalg.norm(disp - med, axis=1)
    return dev <= np.maximum(base_tol, rel_tol * np.linalg.norm(med, axis=1))


def build_tracks_device(features: list, n_obs_max: int | None = None) -> list:
    """`build_tracks(features, default_matcher)` (miniba.py:555-602) with the
    exhaustive pairwise descriptor matching of all frame pairs in ONE device
    call (match_batch -> mba_match_pairs); the flow filter and the union-find
    grouping run on the host."""
    from .miniba import match_batch
    n = len(features)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    res = dict(zip(pairs, match_batch([f[1] for f in features], pairs)))

    def matcher_from_batch(i, j):
        ia, ib, sc = res[(i, j)]
        keep = filter_matches_flow(features[i][0], features[j][0], ia, ib)
        return ia[keep], ib[keep], sc[keep]
    return _group_tracks(features, matcher_from_batch, n_obs_max)


def build_tracks(features: list, matcher, n_obs_max: int | None = None) -> list:
    """Union-find over all pairwise matches; tracks with two keypoints in one
    frame are dropped; observations ordered by frame; optionally capped to the
    most recent n_obs_max. Sorted by (first frame, first keypoint)."""
    return _group_tracks(features, lambda i, j: matcher(features[i], features[j]), n_obs_max)


def _group_tracks(features: list, pair_matches, n_obs_max: int | None) -> list:
    parent: dict = {}
    n = len(features)
    for i in range(n):
        for j in range(i + 1, n):
            ia, ib, _ = pair_matches(i, j)
            for a, b in zip(ia, ib):
                ra, rb = _find(parent, (i, int(a))), _find(parent, (j, int(b)))
                if ra != rb:
                    parent[rb] = ra
    groups: dict = {}
    for key in list(parent):
        groups.setdefault(_find(parent, key), []).append(key)
    tracks = []
    for members in groups.values():
        frames = [m[0] for m in members]
        if len(members) < 2 or len(set(frames)) != len(frames):
            continue
        members.sort()
        obs = [(fr, kp, float(features[fr][0][kp][0]), float(features[fr][0][kp][1]))
               for fr, kp in members]
        tracks.append(obs if n_obs_max is None else obs[-n_obs_max:])
    tracks.sort(key=lambda o: (o[0][0], o[0][1]))
    return tracks


def _midpoints(Ra, ta, Rb, tb, xa, xb):
    ca, cb = -Ra.T @ ta, -Rb.T @ tb
    da = np.c_[xa, np.ones(len(xa))] @ Ra
    db = np.c_[xb, np.ones(len(xb))] @ Rb
    da /= np.linalg.norm(da, axis=1, keepdims=True)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    w0 = ca - cb
    b = np.sum(da * db, axis=1)
    d, e = da @ w0, db @ w0
    den = 1.0 - b * b
    den = np.where(np.abs(den) < 1e-12, 1e-12, den)
    s, u = (b * e - d) / den, (e - b * d) / den
    return 0.5 * (ca + s[:, None] * da + cb + u[:, None] * db)


def _essential(xa, xb):
    def norm(x):
        m = x.mean(axis=0)
        s = np.sqrt(2.0) / max(np.mean(np.linalg.norm(x - m, axis=1)), 1e-12)
        return (x - m) * s, np.array([[s, 0, -s * m[0]], [0, s, -s * m[1]], [0, 0, 1.0]])
    na, Ta = norm(xa)
    nb, Tb = norm(xb)
    A = np.c_[nb[:, :1] * na, nb[:, :1], nb[:, 1:2] * na, nb[:, 1:2], na, np.ones(len(na))]
    F = Tb.T @ np.linalg.svd(A, full_matrices=False)[2][-1].reshape(3, 3) @ Ta
    u, s, vt = np.linalg.svd(F)
    m = 0.5 * (s[0] + s[1])
    return u @ np.diag([m, m, 0.0]) @ vt


def _relative_pose(E, xa, xb):
    u, _, vt = np.linalg.svd(E)
    u = -u if np.linalg.det(u) < 0 else u
    vt = -vt if np.linalg.det(vt) < 0 else vt
    Wm = np.array([[0.0, -1, 0], [1, 0, 0], [0, 0, 1]])
    best = None
    for R in (u @ Wm @ vt, u @ Wm.T @ vt):
        for sgn in (1.0, -1.0):
            t = sgn * u[:, 2]
            X = _midpoints(np.eye(3), np.zeros(3), R, t, xa, xb)
            votes = int(np.sum((X[:, 2] > 0) & ((X @ R.T + t)[:, 2] > 0)))
            if best is None or votes > best[0]:
                best = (votes, R, t)
    return best[1], best[2]


def _two_view_init(track_obs, n, intr0):
    from scipy.spatial.transform import Rotation, Slerp
    px = [dict() for _ in range(n)]
    for j, obs in enumerate(track_obs):
        for fr, _, x, y in obs:
            px[fr][j] = (x, y)
    best = None
    for i in range(n):
        for j in range(i + 1, n):
            shared = sorted(px[i].keys() & px[j].keys())
            if len(shared) < 30:
                continue
            pa = np.array([px[i][k] for k in shared])
            pb = np.array([px[j][k] for k in shared])
            disp = float(np.median(np.linalg.norm(pb - pa, axis=1)))
            if best is None or disp > best[0]:
                best = (disp, i, j, shared, pa, pb)
    if best is None:
        return None
    _, ia, ib, shared, pa, pb = best
    pp = np.array([intr0.cx, intr0.cy])
    xa, xb = (pa - pp) / intr0.focal, (pb - pp) / intr0.focal
    R, t = _relative_pose(_essential(xa, xb), xa, xb)
    sl = Slerp([float(ia), float(ib)], Rotation.from_matrix(np.stack([np.eye(3), R])))
    Rs, ts = np.empty((n, 3, 3)), np.empty((n, 3))
    for fr in range(n):
        fc = float(np.clip(fr, ia, ib))
        Rs[fr] = sl(fc).as_matrix()
        ts[fr] = (fc - ia) / max(ib - ia, 1) * t
    tri = _midpoints(np.eye(3), np.zeros(3), R, t, xa, xb)
    front = tri[:, 2] > 0
    dmed = float(np.median(tri[front, 2])) if np.any(front) else 1.0
    row = {k: i for i, k in enumerate(shared)}
    pts = np.empty((len(track_obs), 3))
    for j, obs in enumerate(track_obs):
        r = row.get(j)
        if r is not None and front[r]:
            pts[j] = tri[r]
        else:
            fr0, _, x0, y0 = obs[0]
            pts[j] = unproject(intr0, Pose.from_matrix(Rs[fr0], ts[fr0]), [[x0, y0]], [dmed])[0]
    return Rs, ts, pts


def bootstrap(features: list, intr: CameraIntrinsics, cfg: CaptureConfig, matcher=None,
              optimize_focal: bool = True):
    """Joint pose / point / focal estimation for the first frames; returns
    (poses, intrinsics, TrackTable, info). Raises BootstrapFailure."""
    from . import miniba as M
    if matcher is None:
        raise NotImplementedError("the feature frontend is out of scope: pass matcher=")
    n = len(features)
    all_tracks = build_tracks(features, matcher, None)
    if len(all_tracks) < M.MIN_BOOTSTRAP_TRACKS:
        raise M.BootstrapFailure(f"{len(all_tracks)} tracks < {M.MIN_BOOTSTRAP_TRACKS}")
    track_obs = [tr for tr in all_tracks if len(tr) >= 3]
    if len(track_obs) < M.MIN_BOOTSTRAP_TRACKS:
        track_obs = all_tracks
    focal0 = cfg.focal_init_factor * intr.width if optimize_focal else intr.focal
    intr0 = CameraIntrinsics(focal0, intr.cx, intr.cy, intr.width, intr.height)
    cam_idx = np.array([fr for obs in track_obs for fr, _, _, _ in obs])
    pt_idx = np.array([j for j, obs in enumerate(track_obs) for _ in obs])
    uv = np.array([(x, y) for obs in track_obs for _, _, x, y in obs], dtype=np.float64)

    def make(Rs, ts, pts):
        return M.BaProblem(R=Rs, t=ts, focal=focal0, cx=intr.cx, cy=intr.cy, points=pts,
                           cam_idx=cam_idx.copy(), pt_idx=pt_idx.copy(), uv=uv.copy(),
                           fixed_cams=np.arange(n) == 0, optimize_focal=optimize_focal)

    def schedule(prob):
        half = cfg.bootstrap_iters // 2
        info1 = M.lm_solve(prob, cfg.lm(half))
        r, _, _ = prob.residuals()
        keep = M.robust_filter(np.linalg.norm(r, axis=1), cfg.lm_mad_factor)
        counts = np.bincount(prob.pt_idx[keep], minlength=len(prob.points))
        keep &= counts[prob.pt_idx] >= 2
        prob.cam_idx, prob.pt_idx, prob.uv = prob.cam_idx[keep], prob.pt_idx[keep], prob.uv[keep]
        if len(prob.uv) == 0:
            raise M.BootstrapFailure("robust filter removed every observation")
        info2 = M.lm_solve(prob, cfg.lm(cfg.bootstrap_iters - half))
        centers = np.einsum("nji,nj->ni", prob.R, -prob.t)
        iu, ju = np.triu_indices(n, 1)
        mean_d = float(np.mean(np.linalg.norm(centers[iu] - centers[ju], axis=1)))
        if mean_d > 1e-12:
            prob.t *= 1.0 / mean_d
            prob.points *= 1.0 / mean_d
        return info1, info2

    def degenerate(prob):
        lo, hi = M.FOCAL_BOUNDS
        return optimize_focal and not (lo * intr.width <= prob.focal <= hi * intr.width)

    ident = Pose.identity()
    pts0 = np.stack([unproject(intr0, ident, [[obs[0][2], obs[0][3]]], [1.0])[0] for obs in track_obs])
    prob = make(np.stack([np.eye(3)] * n), np.zeros((n, 3)), pts0)
    info1, info2 = schedule(prob)
    rescued = False
    if degenerate(prob):
        init = _two_view_init(track_obs, n, intr0)
        if init is not None:
            prob = make(*init)
            info1, info2 = schedule(prob)
            rescued = True
            R0, t0 = prob.R[0].copy(), prob.t[0].copy()
            prob.points = prob.points @ R0.T + t0
            for c in range(n):
                Rc = prob.R[c] @ R0.T
                prob.t[c] = prob.t[c] - Rc @ t0
                prob.R[c] = Rc
        if degenerate(prob):
            raise M.BootstrapFailure(f"degenerate solution: focal {prob.focal:.1f} outside "
                                     f"[{M.FOCAL_BOUNDS[0]}, {M.FOCAL_BOUNDS[1]}] x width {intr.width}")
    poses = [Pose.from_matrix(prob.R[i], prob.t[i]) for i in range(n)]
    intr_out = CameraIntrinsics(prob.focal, intr.cx, intr.cy, intr.width, intr.height)
    table = TrackTable(cfg.n_obs_max)
    surviving = np.unique(prob.pt_idx)
    for j in surviving:
        table.new_track(track_obs[j], point=prob.points[j].copy())
    info = dict(costs=np.concatenate([info1["costs"], info2["costs"]]), mean_err=info2["mean_err"],
                n_tracks=len(surviving), focal=prob.focal, rescued=rescued)
    return poses, intr_out, table, info
