"""Bootstrap: joint pose / point / focal estimation for the first window of
frames (the reference's `bootstrap`, gsrecon/miniba.py:729-854), built around
the device.

  features --(all frame pairs matched in one device call, mba_match_pairs;
              flow-consistency filter)--> matches
           --(connected components of the match graph)--> tracks
           --(identity poses, depth-1 points, focal = factor x width)--> problem
           --(mba_bootstrap_schedule: solve, robust filter + compaction,
              solve, gauge -- one device sequence, one upload, one download)-->
           poses, focal, points, surviving tracks

`bootstrap_batch` runs many windows through one device schedule (problems
batched like lm_solve_batch); `bootstrap` is the reference's single-window
API on top of it. When self-calibration collapses (focal outside
FOCAL_BOUNDS x width) the window is re-solved once from a two-view
initialisation (8-point essential matrix of the widest-baseline pair, poses
interpolated along it), as the reference does.
"""
from __future__ import annotations

import numpy as np

from .config import CaptureConfig
from .scene import CameraIntrinsics, Pose, TrackTable, unproject

# ---------------------------------------------------------------------------
# matching and tracks (miniba.py:537-602, frontend.py:188-250)


def filter_matches_flow(kps_a, kps_b, idx_a, idx_b, k: int = 6, base_tol: float = 3.0,
                        rel_tol: float = 0.5) -> np.ndarray:
    """Flow-consistency mask (frontend.py:188-207): a match survives when its
    displacement is within max(base_tol, rel_tol |m|) of m, the per-axis
    median displacement of its k nearest matched neighbours in image a."""
    from scipy.spatial import cKDTree
    n = len(idx_a)
    if n <= k:
        return np.ones(n, dtype=bool)
    src = np.asarray(kps_a)[np.asarray(idx_a)]
    flow = np.asarray(kps_b)[np.asarray(idx_b)] - src
    nbr = cKDTree(src).query(src, k=k + 1)[1][:, 1:]     # the point itself comes first
    m = np.median(flow[nbr], axis=1)
    tol = np.maximum(base_tol, rel_tol * np.linalg.norm(m, axis=1))
    return np.linalg.norm(flow - m, axis=1) <= tol


def default_matcher(feat_a, feat_b):
    """The reference's default matcher (miniba.py:594-602): mutual-nearest
    Hamming matching with the ratio test (device, mba_match_pairs) followed by
    the flow-consistency filter. feat_* = (keypoints (N,2), descriptors (N,32))."""
    from .miniba import match_batch
    ia, ib, sc = match_batch([feat_a[1], feat_b[1]], [(0, 1)])[0]
    keep = filter_matches_flow(feat_a[0], feat_b[0], ia, ib)
    return ia[keep], ib[keep], sc[keep]


def tracks_from_matches(features: list, pair_matches: dict, n_obs_max: int | None = None) -> list:
    """Group pairwise matches into tracks: the connected components of the
    graph whose nodes are (frame, keypoint) and whose edges are matches.
    A component is a track when it has >= 2 members from distinct frames;
    observations are (frame, kp, x, y) in (frame, kp) order, optionally
    capped to the last n_obs_max; tracks are ordered by their first
    observation (the grouping and order of build_tracks, miniba.py:555-591)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    sizes = np.array([len(f[0]) for f in features], dtype=np.int64)
    base = np.concatenate([[0], np.cumsum(sizes)])
    us, vs = [], []
    for (i, j), (ia, ib) in pair_matches.items():
        if len(ia):
            us.append(base[i] + np.asarray(ia, np.int64))
            vs.append(base[j] + np.asarray(ib, np.int64))
    if not us:
        return []
    u, v = np.concatenate(us), np.concatenate(vs)
    N = int(base[-1])
    graph = coo_matrix((np.ones(len(u), np.int8), (u, v)), shape=(N, N))
    _, label = connected_components(graph, directed=False)
    nodes = np.unique(np.concatenate([u, v]))            # keypoints that take part in a match
    frame = np.searchsorted(base, nodes, side="right") - 1
    kp = nodes - base[frame]
    lab = label[nodes]
    order = np.lexsort((kp, frame, lab))
    lab, frame, kp = lab[order], frame[order], kp[order]
    cut = np.flatnonzero(np.diff(lab)) + 1
    starts = np.concatenate([[0], cut])
    ends = np.concatenate([cut, [len(lab)]])
    tracks = []
    for s, e in zip(starts, ends):
        if e - s < 2 or np.any(frame[s + 1:e] == frame[s:e - 1]):
            continue                                        # singleton / two keypoints of one frame
        obs = [(int(fr), int(k), float(features[fr][0][k][0]), float(features[fr][0][k][1]))
               for fr, k in zip(frame[s:e], kp[s:e])]
        tracks.append(obs if n_obs_max is None else obs[-n_obs_max:])
    tracks.sort(key=lambda o: (o[0][0], o[0][1]))
    return tracks


def build_tracks(features: list, matcher, n_obs_max: int | None = None) -> list:
    """build_tracks (miniba.py:555-591) with a caller-supplied pairwise matcher."""
    n = len(features)
    pm = {}
    for i in range(n):
        for j in range(i + 1, n):
            ia, ib, _ = matcher(features[i], features[j])
            pm[(i, j)] = (ia, ib)
    return tracks_from_matches(features, pm, n_obs_max)


def build_tracks_device(features: list, n_obs_max: int | None = None) -> list:
    """build_tracks(features, default_matcher) with every frame pair of the
    window matched in ONE device call (mba_match_pairs), then the flow filter
    and the component grouping on the host."""
    from .miniba import match_batch
    n = len(features)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    pm = {}
    if pairs:
        for (i, j), (ia, ib, _) in zip(pairs, match_batch([f[1] for f in features], pairs)):
            keep = filter_matches_flow(features[i][0], features[j][0], ia, ib)
            pm[(i, j)] = (ia[keep], ib[keep])
    return tracks_from_matches(features, pm, n_obs_max)


# ---------------------------------------------------------------------------
# two-view initialisation (the rescue path, miniba.py:605-726)


def _ray_midpoints(R1, t1, R2, t2, x1, x2):
    """Closest-point midpoints of the viewing rays of normalised image points
    x1 (camera 1) and x2 (camera 2)."""
    o1, o2 = -R1.T @ t1, -R2.T @ t2
    h1 = np.concatenate([x1, np.ones((len(x1), 1))], axis=1) @ R1
    h2 = np.concatenate([x2, np.ones((len(x2), 1))], axis=1) @ R2
    d1 = h1 / np.linalg.norm(h1, axis=1, keepdims=True)
    d2 = h2 / np.linalg.norm(h2, axis=1, keepdims=True)
    w = o1 - o2
    cos = np.einsum("ij,ij->i", d1, d2)
    p, q = d1 @ w, d2 @ w
    den = 1.0 - cos * cos
    den = np.where(np.abs(den) < 1e-12, 1e-12, den)
    s1 = (cos * q - p) / den
    s2 = (q - cos * p) / den
    return 0.5 * (o1 + s1[:, None] * d1 + o2 + s2[:, None] * d2)


def _hartley(x):
    c = x.mean(axis=0)
    s = np.sqrt(2.0) / max(float(np.mean(np.linalg.norm(x - c, axis=1))), 1e-12)
    T = np.array([[s, 0.0, -s * c[0]], [0.0, s, -s * c[1]], [0.0, 0.0, 1.0]])
    return (x - c) * s, T


def essential_8pt(x1, x2):
    """Normalised 8-point essential matrix, x2^T E x1 = 0, projected to equal
    non-zero singular values."""
    n1, T1 = _hartley(x1)
    n2, T2 = _hartley(x2)
    h1 = np.concatenate([n1, np.ones((len(n1), 1))], axis=1)
    h2 = np.concatenate([n2, np.ones((len(n2), 1))], axis=1)
    A = (h2[:, :, None] * h1[:, None, :]).reshape(len(h1), 9)     # rows kron(h2, h1)
    E = T2.T @ np.linalg.svd(A, full_matrices=False)[2][-1].reshape(3, 3) @ T1
    U, sv, Vt = np.linalg.svd(E)
    m = 0.5 * (sv[0] + sv[1])
    return U @ np.diag([m, m, 0.0]) @ Vt


def relative_pose(E, x1, x2):
    """(R, t) of camera 2 relative to camera 1 = identity: the decomposition
    of E with the most points in front of both cameras (first on ties, in the
    order (W, +t), (W, -t), (W^T, +t), (W^T, -t))."""
    U, _, Vt = np.linalg.svd(E)
    if np.linalg.det(U) < 0:
        U = -U
    if np.linalg.det(Vt) < 0:
        Vt = -Vt
    W = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    best, best_votes = None, -1
    for R in (U @ W @ Vt, U @ W.T @ Vt):
        for t in (U[:, 2], -U[:, 2]):
            X = _ray_midpoints(np.eye(3), np.zeros(3), R, t, x1, x2)
            votes = int(np.count_nonzero((X[:, 2] > 0) & ((X @ R.T + t)[:, 2] > 0)))
            if votes > best_votes:
                best, best_votes = (R, t), votes
    return best


def two_view_init(tracks: list, n: int, intr0: CameraIntrinsics, min_shared: int = 30):
    """Poses and points from the frame pair with the largest median
    displacement among pairs sharing >= min_shared tracks; the other cameras
    are interpolated along the pair by frame index (clamped outside it).
    Returns (R (n,3,3), t (n,3), points) or None."""
    from scipy.spatial.transform import Rotation, Slerp
    seen = np.zeros((n, len(tracks)), dtype=bool)
    px = np.zeros((n, len(tracks), 2))
    for j, obs in enumerate(tracks):
        for fr, _, x, y in obs:
            seen[fr, j] = True
            px[fr, j] = (x, y)
    best = None
    for i in range(n):
        for j in range(i + 1, n):
            shared = np.flatnonzero(seen[i] & seen[j])
            if len(shared) < min_shared:
                continue
            disp = float(np.median(np.linalg.norm(px[j, shared] - px[i, shared], axis=1)))
            if best is None or disp > best[0]:
                best = (disp, i, j, shared)
    if best is None:
        return None
    _, ia, ib, shared = best
    pp = np.array([intr0.cx, intr0.cy])
    x1 = (px[ia, shared] - pp) / intr0.focal
    x2 = (px[ib, shared] - pp) / intr0.focal
    R, t = relative_pose(essential_8pt(x1, x2), x1, x2)
    interp = Slerp([float(ia), float(ib)], Rotation.from_matrix(np.stack([np.eye(3), R])))
    fc = np.clip(np.arange(n, dtype=np.float64), ia, ib)
    Rs = np.stack([interp(f).as_matrix() for f in fc])
    ts = ((fc - ia) / max(ib - ia, 1))[:, None] * t[None, :]
    X = _ray_midpoints(np.eye(3), np.zeros(3), R, t, x1, x2)
    front = X[:, 2] > 0
    depth = float(np.median(X[front, 2])) if front.any() else 1.0
    row = np.full(len(tracks), -1)
    row[shared] = np.arange(len(shared))
    pts = np.empty((len(tracks), 3))
    for j, obs in enumerate(tracks):
        r = row[j]
        if r >= 0 and front[r]:
            pts[j] = X[r]
        else:
            fr0, _, x0, y0 = obs[0]
            pts[j] = unproject(intr0, Pose.from_matrix(Rs[fr0], ts[fr0]), [[x0, y0]], [depth])[0]
    return Rs, ts, pts


# ---------------------------------------------------------------------------
# the device schedule


def _window_problem(tracks, n, intr, focal0, optimize_focal, init=None):
    """BaProblem dict of a window: observations track-major (point-major)."""
    lengths = np.array([len(o) for o in tracks])
    obs = np.array([(fr, x, y) for o in tracks for fr, _, x, y in o], dtype=np.float64).reshape(-1, 3)
    cam_idx = obs[:, 0].astype(np.int64)
    pt_idx = np.repeat(np.arange(len(tracks)), lengths)
    uv = np.ascontiguousarray(obs[:, 1:])
    if init is None:
        # the paper's start: coincident cameras, points at depth 1 along the
        # first observation's ray (identity pose: unproject is exact here)
        first = np.array([o[0][2:] for o in tracks], dtype=np.float64).reshape(-1, 2)
        pts = np.stack([(first[:, 0] - intr.cx) / focal0, (first[:, 1] - intr.cy) / focal0,
                        np.ones(len(tracks))], axis=1)
        R, t = np.stack([np.eye(3)] * n), np.zeros((n, 3))
    else:
        R, t, pts = init
    return dict(R=np.array(R, dtype=np.float64), t=np.array(t, dtype=np.float64), focal=float(focal0),
                cx=float(intr.cx), cy=float(intr.cy), points=np.array(pts, dtype=np.float64),
                cam_idx=cam_idx, pt_idx=pt_idx, uv=uv, fixed_cams=np.arange(n) == 0,
                optimize_focal=bool(optimize_focal), optimize_points=True)


def schedule_batch(problems: list, cfg: CaptureConfig, precision: str = "f64") -> list:
    """run_schedule (miniba.py:782-805) for a batch of problem dicts as one
    device sequence (mba_bootstrap_schedule). Returns per problem a dict with
    the refined R, t, focal, points, alive (points that keep observations),
    costs1 / costs2 traces, mean_err (second half) and n_kept."""
    import ctypes as ct

    from paper_2506_05558_b200 import _lib, solver
    from paper_2506_05558_b200._lib import ptr
    torch = _lib.torch_cuda()
    L = _lib.lib()
    hb = solver.pack_problems(problems)
    db = solver.to_device(hb)
    half = cfg.bootstrap_iters // 2
    p1 = solver.LmParams(lambda_init=cfg.lm_lambda_init, nu=cfg.lm_nu, delta=cfg.lm_huber_delta,
                         max_iters=half, precision=precision)
    p2 = solver.LmParams(lambda_init=cfg.lm_lambda_init, nu=cfg.lm_nu, delta=cfg.lm_huber_delta,
                         max_iters=cfg.bootstrap_iters - half, precision=precision)
    s1 = solver.Solution(db, p1.max_iters)
    s2 = solver.Solution(db, p2.max_iters)
    # the second half continues in place from the first half's state
    for k in ("R", "t", "focal", "points"):
        setattr(s2, k, getattr(s1, k))
    d, c1, o1 = solver.descriptors(db, p1, s1)
    _, c2, o2 = solver.descriptors(db, p2, s2)
    o2.R_in, o2.t_in, o2.focal_in, o2.points_in = o1.R_out, o1.t_out, o1.focal_out, o1.points_out
    B, K, P = db.n_problems, int(db.obs.shape[0]), int(db.points.numel() // 3)
    dev = db.obs.device
    obs2 = torch.empty_like(db.obs)
    lo2 = torch.empty((K, 2), dtype=torch.float32, device=dev) if db.obs_lo is not None else None
    off2 = torch.empty(B + 1, dtype=torch.int64, device=dev)
    n_kept = torch.empty(B, dtype=torch.int64, device=dev)
    alive = torch.empty(P, dtype=torch.uint8, device=dev)
    scale = torch.empty(B, dtype=torch.float64, device=dev)
    nbytes = int(L.mba_bootstrap_workspace_bytes(ct.byref(d), ct.byref(c1)))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _lib.check(L.mba_bootstrap_schedule(ct.byref(d), ct.byref(c1), ct.byref(c2), float(cfg.lm_mad_factor),
                                        ct.byref(o1), ct.byref(o2), ptr(obs2), ptr(lo2), ptr(off2),
                                        ptr(n_kept), ptr(alive), ptr(scale), ptr(ws), nbytes,
                                        _lib.stream_ptr()), "mba_bootstrap_schedule")
    R, t, f, X = (s1.R.cpu().numpy(), s1.t.cpu().numpy(), s1.focal.cpu().numpy(), s1.points.cpu().numpy())
    keep, alv = n_kept.cpu().numpy(), alive.cpu().numpy().astype(bool)
    st2 = s2.final_stats.cpu().numpy()
    n1, n2 = s1.n_iters.cpu().numpy(), s2.n_iters.cpu().numpy()
    c1h, c2h = s1.costs.cpu().numpy(), s2.costs.cpu().numpy()
    out = []
    for b in range(B):
        cs, ps = slice(hb.cam_off[b], hb.cam_off[b + 1]), slice(hb.pt_off[b], hb.pt_off[b + 1])
        out.append(dict(R=R[cs].copy(), t=t[cs].copy(), focal=float(f[b]), points=X[ps].copy(),
                        alive=alv[ps].copy(), n_kept=int(keep[b]),
                        costs1=c1h[b, :n1[b] + 1].copy(), costs2=c2h[b, :n2[b] + 1].copy(),
                        mean_err=float(st2[b, 1] / max(st2[b, 3], 1.0))))
    return out


def _degenerate(focal, width, optimize_focal):
    from .miniba import FOCAL_BOUNDS
    return optimize_focal and not (FOCAL_BOUNDS[0] * width <= focal <= FOCAL_BOUNDS[1] * width)


def _anchor_first_camera(res):
    """Re-express a solution in the frame of its first camera (the spec gauge
    after a two-view rescue, miniba.py:831-838)."""
    R0, t0 = res["R"][0].copy(), res["t"][0].copy()
    res["points"] = res["points"] @ R0.T + t0
    for c in range(len(res["R"])):
        Rc = res["R"][c] @ R0.T
        res["t"][c] = res["t"][c] - Rc @ t0
        res["R"][c] = Rc


def bootstrap_batch(windows: list, intrs: list, cfg: CaptureConfig, matcher=None,
                    optimize_focal: bool = True, precision: str = "f64") -> list:
    """Bootstrap many independent windows: one device schedule for all of
    them, then one more for the windows that need the two-view rescue.
    Returns per window (poses, intrinsics, TrackTable, info) or the
    BootstrapFailure instance that window raised."""
    from . import miniba as M
    metas, probs = [], []
    for features, intr in zip(windows, intrs):
        n = len(features)
        if n > 64:   # the device gauge step holds up to 64 camera centres per window
            raise ValueError(f"bootstrap window of {n} frames (at most 64)")
        tracks = build_tracks_device(features) if matcher is None else build_tracks(features, matcher)
        if len(tracks) < M.MIN_BOOTSTRAP_TRACKS:
            metas.append(M.BootstrapFailure(f"{len(tracks)} tracks < {M.MIN_BOOTSTRAP_TRACKS}"))
            continue
        # >= 3-observation tracks carry redundancy; fall back to all tracks
        long_tracks = [o for o in tracks if len(o) >= 3]
        use = long_tracks if len(long_tracks) >= M.MIN_BOOTSTRAP_TRACKS else tracks
        focal0 = cfg.focal_init_factor * intr.width if optimize_focal else intr.focal
        metas.append((use, n, intr, focal0))
        probs.append(_window_problem(use, n, intr, focal0, optimize_focal))
    live = [i for i, m in enumerate(metas) if not isinstance(m, Exception)]
    results = dict(zip(live, schedule_batch(probs, cfg, precision))) if probs else {}
    rescued = {}
    redo, redo_probs = [], []
    for i in live:
        use, n, intr, focal0 = metas[i]
        if results[i]["n_kept"] == 0:
            metas[i] = M.BootstrapFailure("robust filter removed every observation")
            continue
        if _degenerate(results[i]["focal"], intr.width, optimize_focal):
            intr0 = CameraIntrinsics(focal0, intr.cx, intr.cy, intr.width, intr.height)
            init = two_view_init(use, n, intr0)
            if init is not None:
                redo.append(i)
                redo_probs.append(_window_problem(use, n, intr, focal0, optimize_focal, init))
    if redo_probs:
        for i, res in zip(redo, schedule_batch(redo_probs, cfg, precision)):
            if res["n_kept"] == 0:
                metas[i] = M.BootstrapFailure("robust filter removed every observation")
                continue
            _anchor_first_camera(res)
            results[i] = res
            rescued[i] = True
    out = []
    for i, m in enumerate(metas):
        if isinstance(m, Exception):
            out.append(m)
            continue
        use, n, intr, focal0 = m
        res = results[i]
        if _degenerate(res["focal"], intr.width, optimize_focal):
            lo, hi = M.FOCAL_BOUNDS
            out.append(M.BootstrapFailure(f"degenerate solution: focal {res['focal']:.1f} outside "
                                          f"[{lo}, {hi}] x width {intr.width}"))
            continue
        poses = [Pose.from_matrix(res["R"][c], res["t"][c]) for c in range(n)]
        intr_out = CameraIntrinsics(res["focal"], intr.cx, intr.cy, intr.width, intr.height)
        table = TrackTable(cfg.n_obs_max)
        surviving = np.flatnonzero(res["alive"])
        for j in surviving:
            table.new_track(use[j], point=res["points"][j].copy())
        info = dict(costs=np.concatenate([res["costs1"], res["costs2"]]), mean_err=res["mean_err"],
                    n_tracks=len(surviving), focal=res["focal"], rescued=bool(rescued.get(i, False)))
        out.append((poses, intr_out, table, info))
    return out


def bootstrap(features: list, intr: CameraIntrinsics, cfg: CaptureConfig, matcher=None,
              optimize_focal: bool = True):
    """The reference's bootstrap (miniba.py:729-854): joint pose / point /
    focal estimation for the first cfg.n_init frames. matcher=None uses the
    default matcher (device matching of every frame pair + flow filter).
    Returns (poses, intrinsics, TrackTable, info); raises BootstrapFailure."""
    res = bootstrap_batch([features], [intr], cfg, matcher=matcher, optimize_focal=optimize_focal)[0]
    if isinstance(res, Exception):
        raise res
    return res
