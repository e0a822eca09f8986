"""Seeded synthetic mini-BA workloads, vectorised over
a batch of independent problems.

The generator follows the reference's oracle scene conventions
(`synthetic.py:272-298`: cameras on a 70 deg arc of radius 2 looking at the
origin, points uniform in a ball of radius 0.6, f = 520, 640x480) and adds the
track model of SURVEY 8d: each point is a track of L ~ U{2..min(6,n)}
consecutive frames starting at s ~ U{0..n-L}; tracks are drawn until the
problem holds K observations. Initial values: camera 0 fixed at ground truth,
others rotated by exp(N(0, 1 deg)) and translated by 1% |t| N(0,1); focal x1.02;
points + N(0, 0.01). Every float input is rounded to fp32 so the device and the
oracle see identical, fp32-representable values.

Observations come out point-major (track-major, cameras ascending inside a
track), the order the device solver consumes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

WIDTH, HEIGHT, F_TRUE = 640, 480, 520.0
CHUNK = 256                      # problems per RNG stream (at most)


def chunk_size(K):
    """Problems per RNG stream: up to 256, about 1M observations per chunk."""
    return int(min(CHUNK, max(1, (1 << 20) // max(int(K), 1))))


@dataclass
class Batch:
    """Flat packed batch of B problems (host numpy)."""
    n_cams: np.ndarray      # (B,) int32
    cam_off: np.ndarray     # (B+1,) int64 offsets into R/t rows
    pt_off: np.ndarray      # (B+1,) int64 offsets into points rows
    obs_off: np.ndarray     # (B+1,) int64 offsets into observation rows
    R: np.ndarray           # (sum n, 3, 3) f64 initial rotations
    t: np.ndarray           # (sum n, 3) f64
    focal: np.ndarray       # (B,) f64
    cx: np.ndarray          # (B,) f64
    cy: np.ndarray          # (B,) f64
    points: np.ndarray      # (sum P, 3) f64
    cam: np.ndarray         # (sum K,) int32 local camera index
    pt: np.ndarray          # (sum K,) int32 local point index
    uv: np.ndarray          # (sum K, 2) f64
    fixed: np.ndarray       # (sum n,) bool
    optimize_focal: bool = True
    optimize_points: bool = True
    gt_R: np.ndarray | None = None
    gt_t: np.ndarray | None = None
    gt_points: np.ndarray | None = None

    @property
    def n_problems(self):
        return len(self.n_cams)

    def problem(self, b):
        """Problem b as the dict layout the oracle uses (BaProblem fields)."""
        c0, c1 = self.cam_off[b], self.cam_off[b + 1]
        p0, p1 = self.pt_off[b], self.pt_off[b + 1]
        o0, o1 = self.obs_off[b], self.obs_off[b + 1]
        return dict(R=self.R[c0:c1].copy(), t=self.t[c0:c1].copy(),
                    focal=float(self.focal[b]), cx=float(self.cx[b]), cy=float(self.cy[b]),
                    points=self.points[p0:p1].copy(),
                    cam_idx=self.cam[o0:o1].astype(np.int64),
                    pt_idx=self.pt[o0:o1].astype(np.int64),
                    uv=self.uv[o0:o1].copy(), fixed_cams=self.fixed[c0:c1].copy(),
                    optimize_focal=self.optimize_focal,
                    optimize_points=self.optimize_points)


def _f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def _rodrigues_batch(w):
    th = np.linalg.norm(w, axis=-1, keepdims=True)
    k = w / np.maximum(th, 1e-300)
    Km = np.zeros(w.shape[:-1] + (3, 3))
    Km[..., 0, 1], Km[..., 0, 2] = -k[..., 2], k[..., 1]
    Km[..., 1, 0], Km[..., 1, 2] = k[..., 2], -k[..., 0]
    Km[..., 2, 0], Km[..., 2, 1] = -k[..., 1], k[..., 0]
    th = th[..., None]
    return np.eye(3) + np.sin(th) * Km + (1.0 - np.cos(th)) * (Km @ Km)


def _arc_cameras(rng, nb, n):
    """(nb, n) look-at cameras on a 70 deg arc of radius 2 (synthetic.py:272-281)."""
    ang = np.deg2rad(70.0) * np.arange(n) / max(n - 1, 1)
    c = np.empty((nb, n, 3))
    c[..., 0] = 2.0 * np.cos(ang)
    c[..., 1] = 2.0 * np.sin(ang)
    c[..., 2] = 0.3 + 0.1 * rng.standard_normal((nb, n))
    target = 0.02 * rng.standard_normal((nb, n, 3))
    z = target - c
    z /= np.linalg.norm(z, axis=-1, keepdims=True)
    x = np.cross(z, np.array([0.0, 0.0, 1.0]))
    x /= np.linalg.norm(x, axis=-1, keepdims=True)
    y = np.cross(z, x)
    R = np.stack([x, y, z], axis=-2)
    t = -np.einsum("bnij,bnj->bni", R, c)
    return R, t


def _chunk(rng, nb, n, K, noise_px, outlier_frac):
    Rg, tg = _arc_cameras(rng, nb, n)
    lmax = min(6, n)
    cap = K // 2 + 1
    L = rng.integers(2, lmax + 1, size=(nb, cap))
    csum = np.cumsum(L, axis=1)
    keep = csum <= K
    P = keep.sum(axis=1)
    u_start = rng.random((nb, cap))
    r_ball = 0.6 * rng.random((nb, cap)) ** (1.0 / 3.0)
    dirs = rng.standard_normal((nb, cap, 3))
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    X_all = dirs * r_ball[..., None]
    # flatten kept tracks (problem-major, then track order)
    bi, ji = np.nonzero(keep)
    Lk = L[bi, ji]
    sk = np.floor(u_start[bi, ji] * (n - Lk + 1)).astype(np.int64)
    Xk = X_all[bi, ji]
    n_obs = int(Lk.sum())
    tr = np.repeat(np.arange(len(Lk)), Lk)
    first = np.cumsum(Lk) - Lk
    pos = np.arange(n_obs) - first[tr]
    cam = sk[tr] + pos
    ob = bi[tr]
    pc = np.einsum("kij,kj->ki", Rg[ob, cam], Xk[tr]) + tg[ob, cam]
    uv = np.stack([F_TRUE * pc[:, 0] / pc[:, 2] + WIDTH / 2.0,
                   F_TRUE * pc[:, 1] / pc[:, 2] + HEIGHT / 2.0], axis=1)
    uv += noise_px * rng.standard_normal(uv.shape)
    if outlier_frac > 0:
        m = rng.random(n_obs) < outlier_frac
        uv[m] = rng.random((int(m.sum()), 2)) * [WIDTH, HEIGHT]
    # initial values
    wrot = np.deg2rad(1.0) * rng.standard_normal((nb, n, 3))
    R0 = _rodrigues_batch(wrot) @ Rg
    tn = np.linalg.norm(tg, axis=-1, keepdims=True)
    t0 = tg + 0.01 * tn * rng.standard_normal((nb, n, 3))
    R0[:, 0], t0[:, 0] = Rg[:, 0], tg[:, 0]
    X0 = Xk + 0.01 * rng.standard_normal(Xk.shape)
    # local point index within the problem
    p_first = np.cumsum(P) - P
    track_global = np.arange(len(Lk))
    pt_local = track_global - p_first[bi]
    return dict(R=Rg, t=tg, R0=R0, t0=t0, P=P, Xg=Xk, X0=X0,
                cam=cam.astype(np.int32), pt=pt_local[tr].astype(np.int32),
                uv=uv, K=np.bincount(ob, minlength=nb))


def _chunk_job(args):
    seed, ci, nb, n_cams, K, noise_px, outlier_frac = args
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 0xBA8D, ci]))
    return _chunk(rng, nb, n_cams, K, noise_px, outlier_frac)


def make_batch(n_problems, n_cams=8, K=2000, seed=0, noise_px=0.5, outlier_frac=0.0, first=0,
               workers=1):
    """Generate problems [first, first + n_problems) of the seeded stream
    (SURVEY 8d). Problem i depends only on (seed, i), so any contiguous shard
    can be generated independently. `workers` > 1 generates chunks in
    parallel processes."""
    ch = chunk_size(K)
    c_lo, c_hi = first // ch, (first + n_problems + ch - 1) // ch
    jobs = [(seed, ci, ch, n_cams, K, noise_px, outlier_frac) for ci in range(c_lo, c_hi)]
    if workers > 1 and len(jobs) > 1:
        from concurrent.futures import ProcessPoolExecutor
        with ProcessPoolExecutor(max_workers=min(workers, len(jobs))) as ex:
            parts = list(ex.map(_chunk_job, jobs))
    else:
        parts = [_chunk_job(j) for j in jobs]
    lo = first - c_lo * ch
    if lo or (c_hi - c_lo) * ch != n_problems:
        parts = _slice_parts(parts, lo, n_problems)
    cat = lambda k: np.concatenate([p[k] for p in parts])
    P = cat("P")
    Kb = cat("K")
    B = n_problems
    n = np.full(B, n_cams, dtype=np.int32)
    off = lambda v: np.concatenate([[0], np.cumsum(v)]).astype(np.int64)
    fixed = np.zeros((B, n_cams), dtype=bool)
    fixed[:, 0] = True
    return Batch(
        n_cams=n, cam_off=off(n), pt_off=off(P), obs_off=off(Kb),
        R=_f32(cat("R0").reshape(-1, 3, 3)), t=_f32(cat("t0").reshape(-1, 3)),
        focal=np.full(B, _f32(1.02 * F_TRUE)), cx=np.full(B, WIDTH / 2.0),
        cy=np.full(B, HEIGHT / 2.0), points=_f32(cat("X0")),
        cam=cat("cam"), pt=cat("pt"), uv=_f32(cat("uv")), fixed=fixed.reshape(-1),
        gt_R=cat("R").reshape(-1, 3, 3), gt_t=cat("t").reshape(-1, 3),
        gt_points=cat("Xg"))


def _slice_parts(parts, lo, count):
    """Keep problems [lo, lo + count) of the concatenated chunk list."""
    keys_b = ("R", "t", "R0", "t0")          # (nb, n, ...)
    out = []
    base = 0
    for p in parts:
        nb = len(p["P"])
        a, b = max(lo - base, 0), min(lo + count - base, nb)
        base += nb
        if a >= b:
            continue
        P, Kb = p["P"], p["K"]
        p_first = np.concatenate([[0], np.cumsum(P)])
        o_first = np.concatenate([[0], np.cumsum(Kb)])
        q = {k: p[k][a:b] for k in keys_b}
        q["P"], q["K"] = P[a:b], Kb[a:b]
        for k in ("Xg", "X0"):
            q[k] = p[k][p_first[a]:p_first[b]]
        for k in ("cam", "pt", "uv"):
            q[k] = p[k][o_first[a]:o_first[b]]
        out.append(q)
    return out


# BASELINE.json configs
CONFIGS = {
    1: dict(n_problems=1, n_cams=5, K=1000, loss="huber", max_iters=20,
            desc="smoke-like: 5-frame window, ~1k observations, fixed 20 LM iterations"),
    2: dict(n_problems=1, n_cams=8, K=20000, loss="huber", max_iters=200,
            desc="single mini-BA, 8 frames, K=20k, Huber"),
    3: dict(n_problems=1024, n_cams=8, K=20000, loss="huber", max_iters=200,
            desc="batched 1,024 x (8 frames, K=20k)"),
    4: dict(n_problems=65536, n_cams=8, K=2000, loss="huber", max_iters=200,
            desc="batched 65,536 x (8 frames, K=2k)"),
    5: dict(n_problems=1, n_cams=32, K=200000, loss="cauchy", max_iters=50,
            outlier_frac=0.2, desc="stress: 32 frames, K=200k, 20% outliers, Cauchy, 50 iters"),
}
