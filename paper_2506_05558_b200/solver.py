"""Host side of the batched mini-BA: packing into the C-ABI layout, device
buffers, the mba_solve call and unpacking of per-problem results.

Layout in HBM (include/miniba.h): problems back to back; observations as
16-byte records {float u, float v, int32 cam, int32 pt} sorted point-major
inside each problem (+ an optional float2 low-order uv correction so the
residual sees the exact float64 pixel); cameras as float64 R (9) and t (3);
points as float64 xyz.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import MbaBatchDesc, MbaLmConfig, MbaOutputs, ptr


@dataclass
class HostBatch:
    """A batch in C-ABI layout, host numpy (optionally pinned via torch)."""
    cam_off: np.ndarray
    pt_off: np.ndarray
    obs_off: np.ndarray
    obs: np.ndarray          # (K, 4) float32 view of MbaObs records
    obs_lo: np.ndarray | None
    fixed: np.ndarray        # uint8 per camera
    cx: np.ndarray
    cy: np.ndarray
    flags: np.ndarray        # uint8 per problem
    R: np.ndarray            # (n, 3, 3) f64
    t: np.ndarray
    focal: np.ndarray
    points: np.ndarray
    max_pairs: int = 0
    max_track: int = 0

    @property
    def n_problems(self):
        return len(self.cx)

    @property
    def max_cams(self):
        return int(np.max(np.diff(self.cam_off))) if self.n_problems else 0

    @property
    def max_obs(self):
        return int(np.max(np.diff(self.obs_off))) if self.n_problems else 0

    @property
    def max_points(self):
        return int(np.max(np.diff(self.pt_off))) if self.n_problems else 0


def _track_stats(obs_off, pt_off, pt):
    """(max over problems of sum_p m_p (m_p + 1) / 2, max m_p), m_p = observations of point p."""
    n_obs = np.diff(obs_off)
    gpt = np.repeat(pt_off[:-1], n_obs) + pt
    m = np.bincount(gpt, minlength=int(pt_off[-1])).astype(np.int64)
    per_pt = m * (m + 1) // 2
    prob = np.repeat(np.arange(len(n_obs)), np.diff(pt_off))
    if not len(n_obs):
        return 0, 0
    return (int(np.bincount(prob, weights=per_pt, minlength=len(n_obs)).max()),
            int(m.max()) if len(m) else 0)


def _records(uv, cam, pt):
    rec = np.empty((len(cam), 4), dtype=np.float32)
    uv32 = uv.astype(np.float32)
    rec[:, 0:2] = uv32
    rec.view(np.int32)[:, 2] = cam
    rec.view(np.int32)[:, 3] = pt
    lo = (uv - uv32.astype(np.float64)).astype(np.float32)
    return rec, lo


def pack_problems(problems) -> HostBatch:
    """Pack BaProblem-like objects or dicts (R,t,focal,cx,cy,points,cam_idx,
    pt_idx,uv,fixed_cams,optimize_focal,optimize_points). Observations are
    stably sorted point-major per problem."""
    get = (lambda p, k: p[k]) if problems and isinstance(problems[0], dict) else getattr
    Rs, ts, pts, recs, los, fixed = [], [], [], [], [], []
    n_c, n_p, n_o, cx, cy, fl, foc = [], [], [], [], [], [], []
    for p in problems:
        R = np.asarray(get(p, "R"), dtype=np.float64).reshape(-1, 3, 3)
        t = np.asarray(get(p, "t"), dtype=np.float64).reshape(-1, 3)
        X = np.asarray(get(p, "points"), dtype=np.float64).reshape(-1, 3)
        cam = np.asarray(get(p, "cam_idx")).reshape(-1)
        pt = np.asarray(get(p, "pt_idx")).reshape(-1)
        uv = np.asarray(get(p, "uv"), dtype=np.float64).reshape(-1, 2)
        if len(uv) == 0:
            raise ValueError("problem has no residuals")
        if not (len(cam) == len(pt) == len(uv)):
            raise ValueError("cam_idx, pt_idx and uv lengths differ")
        n = len(R)
        if cam.min() < 0 or cam.max() >= n or pt.min() < 0 or pt.max() >= len(X):
            raise IndexError("observation index out of range")
        if np.any(pt[1:] < pt[:-1]):
            order = np.argsort(pt, kind="stable")
            cam, pt, uv = cam[order], pt[order], uv[order]
        rec, lo = _records(uv, cam.astype(np.int32), pt.astype(np.int32))
        Rs.append(R); ts.append(t); pts.append(X); recs.append(rec); los.append(lo)
        fc = np.asarray(get(p, "fixed_cams"), dtype=bool).reshape(-1)
        if len(fc) != n:   # a wrong length would shift every later problem's flags
            raise ValueError(f"fixed_cams has {len(fc)} entries for {n} cameras")
        fixed.append(fc.astype(np.uint8))
        n_c.append(n); n_p.append(len(X)); n_o.append(len(uv))
        cx.append(float(get(p, "cx"))); cy.append(float(get(p, "cy"))); foc.append(float(get(p, "focal")))
        of = bool(get(p, "optimize_focal"))
        try:
            op = bool(get(p, "optimize_points"))
        except (KeyError, AttributeError):
            op = True
        fl.append((1 if of else 0) | (2 if op else 0))
    off = lambda v: np.concatenate([[0], np.cumsum(v)]).astype(np.int64)
    lo = np.concatenate(los)
    obs = np.concatenate(recs)
    pt_off, obs_off = off(n_p), off(n_o)
    return HostBatch(cam_off=off(n_c), pt_off=pt_off, obs_off=obs_off, obs=obs,
                     obs_lo=lo if np.any(lo) else None, fixed=np.concatenate(fixed),
                     cx=np.array(cx), cy=np.array(cy), flags=np.array(fl, dtype=np.uint8),
                     R=np.concatenate(Rs), t=np.concatenate(ts), focal=np.array(foc),
                     points=np.concatenate(pts),
                     **dict(zip(("max_pairs", "max_track"),
                                _track_stats(obs_off, pt_off, obs.view(np.int32)[:, 3]))))


def pack_synth(b) -> HostBatch:
    """Pack a synth.Batch (already point-major, fp32-representable uv)."""
    rec, lo = _records(b.uv, b.cam, b.pt)
    flags = np.full(b.n_problems, (1 if b.optimize_focal else 0) | (2 if b.optimize_points else 0),
                    dtype=np.uint8)
    return HostBatch(cam_off=b.cam_off, pt_off=b.pt_off, obs_off=b.obs_off, obs=rec,
                     obs_lo=lo if np.any(lo) else None, fixed=b.fixed.astype(np.uint8), cx=b.cx,
                     cy=b.cy, flags=flags, R=b.R, t=b.t, focal=b.focal, points=b.points,
                     **dict(zip(("max_pairs", "max_track"), _track_stats(b.obs_off, b.pt_off, b.pt))))


@dataclass
class DeviceBatch:
    n_problems: int
    max_cams: int
    max_obs: int
    max_points: int
    max_pairs: int
    max_track: int
    cam_off: object
    pt_off: object
    obs_off: object
    obs: object
    obs_lo: object
    fixed: object
    cx: object
    cy: object
    flags: object
    R: object
    t: object
    focal: object
    points: object
    h2d_bytes: int = 0


_INPUT_FIELDS = ("cam_off", "pt_off", "obs_off", "obs", "obs_lo", "fixed", "cx", "cy", "flags",
                 "R", "t", "focal", "points")


def pin(hb: HostBatch):
    """Host tensors (pinned) for every input field, for timed H2D copies."""
    torch = _lib.torch_cuda()
    out = {}
    for k in _INPUT_FIELDS:
        a = getattr(hb, k)
        out[k] = None if a is None else torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    return out


def to_device(hb: HostBatch, device=None, pinned=None) -> DeviceBatch:
    torch = _lib.torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    src = pinned if pinned is not None else {
        k: (None if getattr(hb, k) is None else torch.from_numpy(np.ascontiguousarray(getattr(hb, k))))
        for k in _INPUT_FIELDS}
    d = {}
    nbytes = 0
    for k in _INPUT_FIELDS:
        a = src[k]
        if a is None:
            d[k] = None
            continue
        d[k] = a.to(dev, non_blocking=True)
        nbytes += a.numel() * a.element_size()
    return DeviceBatch(n_problems=hb.n_problems, max_cams=hb.max_cams, max_obs=hb.max_obs,
                       max_points=hb.max_points, max_pairs=hb.max_pairs, max_track=hb.max_track,
                       h2d_bytes=nbytes, **d)


# LmParams.kernel -> MbaLmConfig.ctas_per_problem (0: planner; < 0: forced path)
KERNELS = {"auto": 0, "cta": -2, "grid": -4, "v4": -9}


@dataclass
class LmParams:
    lambda_init: float = 1e-5
    nu: float = 2.0
    delta: float = 2.0
    max_iters: int = 200
    loss: str = "huber"
    precision: str = "f64"
    fail_at: tuple = ()
    kernel: str = "auto"      # "auto" | "v4" (cluster-resident) | "cta" (CTA per problem)
    #                           | "grid" (whole GPU per problem)

    @staticmethod
    def from_cfg(cfg, **over):
        p = LmParams(lambda_init=cfg.lambda_init, nu=cfg.nu, delta=cfg.huber_delta,
                     max_iters=cfg.max_iters, loss=getattr(cfg, "loss", "huber"),
                     precision=getattr(cfg, "precision", "f64"))
        for k, v in over.items():
            setattr(p, k, v)
        return p


class Solution:
    """Device-resident outputs of one mba_solve call."""

    def __init__(self, db: DeviceBatch, max_iters: int):
        torch = _lib.torch_cuda()
        dev = db.obs.device
        B = db.n_problems
        f64 = dict(dtype=torch.float64, device=dev)
        self.R = torch.empty_like(db.R)
        self.t = torch.empty_like(db.t)
        self.focal = torch.empty_like(db.focal)
        self.points = torch.empty_like(db.points)
        self.costs = torch.zeros((B, max_iters + 1), **f64)
        self.lambdas = torch.zeros((B, max(max_iters, 1)), **f64)
        self.accepted = torch.zeros((B, max(max_iters, 1)), dtype=torch.uint8, device=dev)
        self.evals = torch.zeros((B, max(max_iters, 1)), dtype=torch.uint8, device=dev)
        self.n_iters = torch.zeros(B, dtype=torch.int32, device=dev)
        self.status = torch.zeros(B, dtype=torch.int32, device=dev)
        self.final_stats = torch.zeros((B, 4), **f64)
        self.max_iters = max_iters

    def summary_tensors(self):
        return (self.n_iters, self.status, self.final_stats)


_WS = {}


def _workspace(nbytes, device):
    torch = _lib.torch_cuda()
    key = (device.index,)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def descriptors(db: DeviceBatch, prm: LmParams, sol: Solution):
    d = MbaBatchDesc(n_problems=db.n_problems, max_cams=db.max_cams, max_obs=db.max_obs,
                     max_points=db.max_points, max_pairs=db.max_pairs, max_track=db.max_track, cam_off=ptr(db.cam_off), pt_off=ptr(db.pt_off),
                     obs_off=ptr(db.obs_off), obs=ptr(db.obs), obs_lo=ptr(db.obs_lo),
                     fixed=ptr(db.fixed), cx=ptr(db.cx), cy=ptr(db.cy), flags=ptr(db.flags))
    c = MbaLmConfig(lambda_init=prm.lambda_init, nu=prm.nu, delta=prm.delta,
                    max_iters=prm.max_iters, loss=_lib.LOSS[prm.loss],
                    precision=_lib.PRECISION[prm.precision],
                    ctas_per_problem=KERNELS[prm.kernel],
                    fail_iters_mask=sum(1 << int(i) for i in prm.fail_at if 0 <= int(i) < 64))
    o = MbaOutputs(R_in=ptr(db.R), t_in=ptr(db.t), focal_in=ptr(db.focal), points_in=ptr(db.points),
                   R_out=ptr(sol.R), t_out=ptr(sol.t), focal_out=ptr(sol.focal),
                   points_out=ptr(sol.points), costs=ptr(sol.costs), lambdas=ptr(sol.lambdas),
                   accepted=ptr(sol.accepted), evals=ptr(sol.evals), n_iters=ptr(sol.n_iters),
                   status=ptr(sol.status), final_stats=ptr(sol.final_stats))
    return d, c, o


def workspace_bytes(db: DeviceBatch, prm: LmParams) -> int:
    """Device workspace mba_solve needs for this batch (mba_workspace_bytes)."""
    d, c = _desc(db, prm)
    return int(_lib.lib().mba_workspace_bytes(ct.byref(d), ct.byref(c)))


def solve(db: DeviceBatch, prm: LmParams, sol: Solution | None = None, ws=None) -> Solution:
    """Enqueue mba_solve on the current stream (asynchronous). `ws`: a caller-
    owned uint8 workspace (needed when solves run concurrently on several
    streams); default: one shared per-device workspace."""
    L = _lib.lib()
    if sol is None:
        sol = Solution(db, prm.max_iters)
    d, c, o = descriptors(db, prm, sol)
    nbytes = L.mba_workspace_bytes(ct.byref(d), ct.byref(c))
    if ws is None or ws.numel() < nbytes:
        ws = _workspace(nbytes, db.obs.device)
    rc = L.mba_solve(ct.byref(d), ct.byref(c), ct.byref(o), ptr(ws), ws.numel(), _lib.stream_ptr())
    _lib.check(rc, "mba_solve")
    return sol


def _desc(db, prm):
    sol = Solution.__new__(Solution)
    for k in ("R", "t", "focal", "points", "costs", "lambdas", "accepted", "evals", "n_iters", "status",
              "final_stats"):
        setattr(sol, k, None)
    d, c, _ = descriptors(db, prm, sol)
    return d, c


def plan(db: DeviceBatch, prm: LmParams) -> int:
    """Device path mba_solve takes (mba_solve_plan): cluster size R > 0 of the
    cluster-resident kernel, or -2 CTA kernel / -4 cooperative grid kernel."""
    d, c = _desc(db, prm)
    return int(_lib.lib().mba_solve_plan(ct.byref(d), ct.byref(c)))


def launches(db: DeviceBatch, prm: LmParams) -> int:
    """Kernel launches per mba_solve call (mba_solve_launches)."""
    d, c = _desc(db, prm)
    return int(_lib.lib().mba_solve_launches(ct.byref(d), ct.byref(c)))


def fetch(sol: Solution, b: int = 0) -> dict:
    """Copy problem b's results to host in the lm_solve return layout."""
    n = int(sol.n_iters[b].item())
    st = sol.final_stats[b].cpu().numpy()
    K = max(st[3], 1.0)
    return dict(costs=sol.costs[b, :n + 1].cpu().numpy(),
                accepted=sol.accepted[b, :n].cpu().numpy().astype(bool),
                lambdas=sol.lambdas[b, :n].cpu().numpy(),
                evals=sol.evals[b, :n].cpu().numpy().astype(np.int32),
                final_rms=float(np.sqrt(st[2] / K)), mean_err=float(st[1] / K),
                status=int(sol.status[b].item()))
