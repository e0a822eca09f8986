"""End-to-end batched solve of a list of BaProblem objects (the engine behind
`gsrecon.miniba.lm_solve_batch`).

The reference's unit of work is one `BaProblem` (miniba.py:65-83) solved in
place by `lm_solve` (miniba.py:223-296). A batch of registration windows or
hypotheses is a Python list of such objects, so the end-to-end path is:

    list of BaProblem --(native walk + threaded gather: _mba_host.Batch)-->
    pinned upload buffer --(H2D, copy stream)--> device raw arrays
    --(mba_pack_obs: stable point-major sort + 16-byte records)-->
    --(mba_solve: the whole LM loop on device)--> solution
    --(D2H, read-back stream)--> pinned --(threaded in-place write-back)-->
    the callers' R / t / points arrays (+ focal rebound), lazy info dicts.

The batch is cut into chunks that flow through a four-slot ring, so the
host walk / gather of chunk i+1 and the write-back of chunk i-1 overlap the
device work of chunk i, and consecutive chunk solves alternate between two
compute streams (the next chunk's problems fill the SMs the previous chunk's
tail leaves idle).
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

from . import _lib
from ._lib import MbaBatchDesc, MbaLmConfig, MbaOutputs, ptr

_HOST = None


def host_module():
    """The native host extension (paper_2506_05558_b200/_mba_host*.so); no
    Python fallback, like the device library."""
    global _HOST
    if _HOST is None:
        try:
            from . import _mba_host
        except ImportError as e:   # pragma: no cover - build problem
            raise RuntimeError("paper_2506_05558_b200/_mba_host is not built: run "
                               "`python -c 'import __graft_entry__ as g; g.build()'`") from e
        _HOST = _mba_host
    return _HOST


def default_threads():
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:   # pragma: no cover
        n = os.cpu_count() or 1
    return max(1, min(16, n))


# upload regions: (name, bytes per camera, per point, per observation, per problem, +1 row)
_REGIONS = (("cam_off", 0, 0, 0, 8, 8), ("pt_off", 0, 0, 0, 8, 8), ("obs_off", 0, 0, 0, 8, 8),
            ("cx", 0, 0, 0, 8, 0), ("cy", 0, 0, 0, 8, 0), ("focal", 0, 0, 0, 8, 0),
            ("R", 72, 0, 0, 0, 0), ("t", 24, 0, 0, 0, 0), ("points", 0, 24, 0, 0, 0),
            ("uv", 0, 0, 8, 0, 0), ("cam", 0, 0, 4, 0, 0), ("pt", 0, 0, 4, 0, 0),
            ("fixed", 1, 0, 0, 0, 0), ("flags", 0, 0, 0, 1, 0), ("uv_lo", 0, 0, 8, 0, 0))


def layout(n_cams, n_pts, n_obs, m):
    """Byte offsets (16-aligned) of the upload regions for a chunk with the
    given totals, and the total size."""
    off, pos = {}, 0
    for name, pc, pp, po, pb, extra in _REGIONS:
        off[name] = pos
        pos += (pc * n_cams + pp * n_pts + po * n_obs + pb * m + extra + 15) & ~15
    # the trailing low-order uv stream is uploaded only when a chunk needs it
    return off, pos


class BatchResult:
    """Per-problem LM info of a batched solve, materialised lazily: item b is
    the dict `lm_solve` returns (costs, accepted, lambdas, final_rms, mean_err;
    plus evals and status), miniba.py:294-296. The traces are held ragged
    (only each problem's n_iters entries, as the device packed them)."""

    def __init__(self, B, max_iters):
        self.max_iters = max_iters
        self.n_iters = np.zeros(B, np.int32)
        self.status = np.zeros(B, np.int32)
        self.final_stats = np.zeros((B, 4))
        self._where = np.full(B, -1, np.int32)   # stored chunk of each problem
        self._pos = np.zeros(B, np.int32)        # its row inside that chunk
        self._chunks = []       # (off, costs, lambdas, accepted, evals)
        self._override = {}

    def add_chunk(self, index, off, costs, lambdas, accepted, evals):
        """Packed traces of the problems `index` (global indices, chunk order)."""
        self._where[index] = len(self._chunks)
        self._pos[index] = np.arange(len(index), dtype=np.int32)
        self._chunks.append((off, costs, lambdas, accepted, evals))

    def __len__(self):
        return len(self.n_iters)

    def __getitem__(self, b):
        if isinstance(b, slice):
            return [self[i] for i in range(*b.indices(len(self)))]
        if b < 0:
            b += len(self)
        if not 0 <= b < len(self):
            raise IndexError(b)
        if b in self._override:
            return dict(self._override[b])
        off, c, lam, acc, ev = self._chunks[self._where[b]]
        j = int(self._pos[b])
        o0, o1 = int(off[j]), int(off[j + 1])
        st = self.final_stats[b]
        K = max(st[3], 1.0)
        return dict(costs=c[o0 + j:o1 + j + 1].copy(), accepted=acc[o0:o1].astype(bool),
                    lambdas=lam[o0:o1].copy(), final_rms=float(np.sqrt(st[2] / K)),
                    mean_err=float(st[1] / K), evals=ev[o0:o1].astype(np.int32),
                    status=int(self.status[b]))

    def __iter__(self):
        for b in range(len(self)):
            yield self[b]

    def set(self, b, info):
        """Store problem b's info dict (problems solved outside the batch)."""
        d = dict(info)
        d.setdefault("evals", np.zeros(len(d["accepted"]), np.int32))
        d.setdefault("status", -3)
        self._override[b] = d
        self.n_iters[b] = len(d["accepted"])
        self.status[b] = d["status"]
        self.final_stats[b] = (d["costs"][-1], d["mean_err"], d["final_rms"] ** 2, 1.0)


# fixed-size outputs read back per chunk; the traces are packed on the device
# first (mba_compact_traces) and read back ragged
_OUT = ("R", "t", "focal", "points", "n_iters", "status", "final_stats", "trace_off")
_TRACES = ("costs", "lambdas", "accepted", "evals")


class _Slot:
    """One ring slot: pinned upload buffer, device raw arrays + records,
    solution buffers and their pinned read-back copies (grown on demand)."""

    def __init__(self, torch, device):
        self.torch, self.device = torch, device
        self.up_h = self.up_d = None
        self.rec = self.lo = self.ws = self.pack_ws = None
        self.out_d = {}
        self.out_h = {}
        self.h2d = self.done = self.read = None

    @staticmethod
    def _grow(t, n, torch, **kw):
        if t is None or t.numel() < n:
            if t is not None:   # the old buffer may still be in use on another stream
                torch.cuda.synchronize()
            t = torch.empty(max(int(n * 1.25), 16), **kw)
        return t

    def ensure(self, up_bytes, K, P, C, B, max_iters):
        torch = self.torch
        u8 = dict(dtype=torch.uint8)
        self.up_h = self._grow(self.up_h, up_bytes, torch, pin_memory=True, **u8)
        self.up_d = self._grow(self.up_d, up_bytes, torch, device=self.device, **u8)
        self.rec = self._grow(self.rec, 16 * K, torch, device=self.device, **u8)
        self.lo = self._grow(self.lo, 8 * K, torch, device=self.device, **u8)
        self.pack_ws = self._grow(self.pack_ws, 4 * max(P, 1), torch, device=self.device, **u8)
        w = max(max_iters, 1)
        f64, u8_, i32 = torch.float64, torch.uint8, torch.int32
        dev_only = dict(costs=(B * (max_iters + 1), f64), lambdas=(B * w, f64), accepted=(B * w, u8_),
                        evals=(B * w, u8_))
        both = dict(R=(C * 9, f64), t=(C * 3, f64), focal=(B, f64), points=(P * 3, f64), n_iters=(B, i32),
                    status=(B, i32), final_stats=(B * 4, f64), trace_off=(B + 1, torch.int64),
                    c_costs=(B * (max_iters + 1), f64), c_lambdas=(B * w, f64), c_accepted=(B * w, u8_),
                    c_evals=(B * w, u8_))
        for k, (n, dt) in dev_only.items():
            self.out_d[k] = self._grow(self.out_d.get(k), n, torch, dtype=dt, device=self.device)
        for k, (n, dt) in both.items():
            self.out_d[k] = self._grow(self.out_d.get(k), n, torch, dtype=dt, device=self.device)
            self.out_h[k] = self._grow(self.out_h.get(k), n, torch, dtype=dt, pin_memory=True)


class BatchSolver:
    """Pipelined host-to-host solver for lists of BaProblem-like objects
    (attributes or dict keys R, t, focal, cx, cy, points, cam_idx, pt_idx, uv,
    fixed_cams, optimize_focal[, optimize_points]).

    `solve(problems)` mutates every problem like `lm_solve` does (R, t,
    points written in place when the arrays are writable float64, rebound
    otherwise; focal rebound) and returns a `BatchResult`."""

    def __init__(self, prm, n_chunks=16, min_chunk=512, threads=None, device=None, ring=4,
                 oversize=None, max_cams=32):
        torch = _lib.torch_cuda()
        self.torch = torch
        self.prm = prm
        self.n_chunks = n_chunks
        self.min_chunk = min_chunk
        self.threads = threads or default_threads()
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.copy = torch.cuda.Stream(self.device)
        self.compute = [torch.cuda.Stream(self.device), torch.cuda.Stream(self.device)]
        self.back = torch.cuda.Stream(self.device)
        self.trace_back = torch.cuda.Stream(self.device)   # packed-trace read-backs (own queue: the
        #                                                    read-back stream holds later chunks' copies)
        self.slots = [_Slot(torch, self.device) for _ in range(ring)]
        self.h2d_bytes = self.d2h_bytes = 0
        self.launches = 0
        # problems with more cameras than mba_solve's fused kernels hold go to
        # `oversize(problem) -> info dict` (the stage-kernel loop)
        self.oversize = oversize
        self.max_cams = max_cams

    def chunks(self, B):
        """Chunk boundaries. With enough chunks the first and last two are
        smaller (weights 1/4, 1/2 ... 1/2, 1/4): the device starts after a
        short first host gather, and the last read-back + write-back, which
        nothing overlaps, is short too."""
        n = max(1, min(self.n_chunks, B // max(self.min_chunk, 1)))
        w = [1.0] * n
        if n >= 6:
            w[0] = w[-1] = 0.25
            w[1] = w[-2] = 0.5
        tot = sum(w)
        cuts, acc = [0], 0.0
        for x in w:
            acc += x
            cuts.append(int(round(B * acc / tot)))
        cuts[-1] = B
        return sorted(set(cuts))

    def solve(self, problems) -> BatchResult:
        torch, prm, H = self.torch, self.prm, host_module()
        problems = list(problems)
        B = len(problems)
        res = BatchResult(B, prm.max_iters)
        if B == 0:
            return res
        cuts = self.chunks(B)
        pending = []
        self.h2d_bytes = self.d2h_bytes = 0
        self.launches = 0
        self.host_s = {}   # host-side seconds per stage of the last call (diagnostics)
        L = _lib.lib()
        import time
        clock = time.perf_counter

        def tick(name, t0):
            self.host_s[name] = self.host_s.get(name, 0.0) + clock() - t0
        for ci, (lo, hi) in enumerate(zip(cuts[:-1], cuts[1:])):
            ring = len(self.slots)
            slot = self.slots[ci % ring]
            # a slot is reused `ring` chunks later: its previous chunk must be
            # written back (host) before the pinned buffers are overwritten
            t0 = clock()
            while pending and pending[0][0] <= ci - ring:
                self._finish(pending.pop(0), res)
            tick("finish", t0)
            t0 = clock()
            chunk = problems[lo:hi]
            try:
                batch = H.Batch(chunk)
                norm = None
            except TypeError:
                # arrays of another dtype / layout (float32, lists, strided
                # views): solve normalised copies, then rebind the results
                norm = [normalise(p) for p in chunk]
                batch = H.Batch(norm)
            co, po, oo = (np.frombuffer(x, np.int64) for x in batch.offsets())
            index = np.arange(lo, hi)
            over = np.flatnonzero(np.diff(co) > self.max_cams)
            if len(over):   # rare: solve those problems outside the batch, keep the rest
                if self.oversize is None:
                    raise ValueError(f"problem {lo + int(over[0])} has more than {self.max_cams} cameras")
                for j in over:
                    res.set(lo + int(j), self.oversize(chunk[j]))
                keep = np.setdiff1d(np.arange(hi - lo), over)
                if not len(keep):
                    continue
                index = lo + keep
                chunk = [chunk[j] for j in keep]
                if norm is not None:
                    norm = [norm[j] for j in keep]
                batch = H.Batch(norm if norm is not None else chunk)
                co, po, oo = (np.frombuffer(x, np.int64) for x in batch.offsets())
            m = len(index)
            C, P, K = int(co[-1]), int(po[-1]), int(oo[-1])
            lay, nbytes = layout(C, P, K, m)
            slot.ensure(nbytes, K, P, C, m, prm.max_iters)
            tick("walk", t0)
            t0 = clock()
            if slot.h2d is not None:
                slot.h2d.synchronize()
            tick("wait_h2d", t0)
            t0 = clock()
            up = slot.up_h.numpy()
            any_lo, max_pairs, max_track, bad = batch.gather(0, m, up, lay, self.threads)
            if any_lo:   # values that are not fp32-representable: the low-order stream too
                batch.gather_lo(0, m, up, lay["uv_lo"], self.threads)
            else:
                nbytes = lay["uv_lo"]
            tick("gather", t0)
            t0 = clock()
            if bad >= 0:
                raise IndexError(f"problem {int(index[bad])}: observation index out of range")
            nc, no, npt = np.diff(co), np.diff(oo), np.diff(po)
            d = self._desc(slot, lay, m, int(nc.max()), int(no.max()), int(npt.max()), max_pairs,
                           max_track, any_lo)
            # H2D (waits until the slot's previous solve no longer reads the inputs)
            if slot.done is not None:
                self.copy.wait_event(slot.done)
            with torch.cuda.stream(self.copy):
                slot.up_d[:nbytes].copy_(slot.up_h[:nbytes], non_blocking=True)
                slot.h2d = torch.cuda.Event()
                slot.h2d.record(self.copy)
            self.h2d_bytes += nbytes
            cs = self.compute[ci % 2]
            cs.wait_event(slot.h2d)
            if slot.read is not None:
                cs.wait_event(slot.read)
            base = slot.up_d.data_ptr()
            with torch.cuda.stream(cs):
                st = _lib.stream_ptr()
                _lib.check(L.mba_pack_obs(m, base + lay["obs_off"], base + lay["pt_off"], base + lay["cam_off"],
                                          base + lay["cam"], base + lay["pt"], base + lay["uv"],
                                          (base + lay["uv_lo"]) if any_lo else None, ptr(slot.rec),
                                          ptr(slot.lo) if any_lo else None,
                                          ptr(slot.pack_ws), slot.pack_ws.numel(), st), "mba_pack_obs")
                c = self._cfg()
                o = self._outs(slot, lay)
                need = L.mba_workspace_bytes(ct.byref(d), ct.byref(c))
                slot.ws = _Slot._grow(slot.ws, need, torch, dtype=torch.uint8, device=self.device)
                _lib.check(L.mba_solve(ct.byref(d), ct.byref(c), ct.byref(o), ptr(slot.ws), slot.ws.numel(), st),
                           "mba_solve")
                od = slot.out_d
                _lib.check(L.mba_compact_traces(m, prm.max_iters, ptr(od["n_iters"]), ptr(od["costs"]),
                                                ptr(od["lambdas"]), ptr(od["accepted"]), ptr(od["evals"]),
                                                ptr(od["trace_off"]), ptr(od["c_costs"]), ptr(od["c_lambdas"]),
                                                ptr(od["c_accepted"]), ptr(od["c_evals"]), st),
                           "mba_compact_traces")
                self.launches += 3 + int(L.mba_solve_launches(ct.byref(d), ct.byref(c)))
                slot.done = torch.cuda.Event()
                slot.done.record(cs)
            self.back.wait_event(slot.done)
            sizes = self._out_sizes(C, P, m)
            with torch.cuda.stream(self.back):
                for k in _OUT:
                    n = sizes[k]
                    slot.out_h[k][:n].copy_(slot.out_d[k][:n], non_blocking=True)
                    self.d2h_bytes += n * slot.out_h[k].element_size()
                slot.read = torch.cuda.Event()
                slot.read.record(self.back)
            pending.append((ci, index, slot, batch, sizes, chunk, norm))
            tick("enqueue", t0)
        t0 = clock()
        while pending:
            self._finish(pending.pop(0), res)
        tick("finish", t0)
        return res

    # ------------------------------------------------------------------
    def _out_sizes(self, C, P, m):
        return dict(R=9 * C, t=3 * C, focal=m, points=3 * P, n_iters=m, status=m, final_stats=4 * m,
                    trace_off=m + 1)

    def _finish(self, item, res):
        import time
        torch = self.torch
        ci, index, slot, batch, sizes, chunk, norm = item
        lo = int(index[0])
        t0 = time.perf_counter()
        slot.read.synchronize()
        self.host_s["wait_read"] = self.host_s.get("wait_read", 0.0) + time.perf_counter() - t0
        m = len(index)
        h = {k: slot.out_h[k][:sizes[k]].numpy() for k in _OUT}
        # the packed traces: only their used prefix crosses PCIe
        off = h["trace_off"].copy()
        tot = int(off[-1])
        with torch.cuda.stream(self.trace_back):
            for k, n in (("c_costs", tot + m), ("c_lambdas", tot), ("c_accepted", tot), ("c_evals", tot)):
                slot.out_h[k][:n].copy_(slot.out_d[k][:n], non_blocking=True)
                self.d2h_bytes += n * slot.out_h[k].element_size()
        self.trace_back.synchronize()
        res.add_chunk(index, off, slot.out_h["c_costs"][:tot + m].numpy().copy(),
                      slot.out_h["c_lambdas"][:tot].numpy().copy(), slot.out_h["c_accepted"][:tot].numpy().copy(),
                      slot.out_h["c_evals"][:tot].numpy().copy())
        status = h["status"]
        if np.any(status < 0):
            b = int(np.flatnonzero(status < 0)[0])
            raise ValueError(f"problem {int(index[b])}: malformed problem (status {int(status[b])})")
        rebind = batch.scatter(0, m, h["R"], h["t"], h["focal"], h["points"], self.threads)
        if rebind:
            self._rebind(batch, norm if norm is not None else chunk, rebind, h)
        if norm is not None:
            for p, q in zip(chunk, norm):
                for k in ("R", "t", "points", "focal"):
                    if k == "points" and not q["optimize_points"]:
                        continue
                    if isinstance(p, dict):
                        p[k] = q[k]
                    else:
                        setattr(p, k, q[k])
        res.n_iters[index] = h["n_iters"]
        res.status[index] = status
        res.final_stats[index] = h["final_stats"].reshape(m, 4)

    def _rebind(self, batch, chunk, idx, h):
        """Problems whose arrays are read-only get new arrays (the reference
        itself rebinds R / t / points on rollback, miniba.py:288)."""
        co, po, _ = (np.frombuffer(x, np.int64) for x in batch.offsets())
        for j in idx:
            p = chunk[j]
            R = h["R"][9 * co[j]:9 * co[j + 1]].reshape(-1, 3, 3).copy()
            t = h["t"][3 * co[j]:3 * co[j + 1]].reshape(-1, 3).copy()
            X = h["points"][3 * po[j]:3 * po[j + 1]].reshape(-1, 3).copy()
            for k, v in (("R", R), ("t", t), ("points", X)):
                if isinstance(p, dict):
                    p[k] = v
                else:
                    setattr(p, k, v)

    def _desc(self, slot, lay, m, max_cams, max_obs, max_points, max_pairs, max_track, any_lo):
        base = slot.up_d.data_ptr()
        vp = ct.c_void_p
        return MbaBatchDesc(n_problems=m, max_cams=max_cams, max_obs=max_obs, max_points=max_points,
                            max_pairs=max_pairs, max_track=max_track, cam_off=vp(base + lay["cam_off"]),
                            pt_off=vp(base + lay["pt_off"]), obs_off=vp(base + lay["obs_off"]),
                            obs=ptr(slot.rec), obs_lo=ptr(slot.lo) if any_lo else None,
                            fixed=vp(base + lay["fixed"]), cx=vp(base + lay["cx"]), cy=vp(base + lay["cy"]),
                            flags=vp(base + lay["flags"]))

    def _cfg(self):
        from .solver import KERNELS
        p = self.prm
        return MbaLmConfig(lambda_init=p.lambda_init, nu=p.nu, delta=p.delta, max_iters=p.max_iters,
                           loss=_lib.LOSS[p.loss], precision=_lib.PRECISION[p.precision],
                           ctas_per_problem=KERNELS[p.kernel],
                           fail_iters_mask=sum(1 << int(i) for i in p.fail_at if 0 <= int(i) < 64))

    def _outs(self, slot, lay):
        base = slot.up_d.data_ptr()
        vp = ct.c_void_p
        od = slot.out_d
        return MbaOutputs(R_in=vp(base + lay["R"]), t_in=vp(base + lay["t"]), focal_in=vp(base + lay["focal"]),
                          points_in=vp(base + lay["points"]), R_out=ptr(od["R"]), t_out=ptr(od["t"]),
                          focal_out=ptr(od["focal"]), points_out=ptr(od["points"]), costs=ptr(od["costs"]),
                          lambdas=ptr(od["lambdas"]), accepted=ptr(od["accepted"]), evals=ptr(od["evals"]),
                          n_iters=ptr(od["n_iters"]), status=ptr(od["status"]),
                          final_stats=ptr(od["final_stats"]))


def normalise(p):
    """Dict copy of a BaProblem-like object with C-contiguous float64 /
    int64 / bool arrays (the native walk's accepted formats)."""
    g = (lambda k, d=None: p.get(k, d)) if isinstance(p, dict) else (lambda k, d=None: getattr(p, k, d))
    f64 = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return dict(R=f64(g("R")), t=f64(g("t")), focal=float(g("focal")), cx=float(g("cx")),
                cy=float(g("cy")), points=f64(g("points")),
                cam_idx=np.ascontiguousarray(np.asarray(g("cam_idx")).reshape(-1), dtype=np.int64),
                pt_idx=np.ascontiguousarray(np.asarray(g("pt_idx")).reshape(-1), dtype=np.int64),
                uv=f64(g("uv")), fixed_cams=np.ascontiguousarray(np.asarray(g("fixed_cams")).reshape(-1),
                                                                dtype=bool),
                optimize_focal=bool(g("optimize_focal")), optimize_points=bool(g("optimize_points", True)))
