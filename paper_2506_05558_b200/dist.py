"""Multi-GPU plumbing for batches of independent problems.

Problems never span GPUs. A batch is split into contiguous problem ranges,
one per rank; ranks solve with no communication, and the only collective is
the final gather of the FULL per-problem outputs -- refined R, t, focal,
points (ragged), final statistics, n_iters, status and the LM traces
(costs, lambdas, accepted, evals) -- to rank 0, which is what lm_solve returns
per problem (miniba.py:265-270, 288, 294-296; "no shared mutable
state across concurrent solves").

The gather moves one byte buffer per rank: every output field of the rank's
shard packed back to back and zero-padded to the largest rank's size (the
per-rank problem / camera / point counts are exchanged once, at set-up), so a
step costs one `gather` (NCCL over NVLink on GPUs, gloo on CPU tensors in the
tests) and rank 0 unpacks views in global problem order.
"""
from __future__ import annotations

SUMMARY_WIDTH = 6   # cost, sum_e, sum_e2, K, n_iters, status

# output field -> (dtype name, elements per camera, per point, per problem, per problem-iteration)
_FIELDS = (("R", "float64", 9, 0, 0, 0), ("t", "float64", 3, 0, 0, 0), ("focal", "float64", 0, 0, 1, 0),
           ("points", "float64", 0, 3, 0, 0), ("final_stats", "float64", 0, 0, 4, 0),
           ("n_iters", "int32", 0, 0, 1, 0), ("status", "int32", 0, 0, 1, 0),
           ("costs", "float64", 0, 0, 1, 1), ("lambdas", "float64", 0, 0, 0, 1),
           ("accepted", "uint8", 0, 0, 0, 1), ("evals", "uint8", 0, 0, 0, 1))
_ITEM = {"float64": 8, "int32": 4, "uint8": 1}


def shard_range(n_problems: int, rank: int, world: int):
    """Contiguous [lo, hi) problem range of `rank`; sizes differ by at most one."""
    return n_problems * rank // world, n_problems * (rank + 1) // world


def field_counts(n_problems: int, n_cams: int, n_points: int, max_iters: int, traces: bool = True):
    """Elements of every output field for a shard with these totals."""
    w = max(max_iters, 1)
    out = {}
    for name, _, pc, pp, pb, pi in _FIELDS:
        if pi and not traces:
            continue
        n = pc * n_cams + pp * n_points + pb * n_problems
        if pi:
            n = n_problems * (max_iters + 1 if name == "costs" else w)
        out[name] = n
    return out


def _layout(counts):
    off, pos = {}, 0
    for name, dt, *_ in _FIELDS:
        if name not in counts:
            continue
        off[name] = pos
        pos += (counts[name] * _ITEM[dt] + 15) & ~15
    return off, pos


class OutputGather:
    """Gather of complete per-problem solver outputs to rank `dst`.

    `local` = (n_problems, n_cams, n_points) of this rank's shard. Set-up
    all-gathers those three numbers (once); `gather(outputs)` packs this rank's
    output tensors (a Solution or a dict of tensors with the field names
    above) into one byte buffer, gathers the buffers and, on `dst`, returns a
    dict of tensors in global problem order (None elsewhere)."""

    def __init__(self, torch, dist, local, max_iters, device, comm_device=None, dst=0, traces=True,
                 group=None):
        self.torch, self.dist, self.dst, self.group = torch, dist, dst, group
        # with a process group the gather always runs the collective (also at
        # world size 1); without one the outputs are returned in place
        self.collective = dist is not None and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.collective else 1
        self.rank = dist.get_rank(group) if self.collective else 0
        self.max_iters, self.traces = max_iters, traces
        self.device = device
        self.comm = comm_device or device
        mine = torch.tensor(list(local), dtype=torch.int64, device=self.comm)
        if self.world > 1:
            allc = [torch.empty_like(mine) for _ in range(self.world)]
            dist.all_gather(allc, mine, group=group)
            self.shards = [tuple(int(x) for x in c.tolist()) for c in allc]
        else:
            self.shards = [tuple(int(x) for x in mine.tolist())]
        self.counts = [field_counts(*s, max_iters, traces) for s in self.shards]
        self.layouts = [_layout(c) for c in self.counts]
        self.nbytes = max(n for _, n in self.layouts)
        u8 = dict(dtype=torch.uint8, device=self.comm)
        self.send = torch.zeros(self.nbytes, **u8)
        self.recv = ([torch.zeros(self.nbytes, **u8) for _ in range(self.world)]
                     if self.rank == dst and self.collective else None)

    @property
    def bytes_per_step(self):
        """Bytes rank dst receives per gather (padded buffers of every rank)."""
        return self.nbytes * self.world

    def _get(self, outputs, name):
        return outputs[name] if isinstance(outputs, dict) else getattr(outputs, name)

    def pack(self, outputs):
        torch = self.torch
        off, _ = self.layouts[self.rank]
        for name, n in self.counts[self.rank].items():
            t = self._get(outputs, name)
            flat = t.reshape(-1)[:n].contiguous().view(torch.uint8)
            self.send[off[name]:off[name] + flat.numel()].copy_(flat, non_blocking=True)
        return self.send

    def gather(self, outputs):
        torch = self.torch
        if not self.collective:
            return {name: self._get(outputs, name).reshape(-1)[:n] for name, n in self.counts[0].items()}
        self.pack(outputs)
        if self.comm != self.device:
            torch.cuda.current_stream().synchronize()
        self.dist.gather(self.send, gather_list=self.recv, dst=self.dst, group=self.group)
        if self.rank != self.dst:
            return None
        out = {}
        for name, dt, *_ in _FIELDS:
            if name not in self.counts[0]:
                continue
            dtype = getattr(torch, dt)
            parts = []
            for r in range(self.world):
                off, _ = self.layouts[r]
                n = self.counts[r][name]
                parts.append(self.recv[r][off[name]:off[name] + n * _ITEM[dt]].view(dtype))
            out[name] = torch.cat(parts)
        return out


class ShardedSolver:
    """Library entry point for a sharded batched solve: this rank's shard
    (a solver.DeviceBatch) is solved by mba_solve with no communication, then
    the complete outputs are gathered to rank 0 (OutputGather).

        ss = ShardedSolver(db_local, prm)        # collective set-up
        full = ss.step()                          # dict in global order on rank 0
    """

    def __init__(self, db, prm, dist=None, comm_device=None, traces=True, group=None):
        from . import _lib, solver
        torch = _lib.torch_cuda()
        if dist is None:
            import torch.distributed as dist
        self.db, self.prm, self.solver = db, prm, solver
        self.sol = solver.Solution(db, prm.max_iters)
        n_cams = int(db.R.shape[0]) if db.R.dim() == 3 else int(db.R.numel() // 9)
        n_pts = int(db.points.numel() // 3)
        self.gather = OutputGather(torch, dist, (db.n_problems, n_cams, n_pts), prm.max_iters,
                                   db.obs.device, comm_device=comm_device, traces=traces, group=group)

    def step(self):
        self.solver.solve(self.db, self.prm, self.sol)
        return self.gather.gather(self.sol)


# ---------------------------------------------------------------------------
# compact per-problem summaries (kept for callers that only need statistics)

def padded_rows(n_problems: int, world: int) -> int:
    return (n_problems + world - 1) // world


def pack_summary(torch, final_stats, n_iters, status, rows: int, device):
    """(rows, 6) float64 tensor of this rank's per-problem summaries, zero-padded."""
    out = torch.zeros((rows, SUMMARY_WIDTH), dtype=torch.float64, device=device)
    m = final_stats.shape[0]
    out[:m, :4] = final_stats
    out[:m, 4] = n_iters.to(torch.float64)
    out[:m, 5] = status.to(torch.float64)
    return out


def gather_summaries(torch, dist, local, n_problems: int, world: int, bufs=None):
    """All-gather the padded per-rank summaries and return them in global
    problem order, (n_problems, 6)."""
    if world == 1:
        return local[:n_problems]
    if bufs is None:
        bufs = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(bufs, local)
    parts = []
    for r in range(world):
        lo, hi = shard_range(n_problems, r, world)
        parts.append(bufs[r][:hi - lo])
    return torch.cat(parts, dim=0)
