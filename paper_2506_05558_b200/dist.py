"""Multi-GPU plumbing for batches of independent problems.

Problems never span GPUs. A batch is split into contiguous problem ranges,
one per rank; ranks solve with no communication and the only
collective is the final gather of fixed-size per-problem summaries
(final cost, sum e, sum e^2, K, n_iters, status) to every rank. Works with
NCCL (GPU) and gloo (CPU tests).
"""
from __future__ import annotations

SUMMARY_WIDTH = 6   # cost, sum_e, sum_e2, K, n_iters, status


def shard_range(n_problems: int, rank: int, world: int):
    """Contiguous [lo, hi) problem range of `rank`; sizes differ by at most one."""
    return n_problems * rank // world, n_problems * (rank + 1) // world


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
    problem order, (n_problems, 6). `bufs` (world tensors like `local`) may be
    passed to avoid allocations in a timed loop."""
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
