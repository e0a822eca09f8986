"""CPU (gloo, world_size 2) tests of the multi-GPU plumbing: contiguous shard
ranges and the final gather of the COMPLETE per-problem outputs (R, t,
focal, ragged points, final statistics, n_iters, status, LM traces) in global
problem order (paper_2506_05558_b200/dist.py). On the GPU box the
same code carries mba_solve outputs over NCCL (bench.py, and the one-GPU
2-rank test in tests/test_gpu_dist.py)."""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

N_PROBLEMS = 7
MAX_ITERS = 5


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_outputs(first, count):
    """Deterministic stand-in for a shard's Solution: problem i has 3 + i % 3
    cameras and 10 + 7 * i points, values derived from the global index."""
    n = [3 + (first + i) % 3 for i in range(count)]
    P = [10 + 7 * (first + i) for i in range(count)]
    g = lambda i, k: np.float64(1000 * (first + i) + k)
    R = np.concatenate([np.full((n[i], 9), g(i, 1)) for i in range(count)])
    t = np.concatenate([np.full((n[i], 3), g(i, 2)) for i in range(count)])
    X = np.concatenate([np.arange(3 * P[i], dtype=np.float64) + g(i, 3) for i in range(count)])
    out = dict(R=R, t=t, points=X, focal=np.array([g(i, 4) for i in range(count)]),
               final_stats=np.array([[g(i, 5 + j) for j in range(4)] for i in range(count)]),
               n_iters=np.array([first + i for i in range(count)], np.int32),
               status=np.array([(first + i) % 3 for i in range(count)], np.int32),
               costs=np.array([[g(i, 10 + j) for j in range(MAX_ITERS + 1)] for i in range(count)]),
               lambdas=np.array([[g(i, 20 + j) for j in range(MAX_ITERS)] for i in range(count)]),
               accepted=np.array([[(first + i + j) % 2 for j in range(MAX_ITERS)] for i in range(count)], np.uint8),
               evals=np.array([[(first + i + j) % 6 for j in range(MAX_ITERS)] for i in range(count)], np.uint8))
    return {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in out.items()}, sum(n), sum(P)


def _worker(rank, world, port, out_path):
    sys.path[:0] = [REPO, os.path.join(REPO, "src")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_05558_b200 import dist as mdist
    lo, hi = mdist.shard_range(N_PROBLEMS, rank, world)
    outs, C, P = _fake_outputs(lo, hi - lo)
    g = mdist.OutputGather(torch, dist, (hi - lo, C, P), MAX_ITERS, torch.device("cpu"))
    for _ in range(2):   # the buffers are reused step after step
        full = g.gather(outs)
    if rank == 0:
        np.savez(out_path, **{k: v.numpy() for k, v in full.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_cover_the_batch():
    from paper_2506_05558_b200 import dist as mdist
    for B in (1, 7, 65536):
        for W in (1, 2, 4, 8):
            got = [mdist.shard_range(B, r, W) for r in range(W)]
            assert got[0][0] == 0 and got[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1


def test_two_rank_gloo_gather_of_full_outputs(tmp_path):
    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    single, _, _ = _fake_outputs(0, N_PROBLEMS)
    for k, v in single.items():
        np.testing.assert_array_equal(got[k], v.numpy().reshape(-1), err_msg=k)


def test_field_counts():
    from paper_2506_05558_b200 import dist as mdist
    c = mdist.field_counts(4, 32, 1000, 200)
    assert c["R"] == 288 and c["points"] == 3000 and c["costs"] == 4 * 201 and c["evals"] == 800
    assert "costs" not in mdist.field_counts(4, 32, 1000, 200, traces=False)
