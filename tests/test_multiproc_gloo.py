"""CPU (gloo, world_size 2) test of the multi-GPU plumbing: contiguous shard
ranges, per-shard problem generation, and the final all-gather of per-problem
summaries in global order. The per-problem work here is the CPU oracle (tests
may use it); on the GPU box the same code paths carry mba_solve results."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

N_PROBLEMS = 7


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _summaries(first, count):
    from oracle import miniba_oracle as O
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(count, n_cams=4, K=240, seed=17, first=first)
    stats, iters, status = [], [], []
    for i in range(count):
        info = O.lm(b.problem(i), max_iters=4)
        e_sum = info["mean_err"] * 240
        stats.append([info["cost"], e_sum, info["final_rms"], float(b.obs_off[i + 1] - b.obs_off[i])])
        iters.append(len(info["accepted"]))
        status.append(0)
    return (torch.tensor(stats, dtype=torch.float64), torch.tensor(iters, dtype=torch.int32),
            torch.tensor(status, dtype=torch.int32))


def _worker(rank, world, port, out_path):
    sys.path[:0] = [REPO, os.path.join(REPO, "src")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_05558_b200 import dist as mdist
    lo, hi = mdist.shard_range(N_PROBLEMS, rank, world)
    fs, it, st = _summaries(lo, hi - lo)
    rows = mdist.padded_rows(N_PROBLEMS, world)
    local = mdist.pack_summary(torch, fs, it, st, rows, "cpu")
    full = mdist.gather_summaries(torch, dist, local, N_PROBLEMS, world)
    if rank == 0:
        np.save(out_path, full.numpy())
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


def test_two_rank_gloo_gather_matches_single_process(tmp_path):
    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    gathered = np.load(out)
    from paper_2506_05558_b200 import dist as mdist
    fs, it, st = _summaries(0, N_PROBLEMS)
    single = mdist.pack_summary(torch, fs, it, st, N_PROBLEMS, "cpu").numpy()
    assert gathered.shape == (N_PROBLEMS, mdist.SUMMARY_WIDTH)
    np.testing.assert_array_equal(gathered, single)   # shard-invariant, bit for bit
