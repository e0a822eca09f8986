"""Sharded solve with the full output gather (paper_2506_05558_b200/dist.py)
on the GPU: two ranks on one GPU (gloo carries the gather on host copies,
the box has one GPU), each solving its contiguous shard with mba_solve; the
gathered R, t, focal, points, statistics, status and traces on rank 0 equal
a single-rank solve of the whole batch bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

N, MAX_IT = 40, 200


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out, precision):
    sys.path[:0] = [REPO, os.path.join(REPO, "src")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2506_05558_b200 import dist as mdist, solver
    from paper_2506_05558_b200.synth import make_batch
    lo, hi = mdist.shard_range(N, rank, world)
    b = make_batch(hi - lo, n_cams=8, K=1500, seed=41, first=lo)
    db = solver.to_device(solver.pack_synth(b))
    ss = mdist.ShardedSolver(db, solver.LmParams(max_iters=MAX_IT, precision=precision),
                             comm_device=torch.device("cpu"))
    for _ in range(2):
        full = ss.step()
    if rank == 0:
        np.savez(out, **{k: v.cpu().numpy() for k, v in full.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("precision", ["f64", "mixed"])
def test_two_rank_sharded_solve_gathers_the_single_rank_solution(precision, cuda_ok, tmp_path):
    from paper_2506_05558_b200 import dist as mdist, solver
    from paper_2506_05558_b200.synth import make_batch
    out = str(tmp_path / "full.npz")
    mp.spawn(_worker, args=(2, _port(), out, precision), nprocs=2, join=True)
    got = np.load(out)
    b = make_batch(N, n_cams=8, K=1500, seed=41)
    db = solver.to_device(solver.pack_synth(b))
    sol = solver.solve(db, solver.LmParams(max_iters=MAX_IT, precision=precision))
    torch.cuda.synchronize()
    counts = mdist.field_counts(N, int(b.cam_off[-1]), int(b.pt_off[-1]), MAX_IT)
    for k, n in counts.items():
        np.testing.assert_array_equal(got[k], getattr(sol, k).reshape(-1)[:n].cpu().numpy(), err_msg=k)


def _nccl_worker(rank, world, port, out):
    sys.path[:0] = [REPO, os.path.join(REPO, "src")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    from paper_2506_05558_b200 import dist as mdist, solver
    from paper_2506_05558_b200.synth import make_batch
    lo, hi = mdist.shard_range(N, rank, world)
    b = make_batch(hi - lo, n_cams=8, K=1500, seed=41, first=lo)
    db = solver.to_device(solver.pack_synth(b))
    ss = mdist.ShardedSolver(db, solver.LmParams(max_iters=MAX_IT), dist=dist,
                             comm_device=torch.device("cuda", 0))
    full = ss.step()
    torch.cuda.synchronize()
    np.savez(out, **{k: v.cpu().numpy() for k, v in full.items()})
    dist.destroy_process_group()


def test_nccl_gather_path_single_rank(cuda_ok, tmp_path):
    """The production collective path -- NCCL process group, device-resident
    byte-packed gather (dist.OutputGather) -- at world size 1 (the box has one
    GPU; NCCL refuses two ranks on the same device): the gathered outputs equal
    the direct solve."""
    from paper_2506_05558_b200 import dist as mdist, solver
    from paper_2506_05558_b200.synth import make_batch
    out = str(tmp_path / "nccl.npz")
    mp.spawn(_nccl_worker, args=(1, _port(), out), nprocs=1, join=True)
    got = np.load(out)
    b = make_batch(N, n_cams=8, K=1500, seed=41)
    db = solver.to_device(solver.pack_synth(b))
    sol = solver.solve(db, solver.LmParams(max_iters=MAX_IT))
    torch.cuda.synchronize()
    counts = mdist.field_counts(N, int(b.cam_off[-1]), int(b.pt_off[-1]), MAX_IT)
    for k, n in counts.items():
        np.testing.assert_array_equal(got[k], getattr(sol, k).reshape(-1)[:n].cpu().numpy(), err_msg=k)
