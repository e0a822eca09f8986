"""The end-to-end batch path on the device: mba_pack_obs (stable point-major
sort + record packing, csrc/mba_pack.cu) against numpy's stable argsort, and
gsrecon.miniba.lm_solve_batch on lists of BaProblem objects against the
device solve of the host-packed batch and against the reference goldens."""
import ctypes as ct

import numpy as np
import pytest

from conftest import golden_cases, load_case
from gpu_helpers import assert_parity, run_device

pytestmark = pytest.mark.gpu


def _pack_device(problems, with_lo):
    import torch
    from paper_2506_05558_b200 import _lib
    from paper_2506_05558_b200._lib import ptr
    L = _lib.lib()
    off = lambda v: np.concatenate([[0], np.cumsum(v)]).astype(np.int64)
    oo = off([len(p["uv"]) for p in problems])
    po = off([len(p["points"]) for p in problems])
    co = off([len(p["R"]) for p in problems])
    cam = np.concatenate([p["cam_idx"] for p in problems]).astype(np.int32)
    pt = np.concatenate([p["pt_idx"] for p in problems]).astype(np.int32)
    uv = np.concatenate([p["uv"] for p in problems]).astype(np.float64)
    uv32 = uv.astype(np.float32)
    uvlo = (uv - uv32.astype(np.float64)).astype(np.float32)   # the host gather's streams
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    K = int(oo[-1])
    rec = torch.zeros((K, 4), dtype=torch.float32, device="cuda")
    lo = torch.zeros((K, 2), dtype=torch.float32, device="cuda") if with_lo else None
    ws = torch.empty(int(L.mba_pack_obs_workspace_bytes(int(po[-1]))), dtype=torch.uint8, device="cuda")
    args = [d(oo), d(po), d(co), d(cam), d(pt), d(uv32), d(uvlo) if with_lo else None]
    rc = L.mba_pack_obs(len(problems), *[ptr(a) for a in args], ptr(rec), ptr(lo), ptr(ws), ws.numel(),
                        _lib.stream_ptr())
    assert rc == 0
    torch.cuda.synchronize()
    return rec.cpu().numpy(), (lo.cpu().numpy() if with_lo else None), oo


def _expected(problems):
    recs, los = [], []
    for p in problems:
        order = np.argsort(p["pt_idx"], kind="stable")
        uv = p["uv"][order]
        r = np.empty((len(order), 4), np.float32)
        r[:, :2] = uv.astype(np.float32)
        r.view(np.int32)[:, 2] = p["cam_idx"][order]
        r.view(np.int32)[:, 3] = p["pt_idx"][order]
        recs.append(r)
        los.append((uv - uv.astype(np.float32).astype(np.float64)).astype(np.float32))
    return np.concatenate(recs), np.concatenate(los)


def _shuffled(p, seed):
    perm = np.random.default_rng(seed).permutation(len(p["uv"]))
    q = dict(p)
    for k in ("cam_idx", "pt_idx", "uv"):
        q[k] = p[k][perm]
    return q


def test_pack_obs_is_numpy_stable_argsort(cuda_ok):
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(24, n_cams=8, K=1500, seed=4)
    probs = []
    for i in range(24):
        p = b.problem(i)
        if i % 3 == 0:
            p = _shuffled(p, i)                                  # random order
        elif i % 3 == 1:
            order = np.argsort(p["cam_idx"], kind="stable")      # camera-major (smoke)
            p = {**p, **{k: p[k][order] for k in ("cam_idx", "pt_idx", "uv")}}
        if i % 4 == 0:
            p["uv"] = p["uv"] + 1e-7 * np.random.default_rng(i).standard_normal(p["uv"].shape)
        probs.append(p)
    # one large problem: more points than the shared-memory count table holds
    big = make_batch(1, n_cams=8, K=40000, seed=9).problem(0)
    probs.append(_shuffled(big, 3))
    rec, lo, oo = _pack_device(probs, True)
    er, el = _expected(probs)
    np.testing.assert_array_equal(rec.view(np.int32), er.view(np.int32))
    np.testing.assert_array_equal(lo, el)
    rec2, _, _ = _pack_device(probs, False)
    np.testing.assert_array_equal(rec2.view(np.int32), er.view(np.int32))


def _baproblems(batch, idx):
    from gsrecon.miniba import BaProblem
    out = []
    for i in idx:
        p = batch.problem(i)
        p["cam_idx"] = p["cam_idx"].astype(np.int64)
        p["pt_idx"] = p["pt_idx"].astype(np.int64)
        out.append(BaProblem(**p))
    return out


@pytest.mark.parametrize("precision", ["f64", "mixed"])
def test_lm_solve_batch_equals_device_solve(precision, cuda_ok):
    """Chunked, pipelined list path == one packed device solve, bit for bit
    (same kernel, same per-problem arithmetic), with several chunks in flight."""
    from gsrecon.config import LmConfig
    from gsrecon.miniba import lm_solve_batch, _SOLVERS
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(700, n_cams=8, K=1200, seed=13)
    probs = _baproblems(b, range(700))
    ref = run_device([b.problem(i) for i in range(700)], dict(max_iters=200), precision)
    _SOLVERS.clear()
    from paper_2506_05558_b200.batch import BatchSolver
    import torch
    bs = BatchSolver(None, n_chunks=5, min_chunk=100)
    _SOLVERS[torch.cuda.current_device()] = bs
    for rep in range(2):
        ps = probs if rep == 0 else _baproblems(b, range(700))
        infos = lm_solve_batch(ps, LmConfig(max_iters=200), precision=precision)
        assert len(infos) == 700
        for i in (0, 1, 99, 100, 101, 350, 699):
            d, r = infos[i], ref[i]
            np.testing.assert_array_equal(d["costs"], r["costs"])
            np.testing.assert_array_equal(d["accepted"], r["accepted"])
            np.testing.assert_array_equal(ps[i].R, r["R"])
            np.testing.assert_array_equal(ps[i].t, r["t"])
            np.testing.assert_array_equal(ps[i].points, r["points"])
            assert ps[i].focal == r["focal"]
    _SOLVERS.clear()


def test_lm_solve_batch_sorts_on_device(cuda_ok):
    """Camera-major / shuffled observation order: the device sort reproduces
    the host's stable argsort exactly (bit-identical solves), and the solution
    agrees with the point-major input under the parity rule (a different
    summation order inside a point only moves the roundoff-level tail)."""
    from gsrecon.config import LmConfig
    from gsrecon.miniba import BaProblem, lm_solve_batch
    from oracle import miniba_oracle as O
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(6, n_cams=8, K=2000, seed=17)
    a = _baproblems(b, range(6))
    sh = [_shuffled(b.problem(i), 100 + i) for i in range(6)]
    s = [BaProblem(**{k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in q.items()}) for q in sh]
    ia = lm_solve_batch(a, LmConfig(max_iters=200))
    is_ = lm_solve_batch(s, LmConfig(max_iters=200))
    host_sorted = run_device(sh, dict(max_iters=200), "f64")
    for i in range(6):
        np.testing.assert_array_equal(is_[i]["costs"], host_sorted[i]["costs"])
        np.testing.assert_array_equal(s[i].points, host_sorted[i]["points"])
        i_star = O.plateau_index(ia[i]["costs"])
        np.testing.assert_array_equal(ia[i]["accepted"][:i_star + 1], is_[i]["accepted"][:i_star + 1])
        assert abs(ia[i]["costs"][-1] - is_[i]["costs"][-1]) <= 1e-9 * ia[i]["costs"][-1]


@pytest.mark.parametrize("path", [p for p in golden_cases() if "fault" not in p])
def test_lm_solve_batch_against_reference_goldens(path, cuda_ok):
    """All golden cases in ONE batched call through the public API."""
    from gsrecon.config import LmConfig
    from gsrecon.miniba import BaProblem, lm_solve_batch
    prob, cfg, out = load_case(path)
    p = BaProblem(**prob)
    info = lm_solve_batch([p], LmConfig(lambda_init=cfg["lambda_init"], nu=cfg["nu"],
                                        huber_delta=cfg["delta"], max_iters=cfg["max_iters"]))[0]
    dev = dict(info, R=p.R, t=p.t, focal=p.focal, points=p.points)
    assert_parity(dev, out["costs"], out["accepted"], out["evals"], out["lambdas"], out["R"], out["t"],
                  float(out["focal"]), label=path)


def test_lm_solve_batch_errors_and_odd_inputs(cuda_ok):
    from gsrecon.config import LmConfig
    from gsrecon.miniba import BaProblem, lm_solve_batch
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(3, n_cams=5, K=500, seed=23)
    ps = _baproblems(b, range(3))
    ps[1].pt_idx = ps[1].pt_idx.copy()
    ps[1].pt_idx[0] = -1
    with pytest.raises(IndexError):
        lm_solve_batch(ps, LmConfig(max_iters=5))
    ps = _baproblems(b, range(3))
    ps[2].fixed_cams = ps[2].fixed_cams[:3]
    with pytest.raises(ValueError):
        lm_solve_batch(ps, LmConfig(max_iters=5))
    # float32 / list inputs go through the normalising path; read-only arrays are rebound
    ref = _baproblems(b, range(3))
    lm_solve_batch(ref, LmConfig(max_iters=30))
    ps = _baproblems(b, range(3))
    ps[0].uv = ps[0].uv.astype(np.float32).astype(np.float64)   # same values
    ps[1].t = ps[1].t.tolist()
    ps[2].R.flags.writeable = False
    lm_solve_batch(ps, LmConfig(max_iters=30))
    for i in range(3):
        np.testing.assert_array_equal(np.asarray(ps[i].t), ref[i].t)
        np.testing.assert_array_equal(ps[i].R, ref[i].R)
        assert isinstance(ps[i].R, np.ndarray)
