"""Native host packer (paper_2506_05558_b200/_mba_host, CPU only): the walk
over a list of BaProblem objects, the threaded gather into the upload layout
and the in-place write-back, checked against plain numpy on the same data."""
import numpy as np
import pytest

from paper_2506_05558_b200 import solver
from paper_2506_05558_b200.batch import host_module, layout, normalise
from paper_2506_05558_b200.synth import make_batch


def _problems(n=12, K=600, seed=2):
    from gsrecon.miniba import BaProblem
    b = make_batch(n, n_cams=6, K=K, seed=seed)
    out = []
    for i in range(n):
        p = b.problem(i)
        if i % 3 == 1:   # int32 indices and camera-major order
            order = np.argsort(p["cam_idx"], kind="stable")
            for k in ("cam_idx", "pt_idx", "uv"):
                p[k] = p[k][order]
            p["cam_idx"] = p["cam_idx"].astype(np.int32)
            p["pt_idx"] = p["pt_idx"].astype(np.int32)
        out.append(BaProblem(**p))
    return b, out


def _gather(probs, threads=3):
    H = host_module()
    hb = H.Batch(probs)
    co, po, oo = (np.frombuffer(x, np.int64) for x in hb.offsets())
    lay, nb = layout(int(co[-1]), int(po[-1]), int(oo[-1]), len(probs))
    buf = np.full(nb, 0xAB, np.uint8)
    ret = hb.gather(0, len(probs), buf, lay, threads)
    return hb, (co, po, oo), lay, buf, ret


def region(buf, lay, name, dtype, count):
    return buf[lay[name]:lay[name] + np.dtype(dtype).itemsize * count].view(dtype)


def test_gather_matches_numpy_concatenation():
    b, probs = _problems()
    hb, (co, po, oo), lay, buf, (any_lo, max_pairs, max_track, bad) = _gather(probs)
    assert len(hb) == len(probs) and bad == -1 and not any_lo
    K, P, C = int(oo[-1]), int(po[-1]), int(co[-1])
    np.testing.assert_array_equal(region(buf, lay, "obs_off", np.int64, len(probs) + 1), oo)
    np.testing.assert_array_equal(region(buf, lay, "uv", np.float32, 2 * K),
                                  np.concatenate([p.uv for p in probs]).ravel().astype(np.float32))
    np.testing.assert_array_equal(region(buf, lay, "cam", np.int32, K),
                                  np.concatenate([p.cam_idx for p in probs]))
    np.testing.assert_array_equal(region(buf, lay, "pt", np.int32, K),
                                  np.concatenate([p.pt_idx for p in probs]))
    np.testing.assert_array_equal(region(buf, lay, "R", np.float64, 9 * C),
                                  np.concatenate([p.R for p in probs]).ravel())
    np.testing.assert_array_equal(region(buf, lay, "points", np.float64, 3 * P),
                                  np.concatenate([p.points for p in probs]).ravel())
    np.testing.assert_array_equal(region(buf, lay, "fixed", np.uint8, C),
                                  np.concatenate([p.fixed_cams for p in probs]).astype(np.uint8))
    np.testing.assert_array_equal(region(buf, lay, "focal", np.float64, len(probs)),
                                  [p.focal for p in probs])
    assert (max_pairs, max_track) == solver._track_stats(b.obs_off, b.pt_off, b.pt)


def test_gather_is_thread_count_invariant_and_flags_low_order_uv():
    _, probs = _problems()
    probs[4].uv = probs[4].uv + 1e-9    # no longer fp32-representable
    outs = [_gather(probs, t) for t in (1, 2, 5)]
    for o in outs[1:]:
        np.testing.assert_array_equal(o[3], outs[0][3])
    assert all(o[4][0] for o in outs)
    # the low-order stream reconstructs the exact float64 pixels
    hb, (co, po, oo), lay, buf, _ = outs[0]
    hb.gather_lo(0, len(probs), buf, lay["uv_lo"], 3)
    K = int(oo[-1])
    hi32 = region(buf, lay, "uv", np.float32, 2 * K).astype(np.float64)
    lo32 = region(buf, lay, "uv_lo", np.float32, 2 * K).astype(np.float64)
    uv = np.concatenate([p.uv for p in probs]).ravel()
    np.testing.assert_array_equal(lo32, (uv - hi32).astype(np.float32).astype(np.float64))
    assert np.abs(hi32 + lo32 - uv).max() < 1e-12


def test_scatter_writes_in_place_and_rebinds_focal():
    _, probs = _problems(n=5)
    R0 = [p.R for p in probs]
    hb, (co, po, oo), *_ = _gather(probs)
    C, P = int(co[-1]), int(po[-1])
    R = np.arange(9 * C, dtype=np.float64)
    t = -np.arange(3 * C, dtype=np.float64)
    f = np.arange(5, dtype=np.float64) + 0.5
    X = np.full(3 * P, 7.0)
    rebind = hb.scatter(0, 5, R, t, f, X, 2)
    assert rebind == []
    for i, p in enumerate(probs):
        assert p.R is R0[i]                      # same array, new values
        np.testing.assert_array_equal(p.R.ravel(), R[9 * co[i]:9 * co[i + 1]])
        np.testing.assert_array_equal(p.t.ravel(), t[3 * co[i]:3 * co[i + 1]])
        assert p.focal == f[i] and isinstance(p.focal, float)
        assert np.all(p.points == 7.0)


def test_read_only_arrays_are_reported_for_rebinding():
    _, probs = _problems(n=3)
    probs[1].R.flags.writeable = False
    hb, (co, po, oo), *_ = _gather(probs)
    C, P = int(co[-1]), int(po[-1])
    rebind = hb.scatter(0, 3, np.zeros(9 * C), np.zeros(3 * C), np.zeros(3), np.zeros(3 * P), 1)
    assert rebind == [1]


def test_walk_errors_follow_the_reference():
    H = host_module()
    _, probs = _problems(n=3)
    probs[1].uv = np.zeros((0, 2))
    probs[1].cam_idx = probs[1].pt_idx = np.zeros(0, np.int64)
    with pytest.raises(ValueError, match="no residuals"):      # miniba.py:229-230
        H.Batch(probs)
    _, probs = _problems(n=3)
    probs[2].fixed_cams = probs[2].fixed_cams[:-1]            # ADVICE: short fixed_cams
    with pytest.raises(ValueError, match="fixed_cams"):
        H.Batch(probs)
    _, probs = _problems(n=3)
    probs[0].pt_idx = probs[0].pt_idx[:-1]
    with pytest.raises(ValueError, match="pt_idx"):
        H.Batch(probs)
    _, probs = _problems(n=3)
    probs[0].uv = probs[0].uv.astype(np.float32)               # other dtype: normalised by Python
    with pytest.raises(TypeError):
        H.Batch(probs)
    H.Batch([normalise(p) for p in probs])


def test_out_of_range_index_is_reported():
    _, probs = _problems(n=4)
    probs[2].pt_idx = probs[2].pt_idx.copy()
    probs[2].pt_idx[5] = len(probs[2].points)
    *_, (any_lo, mp, mt, bad) = _gather(probs)
    assert bad == 2


def test_dict_problems_are_accepted():
    b = make_batch(3, n_cams=4, K=300, seed=5)
    dicts = [b.problem(i) for i in range(3)]
    hb, (co, po, oo), lay, buf, ret = _gather(dicts)
    assert ret[3] == -1 and int(oo[-1]) == int(b.obs_off[-1])


def test_pack_problems_checks_fixed_cams_length():
    b = make_batch(2, n_cams=4, K=300, seed=5)
    ps = [b.problem(i) for i in range(2)]
    ps[0]["fixed_cams"] = ps[0]["fixed_cams"][:3]
    with pytest.raises(ValueError, match="fixed_cams"):
        solver.pack_problems(ps)
