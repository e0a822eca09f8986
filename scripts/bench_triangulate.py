"""Measurement of the SURVEY 8(f)-4 row: batched triangulation
(mba_triangulate, one thread per track) against the oracle restatement of
triangulate (miniba.py:458-530) on a bounded CPU sample of the same tracks.

    python scripts/bench_triangulate.py [--tracks 1000000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "src")]


def make_tracks(T, n_cams=12, seed=3):
    from gsrecon.scene import exp_so3
    rng = np.random.default_rng(seed)
    f, cx, cy = 520.0, 320.0, 240.0
    Rs = np.stack([exp_so3(rng.normal(0, 0.15, 3)) for _ in range(n_cams)])
    centers = np.stack([np.array([np.cos(a), 0.1 * np.sin(3 * a), np.sin(a)]) * 2.0 - np.array([0, 0, 2.0])
                        for a in np.linspace(-0.6, 0.6, n_cams)])
    ts = -np.einsum("nij,nj->ni", Rs, centers)
    m = rng.integers(2, 9, T)
    off = np.concatenate([[0], np.cumsum(m)]).astype(np.int64)
    cam = np.concatenate([np.sort(rng.choice(n_cams, size=k, replace=False)) for k in m]).astype(np.int32)
    X = rng.uniform(-0.5, 0.5, (T, 3)) + np.array([0.0, 0.0, 1.0])
    Xo = np.repeat(X, m, axis=0)
    pc = np.einsum("nij,nj->ni", Rs[cam], Xo) + ts[cam]
    uv = np.stack([f * pc[:, 0] / pc[:, 2] + cx, f * pc[:, 1] / pc[:, 2] + cy], 1) + rng.normal(0, 0.5, (len(cam), 2))
    return Rs, ts, cam, uv, off, (f, cx, cy)


def _peak():
    try:
        return json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except OSError:
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tracks", type=int, default=1_000_000)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--cpu-tracks", type=int, default=3000)
    a = ap.parse_args()
    import torch
    from oracle import miniba_oracle as O
    from paper_2506_05558_b200 import _lib
    from paper_2506_05558_b200._lib import ptr
    Rs, ts, cam, uv, off, (f, cx, cy) = make_tracks(a.tracks)
    T = a.tracks
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    dR, dt, dcam, duv, doff = dev(Rs), dev(ts), dev(cam), dev(uv), dev(off)
    X = torch.empty((T, 3), dtype=torch.float64, device="cuda")
    st = torch.empty(T, dtype=torch.int32, device="cuda")
    err = torch.empty(T, dtype=torch.float64, device="cuda")
    L = _lib.lib()

    def run():
        _lib.check(L.mba_triangulate(T, ptr(doff), ptr(dcam), ptr(duv), len(Rs), ptr(dR), ptr(dt), f, cx, cy,
                                     8.0, 0.5, 3, ptr(X), ptr(st), ptr(err), _lib.stream_ptr()),
                   "mba_triangulate")

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.steps)]
    for s in range(a.steps):
        ev[2 * s].record()
        run()
        ev[2 * s + 1].record()
    torch.cuda.synchronize()
    ms = float(np.median([ev[2 * s].elapsed_time(ev[2 * s + 1]) for s in range(a.steps)]))
    Xh, sh = X.cpu().numpy(), st.cpu().numpy()
    n = min(a.cpu_tracks, T)
    t0 = time.perf_counter()
    agree, worst = 0, 0.0
    for k in range(n):
        sl = slice(off[k], off[k + 1])
        Xr, sr = O.triangulate(Rs[cam[sl]], ts[cam[sl]], uv[sl], f, cx, cy)
        if sr == sh[k]:
            agree += 1
            if sr == 0:
                worst = max(worst, float(np.abs(Xr - Xh[k]).max()))
    t_cpu = time.perf_counter() - t0
    obs_bytes = off[-1] * (2 * 8 + 4) + T * (8 + 3 * 8 + 4 + 8)
    print(json.dumps({
        "metric": "batched triangulation (miniba.py:458-530): tracks/s",
        "config": {"tracks": T, "views_per_track": "2..8 (mean %.2f)" % (off[-1] / T), "cameras": len(Rs),
                   "gn_steps": 3, "data": "synthetic, 0.5 px noise"},
        "device": {"ms_per_call": ms, "tracks_per_s": T / (ms / 1e3),
                   "hbm_gbs_algorithmic": obs_bytes / (ms / 1e3) / 1e9, "kernel": "mba_triangulate"},
        "roofline": {"bytes_per_launch": float(obs_bytes), "achieved_gbs": obs_bytes / (ms / 1e3) / 1e9,
                     "peak_gbs": _peak(), "frac": obs_bytes / (ms / 1e3) / 1e9 / _peak(),
                     "larger_than_l2": bool(obs_bytes > 126 * 2 ** 20),
                     "bytes_model": "per observation cam 4 + uv 16 B; per track offset 8, X 24, status 4, err 8 B"},
        "cpu_oracle": {"tracks": n, "seconds": t_cpu, "tracks_per_s": n / t_cpu, "cores": 1,
                       "kind": "port (oracle/miniba_oracle.triangulate, numpy)"},
        "parity": {"tracks": n, "status_agree": agree, "max_abs_X_diff": worst,
                   "ok_fraction": float((sh == 0).mean())},
    }))


if __name__ == "__main__":
    main()
