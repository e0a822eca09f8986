"""Measurement of the SURVEY 8(f)-3 row: exhaustive pairwise descriptor
matching of a bootstrap window (every frame pair; frontend.match as called by
build_tracks, miniba.py:555-591) in one device call (mba_match_pairs) against
the oracle restatement on CPU, with parity on the same descriptors.

    python scripts/bench_match.py [--frames 8 --per-frame 2000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "src")]


def make(frames, per, seed=5):
    rng = np.random.default_rng(seed)
    world = rng.integers(0, 256, (int(per * 1.4), 32), dtype=np.uint8)
    out = []
    for _ in range(frames):
        vis = rng.choice(len(world), size=per, replace=False)
        d = world[vis].copy()
        nb = rng.integers(0, 256, (per, 8))
        rows = np.repeat(np.arange(per), 8)
        np.bitwise_xor.at(d, (rows, (nb // 8).reshape(-1)), (1 << (nb % 8)).reshape(-1).astype(np.uint8))
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--per-frame", type=int, default=2000)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    import torch
    from gsrecon import miniba as M
    from oracle import miniba_oracle as O
    descs = make(a.frames, a.per_frame)
    pairs = [(i, j) for i in range(a.frames) for j in range(i + 1, a.frames)]
    res = M.match_batch(descs, pairs)     # warm-up + result
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        M.match_batch(descs, pairs)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    same = 0
    for p, (i, j) in enumerate(pairs):
        ia, ib, sc = O.match(descs[i], descs[j])
        same += int(np.array_equal(ia, res[p][0]) and np.array_equal(ib, res[p][1]) and np.array_equal(sc, res[p][2]))
    t_cpu = time.perf_counter() - t0
    print(json.dumps({
        "metric": "exhaustive pairwise descriptor matching of a window (build_tracks' matcher)",
        "config": {"frames": a.frames, "descriptors_per_frame": a.per_frame, "pairs": len(pairs),
                   "distances": a.per_frame ** 2 * len(pairs)},
        "device": {"seconds_per_window_host_to_host": float(np.median(ts)), "kernel": "mba_match_pairs",
                   "note": "includes H2D of the descriptors and D2H of the matches"},
        "cpu_oracle": {"seconds_per_window": t_cpu, "cores": 1, "kind": "port (oracle/miniba_oracle.match, numpy)"},
        "parity": {"pairs_identical": same, "pairs": len(pairs), "matches": int(sum(len(r[0]) for r in res))},
    }))


if __name__ == "__main__":
    main()
