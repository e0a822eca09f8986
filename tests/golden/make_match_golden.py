"""Golden fixture for device descriptor matching: random
256-bit descriptors for 8 frames with planted correspondences (a few flipped
bits, duplicates for ratio-test ties, unmatched distractors), matched for all 28
frame pairs by the UNMODIFIED reference `gsrecon.frontend.match`
(frontend.py:220-250). Run in the survey container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_match_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from gsrecon import frontend as F   # noqa: E402  (the reference package)


def main():
    rng = np.random.default_rng(77)
    n_frames, n_world = 8, 420
    world = rng.integers(0, 256, (n_world, 32), dtype=np.uint8)
    descs, offs = [], [0]
    for fr in range(n_frames):
        vis = np.sort(rng.choice(n_world, size=int(rng.integers(180, 300)), replace=False))
        d = world[vis].copy()
        flips = rng.integers(0, 256, (len(d), int(rng.integers(2, 12))))
        for r in range(len(d)):                        # a few noisy bits per observation
            for b in flips[r]:
                d[r, b // 8] ^= np.uint8(1 << (b % 8))
        extra = rng.integers(0, 256, (int(rng.integers(20, 60)), 32), dtype=np.uint8)   # distractors
        dup = d[rng.choice(len(d), size=5)]                                              # exact duplicates
        d = np.concatenate([d, extra, dup])
        d = d[rng.permutation(len(d))]
        descs.append(d)
        offs.append(offs[-1] + len(d))
    ia_all, ib_all, sc_all, poff = [], [], [], [0]
    pairs = []
    for i in range(n_frames):
        for j in range(i + 1, n_frames):
            ia, ib, sc = F.match(descs[i], descs[j])
            ia_all.append(ia); ib_all.append(ib); sc_all.append(sc)
            poff.append(poff[-1] + len(ia))
            pairs.append((i, j))
    np.savez_compressed(os.path.join(HERE, "match.npz"), desc=np.concatenate(descs), desc_off=np.array(offs),
                        pairs=np.array(pairs, dtype=np.int32), idx_a=np.concatenate(ia_all),
                        idx_b=np.concatenate(ib_all), score=np.concatenate(sc_all), pair_off=np.array(poff))
    print("frames", n_frames, "pairs", len(pairs), "matches", poff[-1])


if __name__ == "__main__":
    main()
