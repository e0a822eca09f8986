"""Golden fixture for track building: 8 frames of synthetic
keypoints + 256-bit descriptors (a 3D scene projected into an arc of cameras,
descriptor noise, distractors), grouped into tracks by the UNMODIFIED reference
`build_tracks(features, default_matcher)` (miniba.py:555-602: frontend.match +
filter_matches_flow + union-find). Run in the survey container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_tracks_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from gsrecon import miniba as M            # noqa: E402  (the reference package)
from gsrecon.scene import exp_so3          # noqa: E402


def main():
    rng = np.random.default_rng(31)
    n_frames, n_pts = 8, 400
    f, cx, cy = 520.0, 320.0, 240.0
    X = rng.uniform(-0.8, 0.8, (n_pts, 3)) + np.array([0, 0, 3.0])
    world_desc = rng.integers(0, 256, (n_pts, 32), dtype=np.uint8)
    feats = []
    for fr in range(n_frames):
        ang = -0.25 + 0.5 * fr / (n_frames - 1)
        R = exp_so3(np.array([0.0, ang, 0.0]))
        t = -R @ np.array([3.0 * np.sin(ang), 0.0, 3.0 - 3.0 * np.cos(ang)])
        pc = X @ R.T + t
        uv = np.stack([f * pc[:, 0] / pc[:, 2] + cx, f * pc[:, 1] / pc[:, 2] + cy], 1)
        vis = np.flatnonzero((rng.random(n_pts) < 0.75) & (uv[:, 0] > 0) & (uv[:, 0] < 640)
                             & (uv[:, 1] > 0) & (uv[:, 1] < 480))
        kp = uv[vis] + rng.normal(0, 0.3, (len(vis), 2))
        d = world_desc[vis].copy()
        for r in range(len(d)):
            for b in rng.integers(0, 256, 6):
                d[r, b // 8] ^= np.uint8(1 << (b % 8))
        extra_kp = rng.uniform([0, 0], [640, 480], (30, 2))
        extra_d = rng.integers(0, 256, (30, 32), dtype=np.uint8)
        kp = np.concatenate([kp, extra_kp])
        d = np.concatenate([d, extra_d])
        perm = rng.permutation(len(kp))
        feats.append((kp[perm], d[perm]))
    tracks = M.build_tracks(feats, M.default_matcher)
    flat = np.array([(ti, fr, k, x, y) for ti, tr in enumerate(tracks) for (fr, k, x, y) in tr])
    np.savez_compressed(os.path.join(HERE, "tracks.npz"),
                        kp=np.concatenate([fe[0] for fe in feats]), desc=np.concatenate([fe[1] for fe in feats]),
                        off=np.concatenate([[0], np.cumsum([len(fe[0]) for fe in feats])]), tracks=flat)
    print("frames", n_frames, "tracks", len(tracks), "observations", len(flat))


if __name__ == "__main__":
    main()
