"""Golden fixture for batched triangulation: random tracks of
2..8 views through the UNMODIFIED reference `gsrecon.miniba.triangulate`
(miniba.py:458-530), including degenerate ones (tiny baseline, parallel rays,
points behind a camera, outlier pixels). Run in the survey container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_triangulate_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from gsrecon import miniba as M            # noqa: E402  (the reference package)
from gsrecon.scene import CameraIntrinsics, Pose, exp_so3   # noqa: E402

CODES = {"need at least two": 1, "baseline angle": 2, "parallel rays": 3, "behind a camera": 4,
         "mean reprojection": 5}


def main():
    rng = np.random.default_rng(2024)
    f, cx, cy = 520.0, 320.0, 240.0
    intr = CameraIntrinsics(f, cx, cy, 640, 480)
    n_cams = 12
    Rs = np.stack([exp_so3(rng.normal(0, 0.15, 3)) for _ in range(n_cams)])
    centers = np.stack([np.array([np.cos(a), 0.1 * np.sin(3 * a), np.sin(a)]) * 2.0 - np.array([0, 0, 2.0])
                        for a in np.linspace(-0.6, 0.6, n_cams)])
    ts = -np.einsum("nij,nj->ni", Rs, centers)
    cams, offs, uvs, kinds = [], [0], [], []
    for tr in range(600):
        kind = rng.integers(0, 10)
        m = int(rng.integers(2, 9))
        sel = np.sort(rng.choice(n_cams, size=m, replace=False))
        X = rng.uniform(-0.5, 0.5, 3) + np.array([0.0, 0.0, 1.0])
        if kind == 0:          # tiny baseline: the same camera twice (identical rays)
            sel = np.array([sel[0]] * m)
        pc = np.einsum("nij,j->ni", Rs[sel], X) + ts[sel]
        uv = np.stack([f * pc[:, 0] / pc[:, 2] + cx, f * pc[:, 1] / pc[:, 2] + cy], 1)
        uv += rng.normal(0, 0.5, uv.shape)
        if kind == 1:          # one wild outlier pixel
            uv[0] += rng.uniform(100, 300, 2)
        if kind == 2:          # a point behind the cameras
            uv = np.stack([f * (-pc[:, 0]) / pc[:, 2] + cx, f * (-pc[:, 1]) / pc[:, 2] + cy], 1)
        cams.append(sel)
        uvs.append(uv)
        offs.append(offs[-1] + m)
        kinds.append(kind)
    cam = np.concatenate(cams).astype(np.int32)
    uv = np.concatenate(uvs)
    offs = np.array(offs, dtype=np.int64)
    X_out = np.zeros((len(kinds), 3))
    status = np.zeros(len(kinds), dtype=np.int32)
    for k in range(len(kinds)):
        sl = slice(offs[k], offs[k + 1])
        poses = [Pose.from_matrix(Rs[c], ts[c]) if hasattr(Pose, "from_matrix") else None for c in cam[sl]]
        try:
            X_out[k] = M.triangulate(poses, uv[sl], intr)
        except M.TriangulationFailure as e:
            msg = str(e)
            status[k] = next(v for key, v in CODES.items() if key in msg)
            X_out[k] = np.nan
    np.savez_compressed(os.path.join(HERE, "triangulate.npz"), R=Rs, t=ts, cam=cam, uv=uv, obs_off=offs,
                        focal=f, cx=cx, cy=cy, X=X_out, status=status)
    print("tracks", len(kinds), "status counts", np.bincount(status, minlength=6).tolist())


if __name__ == "__main__":
    main()
