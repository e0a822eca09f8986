"""The oracle's triangulation restatement (miniba.py:458-530) against the
unmodified reference's outputs (tests/golden/triangulate.npz: 600 tracks of
2..8 views incl. tiny baselines, outliers and points behind the cameras)."""
import numpy as np

from conftest import GOLDEN
from oracle import miniba_oracle as O


def test_oracle_triangulate_matches_reference():
    z = np.load(f"{GOLDEN}/triangulate.npz")
    off = z["obs_off"]
    for k in range(len(off) - 1):
        sl = slice(off[k], off[k + 1])
        cams = z["cam"][sl]
        X, st = O.triangulate(z["R"][cams], z["t"][cams], z["uv"][sl], float(z["focal"]), float(z["cx"]),
                              float(z["cy"]))
        assert st == z["status"][k], k
        if st == 0:
            np.testing.assert_allclose(X, z["X"][k], rtol=0, atol=1e-12)
