"""Oracle restatements of the SURVEY 8(f) rows against the unmodified
reference's outputs: triangulate (miniba.py:458-530; tests/golden/triangulate.npz,
600 tracks of 2..8 views incl. tiny baselines, outliers and points behind the
cameras) and frontend.match (frontend.py:220-250; tests/golden/match.npz)."""
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


def test_oracle_match_matches_reference():
    """The oracle's descriptor matching restatement (frontend.py:220-250)
    against the reference's outputs for 28 frame pairs (tests/golden/match.npz)."""
    z = np.load(f"{GOLDEN}/match.npz")
    off, po = z["desc_off"], z["pair_off"]
    for p, (i, j) in enumerate(z["pairs"]):
        ia, ib, sc = O.match(z["desc"][off[i]:off[i + 1]], z["desc"][off[j]:off[j + 1]])
        np.testing.assert_array_equal(ia, z["idx_a"][po[p]:po[p + 1]])
        np.testing.assert_array_equal(ib, z["idx_b"][po[p]:po[p + 1]])
        np.testing.assert_array_equal(sc, z["score"][po[p]:po[p + 1]])


def test_track_grouping_with_oracle_matcher_matches_reference():
    """The host half of track building (flow filter + union-find grouping in
    gsrecon._bootstrap) fed by the oracle matcher reproduces the reference's
    build_tracks(features, default_matcher) exactly (tests/golden/tracks.npz)."""
    from gsrecon._bootstrap import build_tracks, filter_matches_flow
    z = np.load(f"{GOLDEN}/tracks.npz")
    off = z["off"]
    feats = [(z["kp"][off[f]:off[f + 1]], z["desc"][off[f]:off[f + 1]]) for f in range(len(off) - 1)]

    def matcher(fa, fb):
        ia, ib, sc = O.match(fa[1], fb[1])
        keep = filter_matches_flow(fa[0], fb[0], ia, ib)
        return ia[keep], ib[keep], sc[keep]
    tracks = build_tracks(feats, matcher)
    flat = np.array([(ti, fr, k, x, y) for ti, tr in enumerate(tracks) for (fr, k, x, y) in tr])
    np.testing.assert_array_equal(flat, z["tracks"])
