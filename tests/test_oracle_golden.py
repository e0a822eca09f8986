"""Pin the CPU oracle (oracle/miniba_oracle.py) against the reference's own
outputs, stored as golden fixtures by tests/golden/make_golden.py."""
import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, golden_ids, load_case
from oracle import miniba_oracle as O


def _rot_err(Ra, Rb):
    # chordal -> geodesic angle; accurate for tiny angles (arccos is not)
    return float(2.0 * np.arcsin(min(1.0, np.linalg.norm(Ra - Rb) / (2.0 * np.sqrt(2.0)))))


@pytest.mark.parametrize("path", golden_cases(), ids=golden_ids())
def test_oracle_matches_reference(path):
    prob, cfg, out = load_case(path)
    info = O.lm(prob, **cfg)
    i_star = O.plateau_index(out["costs"], tau=1e-9)
    n = i_star + 1
    assert np.array_equal(info["accepted"][:n], out["accepted"][:n])
    assert np.array_equal(info["evals"][:n], out["evals"][:n])
    np.testing.assert_allclose(info["lambdas"][:n], out["lambdas"][:n], rtol=0, atol=0)
    np.testing.assert_allclose(info["costs"][-1], out["costs"][-1], rtol=1e-9, atol=1e-20)
    for c in range(prob["R"].shape[0]):
        assert _rot_err(prob["R"][c], out["R"][c]) < 1e-9
    np.testing.assert_allclose(prob["t"], out["t"], rtol=1e-7, atol=1e-9)
    np.testing.assert_allclose(prob["focal"], float(out["focal"]), rtol=1e-9)


def test_oracle_stages_match_reference():
    z = np.load(f"{GOLDEN}/stages_smoke.npz")
    p = {k: z[k] for k in ("R", "t", "points", "cam_idx", "pt_idx", "uv", "fixed_cams")}
    p.update(focal=float(z["focal"]), cx=float(z["cx"]), cy=float(z["cy"]),
             optimize_focal=True, optimize_points=True)
    r, pc, bad = O.residuals(p)
    np.testing.assert_array_equal(r, z["r"])
    A, F, B = O.jacobians(p, pc, bad)
    np.testing.assert_allclose(A, z["A"], rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(B, z["B"], rtol=1e-13, atol=1e-12)
    np.testing.assert_array_equal(F, z["F"])
    w = O.robust_weights(np.linalg.norm(r, axis=1), 2.0)
    blocks = O.normal_equations(p, w, r, A, F, B)
    for got, name in zip(blocks, ("U", "g_c", "V", "g_p", "Wf")):
        np.testing.assert_allclose(got, z[name], rtol=1e-12, atol=1e-9)
    dc, dp = O.damped_step(*blocks, float(z["lam"]), "schur")
    np.testing.assert_allclose(dc, z["dc_schur"], rtol=1e-9, atol=1e-12)
    dc2, dp2 = O.damped_step(*blocks, float(z["lam"]), "dense")
    np.testing.assert_allclose(dc2, z["dc_dense"], rtol=1e-9, atol=1e-12)


def test_oracle_pose_lm_matches_reference():
    z = np.load(f"{GOLDEN}/pose_lm.npz")
    R, t, c = O.pose_lm(z["R0"], z["t0"], z["X"], z["uv"], float(z["focal"]),
                        float(z["cx"]), float(z["cy"]), int(z["iters"]))
    np.testing.assert_allclose(c, z["cost_out"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(t, z["t_out"], rtol=1e-9, atol=1e-12)
    R, t, c = O.pose_lm(z["Rf0"], z["tf0"], z["Xf"], z["uvf"], float(z["focal"]),
                        float(z["cx"]), float(z["cy"]), int(z["iters_f"]))
    np.testing.assert_allclose(c, z["costf_out"], rtol=1e-10)


def test_plateau_index():
    costs = np.array([10.0, 5.0, 4.0, 4.0 + 1e-12, 4.0])
    assert O.plateau_index(costs) == 1
    assert O.plateau_index(np.array([3.0, 3.0])) == 0


def test_cauchy_loss_consistency():
    e = np.linspace(0, 20, 101)
    d = 2.0
    # d rho / d e = w * e for IRLS
    h = 1e-6
    rho = lambda x: O.robust_cost(np.array([x]), d, "cauchy")
    for x in e[1:]:
        g = (rho(x + h) - rho(x - h)) / (2 * h)
        w = O.robust_weights(np.array([x]), d, "cauchy")[0]
        assert abs(g - w * x) < 1e-6 * max(1.0, abs(g))


def test_empty_problem_raises():
    p = dict(R=np.eye(3)[None], t=np.zeros((1, 3)), focal=500.0, cx=0.0, cy=0.0,
             points=np.zeros((0, 3)), cam_idx=np.zeros(0, np.int64), pt_idx=np.zeros(0, np.int64),
             uv=np.zeros((0, 2)), fixed_cams=np.array([True]), optimize_focal=True,
             optimize_points=True)
    with pytest.raises(ValueError):
        O.lm(p)
