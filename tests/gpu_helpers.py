"""Helpers shared by the GPU parity tests: run the device solver on oracle-
layout problem dicts and compare against oracle / golden outputs under the
adopted parity rule."""
import numpy as np

from oracle import miniba_oracle as O

# BASELINE.json north-star final-value tolerances
COST_RTOL = 1e-4
ROT_TOL = 1e-4
TRANS_RTOL = 1e-4


def run_device(problems, lm_cfg, precision="mixed", kernel="auto"):
    from paper_2506_05558_b200 import solver
    hb = solver.pack_problems(problems)
    db = solver.to_device(hb)
    prm = solver.LmParams(lambda_init=lm_cfg.get("lambda_init", 1e-5), nu=lm_cfg.get("nu", 2.0),
                          delta=lm_cfg.get("delta", 2.0), max_iters=lm_cfg.get("max_iters", 200),
                          loss=lm_cfg.get("loss", "huber"), precision=precision,
                          fail_at=tuple(lm_cfg.get("fail_at", ())), kernel=kernel)
    sol = solver.solve(db, prm)
    R, t, f, X = (sol.R.cpu().numpy(), sol.t.cpu().numpy(), sol.focal.cpu().numpy(),
                  sol.points.cpu().numpy())
    outs = []
    for b in range(len(problems)):
        info = solver.fetch(sol, b)
        c0, c1 = hb.cam_off[b], hb.cam_off[b + 1]
        p0, p1 = hb.pt_off[b], hb.pt_off[b + 1]
        info.update(R=R[c0:c1], t=t[c0:c1], focal=float(f[b]), points=X[p0:p1])
        outs.append(info)
    return outs


def rot_err(Ra, Rb):
    return float(2.0 * np.arcsin(min(1.0, np.linalg.norm(Ra - Rb) / (2.0 * np.sqrt(2.0)))))


def assert_parity(dev, ref_costs, ref_acc, ref_evals, ref_lams, ref_R, ref_t, ref_focal,
                  tau=1e-9, kappa=0.0, label=""):
    """Traces identical through i*; final values within the BASELINE tolerances."""
    i_star = O.plateau_index(ref_costs, tau=tau, kappa=kappa)
    n = i_star + 1
    assert len(dev["accepted"]) >= n, f"{label}: device stopped at {len(dev['accepted'])} < i*+1={n}"
    np.testing.assert_array_equal(dev["accepted"][:n], ref_acc[:n], err_msg=f"{label} accepted")
    np.testing.assert_array_equal(dev["evals"][:n], ref_evals[:n], err_msg=f"{label} evals")
    np.testing.assert_allclose(dev["lambdas"][:n], ref_lams[:n], rtol=1e-12, err_msg=f"{label} lambdas")
    c_ref = ref_costs[-1]
    assert abs(dev["costs"][-1] - c_ref) <= COST_RTOL * abs(c_ref) + 1e-12, \
        f"{label}: final cost {dev['costs'][-1]} vs {c_ref}"
    for c in range(len(ref_R)):
        assert rot_err(dev["R"][c], ref_R[c]) <= ROT_TOL, f"{label}: rotation {c}"
    scale = max(np.linalg.norm(ref_t, axis=1).max(), 1e-12)
    assert np.abs(dev["t"] - ref_t).max() <= TRANS_RTOL * scale, f"{label}: translation"
    assert abs(dev["focal"] - ref_focal) <= 1e-4 * abs(ref_focal), f"{label}: focal"
    # accepted costs never increase (smoke_miniba.py:79-81)
    assert np.all(np.diff(dev["costs"]) <= 1e-12 * max(1.0, abs(dev["costs"][0])))
