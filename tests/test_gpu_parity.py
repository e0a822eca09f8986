"""Device parity: the sm_100a solver against the reference's golden outputs
and against the CPU oracle on seeded synthetic problems (SURVEY.md 8c rule:
accept/reject, backtrack counts and lambda identical through the plateau
index i*; final cost rel <= 1e-4, rotation <= 1e-4 rad, translation rel <= 1e-4)."""
import numpy as np
import pytest

from conftest import golden_cases, golden_ids, load_case
from gpu_helpers import assert_parity, rot_err, run_device
from oracle import miniba_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kernel", ["cta", "grid", "v4"])
@pytest.mark.parametrize("path", golden_cases(), ids=golden_ids())
def test_solver_matches_reference_golden(path, kernel, cuda_ok):
    """float64 mode (the API default): exact trace parity through i* (fp64
    rule) and the BASELINE final-value tolerances on every golden case, for
    the cluster-resident, CTA-per-problem and whole-GPU kernels."""
    prob, cfg, out = load_case(path)
    dev = run_device([prob], cfg, "f64", kernel=kernel)[0]
    assert_parity(dev, out["costs"], out["accepted"], out["evals"], out["lambdas"], out["R"],
                  out["t"], float(out["focal"]), label=f"{path}:f64")


# The one golden case mixed precision does not reproduce: 20 % outliers under
# Huber, a trace that is pre-plateau for all 40 iterations; at iteration 20 the
# reference accepts the 1/8 step by a relative margin of ~1e-5 and the fp32
# Schur step (fp32 Jacobians) misses it by a hair, accepting at 1/16 instead.
# A property of fp32 linearisation, not of the kernel; f64 (the default)
# reproduces it exactly.
MIXED_KNOWN_DEPARTURES = {"outliers20"}


def _mixed_cases():
    out = []
    for p in golden_cases():
        name = p.split("lm_")[-1][:-4]
        marks = [pytest.mark.xfail(strict=True, reason="fp32 near-tie backtrack decision")] \
            if name in MIXED_KNOWN_DEPARTURES else []
        out.append(pytest.param(p, id=name, marks=marks))
    return out


@pytest.mark.parametrize("path", _mixed_cases())
def test_mixed_precision_against_golden(path, cuda_ok):
    """Mixed precision (fp32 linearise/Schur/LDL^T, fp64 state and cost) on
    the cluster-resident kernel, held to the SAME rule as f64: traces identical
    through the fp64 plateau index, BASELINE final tolerances on raw R, t, f.
    (The gauge-consistent step projection in mba_v4.cu is what keeps fp32
    Jacobians from drifting along the free scale gauge of one-fixed-camera
    problems.)"""
    prob, cfg, out = load_case(path)
    dev = run_device([prob], cfg, "mixed", kernel="v4")[0]
    assert_parity(dev, out["costs"], out["accepted"], out["evals"], out["lambdas"], out["R"],
                  out["t"], float(out["focal"]), label=f"{path}:mixed")


@pytest.mark.parametrize("kernel", ["cta", "v4"])
@pytest.mark.parametrize("precision", ["mixed", "f64"])
def test_batched_matches_oracle_and_is_shard_invariant(precision, kernel, cuda_ok):
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(12, n_cams=8, K=2000, seed=3)
    probs = [b.problem(i) for i in range(12)]
    cfg = dict(max_iters=200)
    dev_all = run_device(probs, cfg, precision, kernel)
    dev_a = run_device(probs[:5], cfg, precision, kernel)
    dev_b = run_device(probs[5:], cfg, precision, kernel)
    for i, d in enumerate(dev_all):
        other = dev_a[i] if i < 5 else dev_b[i - 5]
        # bit-identical regardless of how the batch is sharded
        np.testing.assert_array_equal(d["costs"], other["costs"])
        np.testing.assert_array_equal(d["points"], other["points"])
        np.testing.assert_array_equal(d["R"], other["R"])
    for i in range(0, 12, 3):
        p = b.problem(i)
        ref = O.lm(p, max_iters=200)
        assert_parity(dev_all[i], ref["costs"], ref["accepted"], ref["evals"], ref["lambdas"],
                      p["R"], p["t"], p["focal"], label=f"batch[{i}]")


def test_deterministic_repeat(cuda_ok):
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(4, n_cams=8, K=2000, seed=9)
    probs = [b.problem(i) for i in range(4)]
    a = run_device(probs, dict(max_iters=50))
    c = run_device(probs, dict(max_iters=50))
    for x, y in zip(a, c):
        np.testing.assert_array_equal(x["costs"], y["costs"])
        np.testing.assert_array_equal(x["points"], y["points"])


@pytest.mark.parametrize("kernel", ["cta", "grid", "auto"])
@pytest.mark.parametrize("precision", ["mixed", "f64"])
def test_paper_scale_single_problem(precision, kernel, cuda_ok):
    """BASELINE config 2: 8 frames, K = 20k, Huber."""
    from paper_2506_05558_b200.synth import make_batch
    p = make_batch(1, n_cams=8, K=20000, seed=2).problem(0)
    dev = run_device([p], dict(max_iters=200), precision, kernel)[0]
    ref = O.lm(p, max_iters=200)
    assert_parity(dev, ref["costs"], ref["accepted"], ref["evals"], ref["lambdas"], p["R"], p["t"],
                  p["focal"], label="cfg2")


@pytest.mark.parametrize("kernel", ["cta", "grid"])
def test_cauchy_outliers_many_cameras(kernel, cuda_ok):
    """Config-5 shape at oracle-friendly size: 16 frames, 20% outliers, Cauchy
    (extension; parity against the oracle only -- unpinned by the reference)."""
    from paper_2506_05558_b200.synth import make_batch
    # 25 iterations: at iteration 27 lambda has decayed to 7e-14 and the
    # oracle's cho_factor fails on the near-singular (scale-gauge) system, a
    # roundoff event that a differently ordered factorisation need not repeat.
    p = make_batch(1, n_cams=16, K=6000, seed=5, outlier_frac=0.2).problem(0)
    dev = run_device([p], dict(max_iters=25, loss="cauchy"), "f64", kernel)[0]
    ref = O.lm(p, max_iters=25, loss="cauchy")
    assert_parity(dev, ref["costs"], ref["accepted"], ref["evals"], ref["lambdas"], p["R"], p["t"],
                  p["focal"], label="cauchy16")


@pytest.mark.parametrize("kernel", ["cta", "grid", "v4"])
def test_fault_injection_matches_oracle(kernel, cuda_ok):
    from paper_2506_05558_b200.synth import make_batch
    p = make_batch(1, n_cams=8, K=2000, seed=4).problem(0)
    fail = (0, 1, 4)
    dev = run_device([p], dict(max_iters=200, fail_at=fail), "f64", kernel)[0]
    ref = O.lm(p, max_iters=200, fail_at=fail)
    for i in fail:
        assert not dev["accepted"][i] and dev["evals"][i] == 0
    assert_parity(dev, ref["costs"], ref["accepted"], ref["evals"], ref["lambdas"], p["R"], p["t"],
                  p["focal"], label="fault")


def test_max_iters_zero_and_one(cuda_ok):
    from paper_2506_05558_b200.synth import make_batch
    p = make_batch(1, n_cams=5, K=600, seed=8).problem(0)
    d0 = run_device([p], dict(max_iters=0))[0]
    assert len(d0["costs"]) == 1 and len(d0["accepted"]) == 0
    np.testing.assert_array_equal(d0["points"], p["points"])
    ref = O.lm(dict(p), max_iters=1)
    d1 = run_device([p], dict(max_iters=1), "f64")[0]
    assert d1["accepted"].tolist() == ref["accepted"].tolist()
    np.testing.assert_allclose(d1["costs"], ref["costs"], rtol=1e-9)


@pytest.mark.parametrize("kernel", ["cta", "v4"])
def test_all_cameras_fixed_focal_only(kernel, cuda_ok):
    """C = 1 (focal only) edge shape."""
    from paper_2506_05558_b200.synth import make_batch
    p = make_batch(1, n_cams=4, K=500, seed=6).problem(0)
    p["fixed_cams"] = np.ones(4, dtype=bool)
    dev = run_device([p], dict(max_iters=40), "f64", kernel)[0]
    ref = O.lm(dict(p), max_iters=40)
    np.testing.assert_allclose(dev["costs"][-1], ref["costs"][-1], rtol=1e-6)
    assert dev["accepted"][:3].tolist() == ref["accepted"][:3].tolist()


@pytest.mark.parametrize("other", ["grid", "v4"])
def test_kernels_agree(other, cuda_ok):
    """All kernels implement the same arithmetic per problem up to reduction
    order: traces agree through i* and final costs to 1e-9 on 64 problems."""
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(64, n_cams=8, K=2000, seed=21)
    probs = [b.problem(i) for i in range(64)]
    w = run_device(probs, dict(max_iters=200), "f64", other)
    c = run_device(probs, dict(max_iters=200), "f64", "cta")
    for x, y in zip(w, c):
        i_star = O.plateau_index(y["costs"])
        assert np.array_equal(x["accepted"][:i_star + 1], y["accepted"][:i_star + 1])
        assert abs(x["costs"][-1] - y["costs"][-1]) <= 1e-9 * y["costs"][-1]


def test_grid_mode_config5_shape(cuda_ok):
    """32 cameras, 20% outliers, Cauchy, across the whole GPU (cooperative
    grid): trace parity with the oracle for 6 iterations at K = 40k (oracle-
    sized version of BASELINE config 5)."""
    from paper_2506_05558_b200.synth import make_batch
    p = make_batch(1, n_cams=32, K=40000, seed=12, outlier_frac=0.2).problem(0)
    dev = run_device([p], dict(max_iters=6, loss="cauchy"), "f64", "grid")[0]
    ref = O.lm(p, max_iters=6, loss="cauchy")
    assert_parity(dev, ref["costs"], ref["accepted"], ref["evals"], ref["lambdas"], p["R"], p["t"],
                  p["focal"], label="grid32")


def test_cluster_kernel_plans(cuda_ok):
    """The auto path takes the cluster-resident kernel: one CTA per config-4
    problem, a 16 (f64) / 8 (mixed) CTA cluster for a config-2 problem."""
    from paper_2506_05558_b200 import solver
    from paper_2506_05558_b200.synth import make_batch
    small = solver.to_device(solver.pack_synth(make_batch(4, n_cams=8, K=2000, seed=1)))
    big = solver.to_device(solver.pack_synth(make_batch(1, n_cams=8, K=20000, seed=2)))
    assert solver.plan(small, solver.LmParams(precision="f64")) == 1
    assert solver.plan(small, solver.LmParams(precision="mixed")) == 1
    assert solver.plan(big, solver.LmParams(precision="f64")) == 16
    assert solver.plan(big, solver.LmParams(precision="mixed")) == 8
    # a full batch of config-3 problems: the planner scores the fitting cluster
    # sizes by resident clusters (B200: 9 in both precisions)
    full = solver.to_device(solver.pack_synth(make_batch(64, n_cams=8, K=20000, seed=3)))
    assert solver.plan(full, solver.LmParams(precision="f64")) in (9, 10, 12, 16)
    assert solver.plan(full, solver.LmParams(precision="mixed")) in (8, 9, 10, 12, 16)


@pytest.mark.parametrize("R", [9, 10, 12])
@pytest.mark.parametrize("precision", ["mixed", "f64"])
def test_non_power_of_two_clusters(R, precision, cuda_ok, monkeypatch):
    """Cluster sizes that tile a GPC better (9/10/12 CTAs, chosen for full
    batches of large problems) split observations at point boundaries and sum
    through DSMEM exactly like the power-of-two plans: oracle parity, and the
    default one-CTA plan reaches the same final costs."""
    from paper_2506_05558_b200 import solver
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(4, n_cams=8, K=3000, seed=31)
    probs = [b.problem(i) for i in range(4)]
    cfg = dict(max_iters=200)
    base = run_device(probs, cfg, precision, "v4")
    monkeypatch.setenv("MBA_V4_R", str(R))
    assert solver.plan(solver.to_device(solver.pack_problems(probs)),
                       solver.LmParams(precision=precision)) == R
    dev = run_device(probs, cfg, precision, "v4")
    for i in range(4):
        assert dev[i]["status"] == base[i]["status"]
        np.testing.assert_allclose(dev[i]["costs"][-1], base[i]["costs"][-1], rtol=1e-6)
    for i in (0, 3):
        q = b.problem(i)                 # the oracle rebinds q's R, t, focal, points
        ref = O.lm(q, max_iters=200)
        assert_parity(dev[i], ref["costs"], ref["accepted"], ref["evals"], ref["lambdas"],
                      q["R"], q["t"], q["focal"], label=f"R{R}[{i}]")


def test_plan_overflow_is_resolved_by_cta_kernel(cuda_ok, monkeypatch):
    """Problems whose slice does not fit the cluster kernel's shared-memory
    plan are flagged and re-solved by the CTA kernel in the same mba_solve:
    results match the oracle either way."""
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(6, n_cams=8, K=2000, seed=11)
    probs = [b.problem(i) for i in range(6)]
    normal = run_device(probs, dict(max_iters=200), "f64", "auto")
    monkeypatch.setenv("MBA_V4_ARENA_CAP", "20000")   # every problem overflows
    forced = run_device(probs, dict(max_iters=200), "f64", "auto")
    for i in (0, 3):
        ref = O.lm(probs[i], max_iters=200)
        for dev in (normal[i], forced[i]):
            assert dev["status"] in (1, 2)
            assert_parity(dev, ref["costs"], ref["accepted"], ref["evals"], ref["lambdas"],
                          probs[i]["R"], probs[i]["t"], probs[i]["focal"], label=f"overflow[{i}]")


def test_heterogeneous_batch_cluster_kernel(cuda_ok):
    """One batch mixing camera counts (3..8), sizes (K 300..3000), free /
    fixed focal, fixed points and two fixed cameras: every problem matches the
    oracle under the parity rule (the cluster kernel plans for the batch maxima
    and handles each problem's own layout)."""
    from paper_2506_05558_b200.synth import make_batch
    probs = []
    specs = [(3, 300, True, True), (8, 3000, True, True), (5, 1200, False, True), (8, 2000, True, False),
             (6, 800, True, True), (4, 600, False, False), (8, 2400, True, True)]
    for s, (n, K, of, op) in enumerate(specs):
        p = make_batch(1, n_cams=n, K=K, seed=100 + s).problem(0)
        p["optimize_focal"] = of
        p["optimize_points"] = op
        if s == 6:
            p["fixed_cams"] = np.array([True, True] + [False] * (n - 2))
        probs.append(p)
    devs = run_device(probs, dict(max_iters=100), "f64", "auto")
    for i, (p, dev) in enumerate(zip(probs, devs)):
        q = dict(p)                      # the oracle rebinds q's R, t, focal, points
        ref = O.lm(q, max_iters=100)
        assert_parity(dev, ref["costs"], ref["accepted"], ref["evals"], ref["lambdas"], q["R"], q["t"],
                      q["focal"], label=f"hetero[{i}]")
        if not p["optimize_points"]:
            np.testing.assert_array_equal(dev["points"], p["points"])


def _cfg5_golden():
    import os
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "stress_cfg5_huber.npz"))
    d = {k: z[k] for k in z.files}
    prob = dict(R=d["R"].astype(np.float64), t=d["t"].astype(np.float64), focal=float(d["focal"]),
                cx=float(d["cx"]), cy=float(d["cy"]), points=d["points"].astype(np.float64),
                cam_idx=d["cam_idx"].astype(np.int64), pt_idx=d["pt_idx"].astype(np.int64),
                uv=d["uv"].astype(np.float64), fixed_cams=d["fixed_cams"].astype(bool),
                optimize_focal=True, optimize_points=True)
    out = {k[4:]: d[k] for k in d if k.startswith("out_")}
    return prob, out, int(d["max_iters"])


@pytest.mark.parametrize("precision", ["f64", "mixed"])
def test_config5_stress_matches_reference_all_50_iterations(precision, cuda_ok):
    """BASELINE config 5 at its stated size -- 32 frames, K = 200k, 20 %
    outliers, 50 LM iterations -- pinned to the UNMODIFIED reference (Huber,
    the reference's only loss; tests/golden/make_cfg5_golden.py, ~23 min of
    CPU). SURVEY 8c: the whole trace is pre-plateau, so all 50 accept/reject
    flags, backtrack counts and lambdas must be identical; final values within
    the BASELINE tolerances."""
    prob, out, iters = _cfg5_golden()
    assert len(prob["uv"]) == 200000 and len(prob["R"]) == 32
    dev = run_device([prob], dict(max_iters=iters), precision, "auto")[0]
    n = len(out["accepted"])
    assert n == iters and len(dev["accepted"]) == n
    np.testing.assert_array_equal(dev["accepted"], out["accepted"])
    np.testing.assert_array_equal(dev["evals"], out["evals"])
    np.testing.assert_allclose(dev["lambdas"], out["lambdas"], rtol=1e-12)
    assert_parity(dev, out["costs"], out["accepted"], out["evals"], out["lambdas"], out["R"], out["t"],
                  float(out["focal"]), label=f"cfg5:{precision}")


def _oracle_job(args):
    import os
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    p, iters = args
    ref = O.lm(p, max_iters=iters)
    return ref, p["R"], p["t"], p["focal"]


@pytest.mark.parametrize("precision", ["f64", "mixed"])
def test_config3_full_batch_on_production_plan(precision, cuda_ok):
    """BASELINE config 3 shape at its stated size: a full batch of 64 problems
    of 8 frames x K = 20k goes through the auto planner's production plan
    (B200: 9-CTA clusters in both precisions, scored by resident clusters),
    and problems spread over the batch match the CPU oracle under the parity
    rule."""
    from concurrent.futures import ProcessPoolExecutor
    from paper_2506_05558_b200 import solver
    from paper_2506_05558_b200.synth import make_batch
    b = make_batch(64, n_cams=8, K=20000, seed=0)
    probs = [b.problem(i) for i in range(64)]
    plan = solver.plan(solver.to_device(solver.pack_problems(probs)), solver.LmParams(precision=precision))
    assert plan == 9, plan
    dev = run_device(probs, dict(max_iters=200), precision, "auto")
    pick = (0, 21, 42, 63)
    with ProcessPoolExecutor(4) as ex:
        refs = list(ex.map(_oracle_job, [(b.problem(i), 200) for i in pick]))
    for i, (ref, R, t, f) in zip(pick, refs):
        assert dev[i]["status"] in (1, 2)
        assert_parity(dev[i], ref["costs"], ref["accepted"], ref["evals"], ref["lambdas"], R, t, f,
                      label=f"cfg3[{i}]:{precision}")


def test_more_than_32_cameras_take_the_stage_kernel_loop(cuda_ok):
    """The reference lm_solve accepts any camera count; problems beyond the
    fused kernel's 32 cameras run the stage-kernel LM loop (device stages,
    host-driven; gsrecon.miniba._lm_stages) and match the oracle."""
    from gsrecon.config import LmConfig
    from gsrecon.miniba import BaProblem, MAX_FUSED_CAMS, lm_solve, lm_solve_batch
    from paper_2506_05558_b200.synth import make_batch
    p = make_batch(1, n_cams=40, K=3000, seed=51).problem(0)
    assert len(p["R"]) > MAX_FUSED_CAMS
    q = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in p.items()}
    ref = O.lm(q, max_iters=30)
    prob = BaProblem(**{k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in p.items()})
    info = lm_solve(prob, LmConfig(max_iters=30))
    dev = dict(info, R=prob.R, t=prob.t, focal=prob.focal)
    assert_parity(dev, ref["costs"], ref["accepted"], ref["evals"], ref["lambdas"], q["R"], q["t"], q["focal"],
                  label="40cams")
    # mixed batch: the 40-camera problem beside fused-kernel problems
    small = make_batch(2, n_cams=8, K=1000, seed=52)
    probs = [BaProblem(**small.problem(0)),
             BaProblem(**{k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in p.items()}),
             BaProblem(**small.problem(1))]
    res = lm_solve_batch(probs, LmConfig(max_iters=30))
    np.testing.assert_array_equal(res[1]["costs"], info["costs"])
    assert res[0]["status"] in (0, 1, 2) and res[2]["status"] in (0, 1, 2)
