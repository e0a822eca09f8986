"""CPU oracle for the mini-BA hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product. Only `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of
`bench.py` may import it. The product path (`src/gsrecon`,
`paper_2506_05558_b200`) runs on the sm_100a kernels and fails loudly without
them.

It restates, in plain numpy/scipy float64, the Levenberg-Marquardt mini bundle
adjustment of the reference package (`pkg/src/gsrecon/miniba.py`; citations
are `miniba.py:<line>` relative to `/root/reference/pkg/src/gsrecon/`):

* projection residuals            -> `residuals`       (miniba.py:85-98)
* Huber cost / weights            -> `robust_cost`, `robust_weights` (miniba.py:46-54)
* Jacobian blocks A, F, B         -> `jacobians`       (miniba.py:101-132)
* normal equations U,g_c,V,g_p,Wf -> `normal_equations` (miniba.py:135-177)
* damped Schur / dense solve      -> `damped_step`     (miniba.py:180-220)
* LM loop with 5-try backtracking -> `lm`              (miniba.py:223-296)
* batched pose-only LM            -> `pose_lm`         (miniba.py:303-389)
* triangulation of one track      -> `triangulate`     (miniba.py:458-530)
* descriptor matching of a pair   -> `match`           (frontend.py:220-250)

Extensions that the reference does NOT have (documented in DESIGN.md):

* `loss="cauchy"`: rho = c^2/2 ln(1 + (e/c)^2), w = 1/(1 + (e/c)^2), c = delta.
  Needed by BASELINE config 5; parity for it is UNPINNED (no reference code).
* `evals` trace: number of trial cost evaluations per iteration (0 after a
  Cholesky failure, b+1 when the step is accepted at fraction 2^-b, 5 when all
  tries are rejected). The reference trace is recovered in
  `tests/golden/make_golden.py` by counting `huber_cost` calls.
* `fail_at`: fault injection -- iterations whose solve is forced to raise
  LinAlgError, to exercise miniba.py:247-251 which never fires naturally.

Pinning: `tests/golden/make_golden.py` runs the reference itself (importable
in the build container only) on the fixture problems and stores inputs and
outputs under `tests/golden/`; `tests/test_oracle_golden.py` checks this
restatement against those fixtures (traces identical through the plateau
index i*, final values to 1e-9).
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import cho_factor, cho_solve

# constants of miniba.py:23-25
LAMBDA_MAX = 1e10
DIAG_FLOOR = 1e-12
BACKTRACK_TRIES = 5
Z_MIN = 1e-12          # behind-camera threshold, miniba.py:91,96
BAD_RESIDUAL = 1e6     # miniba.py:97


# ----------------------------------------------------------------------------
# geometry helpers (scene.py:126-143)

def hat(v):
    """3-vector -> skew-symmetric matrix (scene.py:138-143)."""
    x, y, z = float(v[0]), float(v[1]), float(v[2])
    return np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])


def rodrigues(w):
    """Axis-angle -> rotation; 2nd-order series below 1e-12 rad (scene.py:126-135)."""
    w = np.asarray(w, dtype=np.float64)
    theta = float(np.linalg.norm(w))
    if theta < 1e-12:
        Wm = hat(w)
        return np.eye(3) + Wm + 0.5 * Wm @ Wm
    Km = hat(w / theta)
    return np.eye(3) + np.sin(theta) * Km + (1.0 - np.cos(theta)) * Km @ Km


# ----------------------------------------------------------------------------
# robust loss (miniba.py:46-54, plus the Cauchy extension)

def robust_cost(e, delta, loss="huber"):
    a = np.abs(e)
    if loss == "huber":
        rho = np.where(a <= delta, 0.5 * a * a, delta * (a - 0.5 * delta))
    elif loss == "cauchy":
        rho = 0.5 * delta * delta * np.log1p((a / delta) ** 2)
    else:
        raise ValueError(f"unknown loss {loss!r}")
    return float(np.sum(rho))


def robust_weights(e, delta, loss="huber"):
    a = np.abs(e)
    if loss == "huber":
        return np.where(a <= delta, 1.0, delta / np.maximum(a, 1e-300))
    if loss == "cauchy":
        return 1.0 / (1.0 + (a / delta) ** 2)
    raise ValueError(f"unknown loss {loss!r}")


# ----------------------------------------------------------------------------
# problem state: a plain dict {R,t,focal,cx,cy,points,cam_idx,pt_idx,uv,
# fixed_cams,optimize_focal,optimize_points}

def residuals(p):
    """(K,2) residuals, (K,3) camera-frame points, (K,) behind-camera mask
    (miniba.py:85-98)."""
    Xw = p["points"][p["pt_idx"]]
    Rk = p["R"][p["cam_idx"]]
    pc = np.einsum("kij,kj->ki", Rk, Xw) + p["t"][p["cam_idx"]]
    depth = pc[:, 2]
    behind = depth <= Z_MIN
    zc = np.where(behind, Z_MIN, depth)
    r = np.empty_like(p["uv"])
    r[:, 0] = p["focal"] * pc[:, 0] / zc + p["cx"] - p["uv"][:, 0]
    r[:, 1] = p["focal"] * pc[:, 1] / zc + p["cy"] - p["uv"][:, 1]
    r[behind] = BAD_RESIDUAL
    return r, pc, behind


def jacobians(p, pc, behind):
    """Per-observation blocks A (K,2,6) [rot | trans], F (K,2), B (K,2,3)
    for the left perturbation R <- exp(w) R (miniba.py:101-132)."""
    f = p["focal"]
    zc = np.where(pc[:, 2] > Z_MIN, pc[:, 2], Z_MIN)
    iz = 1.0 / zc
    K = pc.shape[0]
    Jp = np.zeros((K, 2, 3))
    Jp[:, 0, 0] = f * iz
    Jp[:, 1, 1] = f * iz
    Jp[:, 0, 2] = -f * pc[:, 0] * iz * iz
    Jp[:, 1, 2] = -f * pc[:, 1] * iz * iz
    Jp[behind] = 0.0
    v = pc - p["t"][p["cam_idx"]]          # R X
    # d p / d w = -[v]x ; -Jp @ [v]x written out per column
    Vx = np.zeros((K, 3, 3))
    Vx[:, 0, 1], Vx[:, 0, 2] = -v[:, 2], v[:, 1]
    Vx[:, 1, 0], Vx[:, 1, 2] = v[:, 2], -v[:, 0]
    Vx[:, 2, 0], Vx[:, 2, 1] = -v[:, 1], v[:, 0]
    A = np.concatenate([-(Jp @ Vx), Jp], axis=2)
    Bm = Jp @ p["R"][p["cam_idx"]]
    F = np.stack([pc[:, 0] * iz, pc[:, 1] * iz], axis=1)
    F[behind] = 0.0
    return A, F, Bm


def n_cam_params(p):
    """C = 6 * #free cameras + [focal] (miniba.py:82-83)."""
    return 6 * int(np.count_nonzero(~p["fixed_cams"])) + int(bool(p["optimize_focal"]))


def normal_equations(p, w, r, A, F, Bm):
    """IRLS normal-equation blocks (miniba.py:135-177).

    U (C,C) arrowhead, g_c (C,), V (P,3,3), g_p (P,3), Wf (P,C,3). The fixed
    cameras feed V, g_p and the focal terms only.
    """
    free = np.flatnonzero(~p["fixed_cams"])
    C = n_cam_params(p)
    P = p["points"].shape[0]
    has_f = bool(p["optimize_focal"])
    pts = p["pt_idx"]
    U = np.zeros((C, C))
    g_c = np.zeros(C)
    V = np.zeros((P, 3, 3))
    g_p = np.zeros((P, 3))
    Wf = np.zeros((P, C, 3))
    wB = Bm * w[:, None, None]
    if p["optimize_points"]:
        np.add.at(V, pts, np.einsum("kia,kib->kab", Bm, wB))
        np.add.at(g_p, pts, np.einsum("kia,ki->ka", wB, r))
    for s, cam in enumerate(free):
        sel = p["cam_idx"] == cam
        As = A[sel]
        wAs = As * w[sel][:, None, None]
        blk = slice(6 * s, 6 * s + 6)
        U[blk, blk] += np.einsum("kia,kib->ab", As, wAs)
        g_c[blk] += np.einsum("kia,ki->a", wAs, r[sel])
        if has_f:
            col = np.einsum("kia,ki->a", wAs, F[sel])
            U[blk, C - 1] += col
            U[C - 1, blk] = U[blk, C - 1]
        if p["optimize_points"]:
            np.add.at(Wf[:, blk, :], pts[sel], np.einsum("kia,kib->kab", wAs, Bm[sel]))
    if has_f:
        U[C - 1, C - 1] += float(np.sum(w * np.einsum("ki,ki->k", F, F)))
        g_c[C - 1] += float(np.sum(w * np.einsum("ki,ki->k", F, r)))
        if p["optimize_points"]:
            np.add.at(Wf[:, C - 1, :], pts, np.einsum("ki,kib->kb", F * w[:, None], Bm))
    return U, g_c, V, g_p, Wf


def damped_step(U, g_c, V, g_p, Wf, lam, method="schur"):
    """Solve (H + lam diag(max(diag H, 1e-12))) delta = -g (miniba.py:180-220).

    Raises np.linalg.LinAlgError on a non-PD reduced system, like the
    reference's cho_factor.
    """
    C = g_c.shape[0]
    P = g_p.shape[0]
    Ud = U.copy()
    Ud[np.diag_indices(C)] += lam * np.maximum(np.diag(U), DIAG_FLOOR)
    Vd = V.copy()
    d3 = np.arange(3)
    Vd[:, d3, d3] += lam * np.maximum(V[:, d3, d3], DIAG_FLOOR)
    if method == "dense":
        n = C + 3 * P
        H = np.zeros((n, n))
        H[:C, :C] = Ud
        for j in range(P):
            o = C + 3 * j
            H[o:o + 3, o:o + 3] = Vd[j]
            H[:C, o:o + 3] = Wf[j]
            H[o:o + 3, :C] = Wf[j].T
        sol = np.linalg.solve(H, -np.concatenate([g_c, g_p.ravel()]))
        return sol[:C], sol[C:].reshape(P, 3)
    if method != "schur":
        raise ValueError(f"unknown method {method!r}")
    if P == 0:
        dc = cho_solve(cho_factor(Ud), -g_c)
        return dc, np.zeros((0, 3))
    Vinv = np.linalg.inv(Vd)
    S = Ud - np.einsum("pad,pde,pbe->ab", Wf, Vinv, Wf)
    b = -g_c + np.einsum("pad,pde,pe->a", Wf, Vinv, g_p)
    dc = cho_solve(cho_factor(S), b)
    dp = np.einsum("pde,pe->pd", Vinv, -g_p - np.einsum("pad,a->pd", Wf, dc))
    return dc, dp


def _apply(p, base, dc, dp, frac):
    """Trial parameters old + frac*step (miniba.py:262-270)."""
    R0, t0, f0, X0 = base
    free = np.flatnonzero(~p["fixed_cams"])
    R = R0.copy()
    t = t0.copy()
    for s, cam in enumerate(free):
        R[cam] = rodrigues(frac * dc[6 * s:6 * s + 3]) @ R0[cam]
        t[cam] = t0[cam] + frac * dc[6 * s + 3:6 * s + 6]
    f = f0 + frac * dc[-1] if p["optimize_focal"] else f0
    X = X0 + frac * dp if p["optimize_points"] else X0
    return R, t, f, X


def lm(p, lambda_init=1e-5, nu=2.0, delta=2.0, max_iters=200, loss="huber",
       method="schur", fail_at=()):
    """LM with multiplicative damping, 5-try backtracking and rollback
    (miniba.py:223-296). Mutates `p` (R, t, focal, points).

    Returns dict(costs, accepted, lambdas, evals, final_rms, mean_err, cost).
    `fail_at`: iterations whose solve is forced to fail (fault injection).
    """
    if p["uv"].shape[0] == 0:
        raise ValueError("problem has no residuals")
    lam = float(lambda_init)
    r, pc, behind = residuals(p)
    e = np.linalg.norm(r, axis=1)
    cost = robust_cost(e, delta, loss)
    costs, accepted, lambdas, evals = [cost], [], [], []
    fail_at = set(fail_at)
    for it in range(max_iters):
        w = robust_weights(e, delta, loss)
        A, F, Bm = jacobians(p, pc, behind)
        blocks = normal_equations(p, w, r, A, F, Bm)
        lambdas.append(lam)
        try:
            if it in fail_at:
                raise np.linalg.LinAlgError("injected")
            dc, dp = damped_step(*blocks, lam, method)
        except np.linalg.LinAlgError:
            lam = min(lam * nu, LAMBDA_MAX)
            accepted.append(False)
            evals.append(0)
            costs.append(cost)
            continue
        base = (p["R"].copy(), p["t"].copy(), p["focal"], p["points"].copy())
        took = None
        tries = 0
        for b in range(BACKTRACK_TRIES):
            frac = 0.5 ** b
            p["R"], p["t"], p["focal"], p["points"] = _apply(p, base, dc, dp, frac)
            r_try, pc_try, behind_try = residuals(p)
            e_try = np.linalg.norm(r_try, axis=1)
            c_try = robust_cost(e_try, delta, loss)
            tries += 1
            if c_try < cost and np.isfinite(c_try):
                took = frac
                break
        evals.append(tries)
        if took is None:
            p["R"], p["t"], p["focal"], p["points"] = base
            lam = min(lam * nu, LAMBDA_MAX)
            accepted.append(False)
            costs.append(cost)
            if lam >= LAMBDA_MAX:
                break
            continue
        lam = max(lam / nu, 1e-15) if took == 1.0 else min(lam * nu, LAMBDA_MAX)
        gain = cost - c_try
        cost, r, e, pc, behind = c_try, r_try, e_try, pc_try, behind_try
        accepted.append(True)
        costs.append(cost)
        if gain <= 1e-15 * max(cost, 1.0):
            break
    return dict(costs=np.array(costs), accepted=np.array(accepted, dtype=bool),
                lambdas=np.array(lambdas), evals=np.array(evals, dtype=np.int32),
                final_rms=float(np.sqrt(np.mean(e ** 2))), mean_err=float(np.mean(e)),
                cost=cost)


# ----------------------------------------------------------------------------
# batched pose-only LM (miniba.py:303-389)

def _rodrigues_batch(w):
    th = np.maximum(np.linalg.norm(w, axis=-1, keepdims=True), 1e-30)
    k = w / th
    Km = np.zeros(w.shape[:-1] + (3, 3))
    Km[..., 0, 1], Km[..., 0, 2] = -k[..., 2], k[..., 1]
    Km[..., 1, 0], Km[..., 1, 2] = k[..., 2], -k[..., 0]
    Km[..., 2, 0], Km[..., 2, 1] = -k[..., 1], k[..., 0]
    th = th[..., None]
    return np.eye(3) + np.sin(th) * Km + (1.0 - np.cos(th)) * (Km @ Km)


def _pose_eval(R, t, X, uv, f, cx, cy, delta):
    pc = X @ np.swapaxes(R, -1, -2) + t[..., None, :]
    ok = pc[..., 2] > Z_MIN
    zc = np.where(ok, pc[..., 2], Z_MIN)
    ru = np.where(ok, f * pc[..., 0] / zc + cx - uv[..., 0], BAD_RESIDUAL)
    rv = np.where(ok, f * pc[..., 1] / zc + cy - uv[..., 1], BAD_RESIDUAL)
    e = np.hypot(ru, rv)
    rho = np.where(e <= delta, 0.5 * e * e, delta * (e - 0.5 * delta))
    return rho.sum(axis=-1), (pc, zc, ru, rv, e, ok)


def pose_lm(R0, t0, X, uv, f, cx, cy, iters, lambda_init=1e-5, nu=2.0, delta=2.0):
    """Batched pose-only LM: single trial per iteration, no backtracking
    (miniba.py:334-389). Returns (R, t, cost)."""
    R = np.array(R0, dtype=np.float64, copy=True)
    t = np.array(t0, dtype=np.float64, copy=True)
    nb = R.shape[0]
    lam = np.full(nb, float(lambda_init))
    cost, aux = _pose_eval(R, t, X, uv, f, cx, cy, delta)
    for _ in range(iters):
        pc, zc, ru, rv, e, ok = aux
        w = robust_weights(e, delta) * ok
        iz = 1.0 / zc
        Jp = np.zeros(pc.shape[:-1] + (2, 3))
        Jp[..., 0, 0] = f * iz
        Jp[..., 1, 1] = f * iz
        Jp[..., 0, 2] = -f * pc[..., 0] * iz * iz
        Jp[..., 1, 2] = -f * pc[..., 1] * iz * iz
        v = pc - t[..., None, :]
        Vx = np.zeros(pc.shape[:-1] + (3, 3))
        Vx[..., 0, 1], Vx[..., 0, 2] = -v[..., 2], v[..., 1]
        Vx[..., 1, 0], Vx[..., 1, 2] = v[..., 2], -v[..., 0]
        Vx[..., 2, 0], Vx[..., 2, 1] = -v[..., 1], v[..., 0]
        J = np.concatenate([-(Jp @ Vx), Jp], axis=-1)
        res = np.stack([ru, rv], axis=-1)
        wJ = J * w[..., None, None]
        H = np.einsum("bmia,bmic->bac", J, wJ)
        g = np.einsum("bmia,bmi->ba", wJ, res)
        d6 = np.arange(6)
        H[:, d6, d6] += lam[:, None] * np.maximum(H[:, d6, d6], DIAG_FLOOR)
        try:
            step = np.linalg.solve(H, -g[..., None])[..., 0]
        except np.linalg.LinAlgError:
            H[:, d6, d6] += 1e-6
            step = np.linalg.solve(H, -g[..., None])[..., 0]
        R_try = _rodrigues_batch(step[:, :3]) @ R
        t_try = t + step[:, 3:]
        c_try, _ = _pose_eval(R_try, t_try, X, uv, f, cx, cy, delta)
        better = c_try < cost
        R = np.where(better[:, None, None], R_try, R)
        t = np.where(better[:, None], t_try, t)
        lam = np.where(better, np.maximum(lam / nu, 1e-15), np.minimum(lam * nu, LAMBDA_MAX))
        cost, aux = _pose_eval(R, t, X, uv, f, cx, cy, delta)
    return R, t, cost


# ----------------------------------------------------------------------------
# triangulation (miniba.py:458-530), status codes instead of exceptions

TRI_OK, TRI_FEW, TRI_BASELINE, TRI_PARALLEL, TRI_BEHIND, TRI_REPROJ = range(6)


def triangulate(Rs, ts, px, f, cx, cy, max_reproj_px=8.0, min_angle_deg=0.5, gn_steps=3):
    """One track: rays of every view (camera centre -R^T t, direction R^T K^-1 uv,
    normalised), the pair with the widest angle (first in (i, j) order on ties),
    the midpoint of its closest points, then `gn_steps` Gauss-Newton steps on
    the reprojection error with H = J^T J + 1e-12 I. Returns (X, status)."""
    n = len(Rs)
    if n < 2:
        return np.full(3, np.nan), TRI_FEW
    px = np.asarray(px, np.float64)
    origins = np.stack([-R.T @ t for R, t in zip(Rs, ts)])
    dirs = np.empty((n, 3))
    for i in range(n):
        d = Rs[i].T @ np.array([(px[i, 0] - cx) / f, (px[i, 1] - cy) / f, 1.0])
        dirs[i] = d / np.linalg.norm(d)
    best = (-1.0, 0, 1)
    for i in range(n):
        for j in range(i + 1, n):
            ang = np.degrees(np.arccos(np.clip(np.abs(dirs[i] @ dirs[j]), -1, 1)))
            if ang > best[0]:
                best = (ang, i, j)
    ang, i, j = best
    if ang <= min_angle_deg:
        return np.full(3, np.nan), TRI_BASELINE
    d1, d2, o1, o2 = dirs[i], dirs[j], origins[i], origins[j]
    a, b, c = d1 @ d1, d1 @ d2, d2 @ d2
    rhs = o2 - o1
    den = a * c - b * b
    if den < 1e-18:
        return np.full(3, np.nan), TRI_PARALLEL
    s_ = (c * (d1 @ rhs) - b * (d2 @ rhs)) / den
    u_ = (b * (d1 @ rhs) - a * (d2 @ rhs)) / den
    X = 0.5 * (o1 + s_ * d1 + o2 + u_ * d2)
    for _ in range(gn_steps):
        J = np.zeros((2 * n, 3))
        r = np.zeros(2 * n)
        for k in range(n):
            pc = Rs[k] @ X + ts[k]
            if pc[2] <= 1e-12:
                return np.full(3, np.nan), TRI_BEHIND
            z = pc[2]
            Jp = np.array([[f / z, 0, -f * pc[0] / z ** 2], [0, f / z, -f * pc[1] / z ** 2]])
            J[2 * k:2 * k + 2] = Jp @ Rs[k]
            r[2 * k] = f * pc[0] / z + cx - px[k, 0]
            r[2 * k + 1] = f * pc[1] / z + cy - px[k, 1]
        X = X - np.linalg.solve(J.T @ J + 1e-12 * np.eye(3), J.T @ r)
    errs = np.empty(n)
    for k in range(n):
        pc = Rs[k] @ X + ts[k]
        if pc[2] <= 1e-12:
            return np.full(3, np.nan), TRI_BEHIND
        errs[k] = np.hypot(f * pc[0] / pc[2] + cx - px[k, 0], f * pc[1] / pc[2] + cy - px[k, 1])
    if errs.mean() > max_reproj_px:
        return np.full(3, np.nan), TRI_REPROJ
    return X, TRI_OK


# ----------------------------------------------------------------------------
# descriptor matching (frontend.py:210-250)

_POPC8 = np.array([bin(i).count("1") for i in range(256)], dtype=np.uint8)


def match(desc_a, desc_b, ratio_max=0.95, bits=256):
    """Mutual nearest neighbours in Hamming distance over packed descriptors,
    best / second-best ratio test (second via np.partition, duplicates
    counted). Returns (idx_a, idx_b, scores) sorted by idx_a."""
    if len(desc_a) == 0 or len(desc_b) == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)
    d = _POPC8[desc_a[:, None, :] ^ desc_b[None, :, :]].sum(axis=-1, dtype=np.int32)

    def nn_ratio(dist):
        nn = np.argmin(dist, axis=1)
        best = dist[np.arange(len(dist)), nn]
        if dist.shape[1] >= 2:
            second = np.partition(dist, 1, axis=1)[:, 1].astype(np.float64)
            ratio = np.where(second > 0, best / np.maximum(second, 1e-12), 1.0)
            return nn, ratio < ratio_max
        return nn, np.ones(len(dist), dtype=bool)

    nn_ab, ok_a = nn_ratio(d)
    nn_ba, ok_b = nn_ratio(d.T)
    ia = np.arange(len(desc_a))
    mutual = (nn_ba[nn_ab] == ia) & ok_a & ok_b[nn_ab]
    idx_a, idx_b = ia[mutual], nn_ab[mutual]
    return idx_a.astype(np.int64), idx_b.astype(np.int64), 1.0 - d[idx_a, idx_b] / float(bits)


# ----------------------------------------------------------------------------
# parity rule

def plateau_index(costs, tau=1e-9, kappa=0.0):
    """i*: first iteration i with |costs[i+1] - costs[-1]| <= tau*costs[-1] + kappa.
    Traces must agree exactly for iterations 0..i*."""
    costs = np.asarray(costs)
    final = costs[-1]
    n_it = len(costs) - 1
    for i in range(n_it):
        if abs(costs[i + 1] - final) <= tau * abs(final) + kappa:
            return i
    return n_it - 1
