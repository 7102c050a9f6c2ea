"""Pins of the CPU oracle (oracle/) to things other than itself (no GPU needed).

Each test names the passage / closed form it pins.  A plausible mistake in the
oracle (a dropped residual term, a flipped sign, a transposed operand, a wrong
elimination formula) fails at least one of: the assembled Newton LU solve, the
paper's doubly augmented solve, brute-force active sets, planted optima or the
KKT certificate.
"""
import json
import math
import os

import numpy as np
import pytest

from gen.planted import config, planted_qp, random_small_qp
from oracle import kkt as okkt
from oracle.active_set import solve_active_set
from oracle.ipm import (FAMILIES, Iterate, Options, Problem, condensed_solve, full_multipliers,
                        initial_point, kkt_norm, max_step, newton_direction, recover_step,
                        reduced_system, residuals, solve, warm_start_point)
from oracle.newton import doubly_augmented_solve, full_newton_step

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_hand_examples.json")))


def _prob_1d(ex):
    return Problem(H=np.array(ex["H"]), g=np.array(ex["g"]), A=np.zeros((0, 1)), l=np.zeros(0),
                   u=np.zeros(0), xl=np.array(ex["xl"]), xu=np.array(ex["xu"]))


def _random_interior_iterate(p: Problem, seed: int) -> Iterate:
    rng = np.random.default_rng(seed)
    x = rng.normal(size=p.n)
    s = {f: rng.uniform(0.1, 3.0, size=p.C[f].shape[0]) for f in FAMILIES}
    lam = {f: rng.uniform(0.1, 3.0, size=p.C[f].shape[0]) for f in FAMILIES}
    return Iterate(x, s, lam, mu=float(rng.uniform(1e-3, 1.0)))


# ---------------------------------------------------------------- hand examples (golden)
def test_hand_1d_interior():
    ex = GOLD["ipm_1d_interior"]
    res = solve(_prob_1d(ex))
    assert res.status == "converged"
    assert abs(res.x[0] - ex["x"][0]) < 1e-6
    assert abs(res.obj - ex["obj"]) < 1e-8


def test_hand_1d_active():
    ex = GOLD["ipm_1d_active"]
    p = _prob_1d(ex)
    res = solve(p)
    assert res.status == "converged"
    assert abs(res.x[0] - ex["x"][0]) < 1e-6
    lam = full_multipliers(p, res.it)
    assert abs(lam["lx"][0] - ex["lam_lx"][0]) < 1e-6


def test_hand_initial_point():
    ex = GOLD["initial_point"]
    p = Problem(H=np.eye(1), g=np.zeros(1), A=np.zeros((0, 1)), l=np.zeros(0), u=np.zeros(0),
                xl=np.array(ex["xl"]), xu=np.array(ex["xu"]))
    it = initial_point(p, Options())
    assert it.x[0] == ex["x0"][0]
    assert it.s["lx"][0] == ex["s_lx"][0] and it.s["ux"][0] == ex["s_ux"][0]
    assert it.mu == pytest.approx(ex["mu0"], rel=0, abs=1e-15)


def test_hand_complementarity():
    ex = GOLD["complementarity"]
    p = Problem(H=np.eye(1), g=np.zeros(1), A=np.zeros((0, 1)), l=np.zeros(0), u=np.zeros(0),
                xl=np.array([0.0]), xu=np.array([np.inf]))
    it = Iterate(np.array([3.0]), {"lA": np.zeros(0), "uA": np.zeros(0), "lx": np.array([ex["s"]]), "ux": np.zeros(0)},
                 {"lA": np.zeros(0), "uA": np.zeros(0), "lx": np.array([ex["lam"]]), "ux": np.zeros(0)}, ex["mu"])
    r = residuals(p, it)
    assert r["clx"][0] == ex["r_c"]


def test_hand_step_length():
    ex = GOLD["step_length"]
    v = {f: np.zeros(0) for f in FAMILIES}
    dv = {f: np.zeros(0) for f in FAMILIES}
    v["lx"] = np.array(ex["s"])
    dv["lx"] = np.array(ex["ds"])
    assert max_step(v, dv, ex["tau"]) == pytest.approx(ex["alpha"], abs=1e-16)
    dv["lx"] = np.array([2.0])
    assert max_step(v, dv, ex["tau"]) == 1.0          # empty ratio set -> 1


def test_hand_condensed_operator():
    ex = GOLD["condensed_scalar"]
    Kv = okkt.condensed_apply(np.array(ex["H"]), np.array(ex["A"]), np.array(ex["sig_b"]),
                              np.array(ex["sig_c"]), np.array(ex["v"]))
    assert Kv.tolist() == ex["Kv"]
    ex = GOLD["colsq_scalar"]
    d = okkt.jacobi_diag(np.array(ex["H"]), np.array(ex["A"]), np.array(ex["sig_b"]), np.array(ex["sig_c"]))
    assert d.tolist() == ex["diag"]


# ---------------------------------------------------------------- elimination pins
@pytest.mark.parametrize("seed", range(10))
def test_condensed_step_matches_full_newton_lu(seed):
    """Block-row elimination (eq:2x2_reduced) + condensation + recovery must give
    the step of the assembled Newton system eq:newton_system solved by LU."""
    q = random_small_qp(6, 5, seed)
    p = Problem.from_data(q)
    it = _random_interior_iterate(p, seed)
    r = residuals(p, it)
    dx, ds, dl = newton_direction(p, it, r)
    dx_f, ds_f, dl_f, (Kf, rhs, sol) = full_newton_step(p, it, r)
    scale = max(1.0, np.max(np.abs(sol)))
    assert np.max(np.abs(dx - dx_f)) <= 1e-10 * scale
    for f in FAMILIES:
        if ds[f].size:
            assert np.max(np.abs(ds[f] - ds_f[f])) <= 1e-10 * scale
            assert np.max(np.abs(dl[f] - dl_f[f])) <= 1e-10 * scale
    # back-substitution of the recovered step into the assembled system
    full = np.concatenate([dx] + [dl[f] for f in FAMILIES] + [ds[f] for f in FAMILIES])
    assert np.linalg.norm(Kf @ full - rhs) <= 1e-8 * np.linalg.norm(rhs)


@pytest.mark.parametrize("seed", range(10))
def test_condensed_matches_doubly_augmented(seed):
    """The paper's own SPD system eq:2x2_augmented and the condensed
    Schur system (D1) have the same solution (<= 1e-10)."""
    q = random_small_qp(7, 6, 100 + seed)
    p = Problem.from_data(q)
    it = _random_interior_iterate(p, seed)
    r = residuals(p, it)
    Q, B, D, r1, r2 = reduced_system(p, it, r)
    dx, dlamA, _ = condensed_solve(Q, B, D, r1, r2)
    dx2, dlamA2, M = doubly_augmented_solve(Q, B, D, r1, r2)
    sc = max(1.0, np.max(np.abs(dx)))
    assert np.max(np.abs(dx - dx2)) <= 1e-10 * sc
    if dlamA.size:
        assert np.max(np.abs(dlamA - dlamA2)) <= 1e-10 * max(1.0, np.max(np.abs(dlamA)))
    # SPD certificate of the doubly augmented matrix
    assert np.max(np.abs(M - M.T)) <= 1e-11 * np.max(np.abs(M))
    np.linalg.cholesky(0.5 * (M + M.T))


def test_condensed_matrix_is_schur_complement():
    """oracle.kkt's K = H + diag(sig_b) + A^T diag(sig_c) A (masked, full-length) equals
    Q + B^T D^-1 B assembled from the compact family blocks of eq:2x2_reduced."""
    q = random_small_qp(8, 6, 7)
    p = Problem.from_data(q)
    it = _random_interior_iterate(p, 3)
    r = residuals(p, it)
    Q, B, D, _, _ = reduced_system(p, it, r)
    B = B.toarray()
    K1 = Q + B.T @ (B / D[:, None])
    sig_b = np.zeros(p.n)
    sig_b[p.J_l] += it.lam["lx"] / it.s["lx"]
    sig_b[p.J_u] += it.lam["ux"] / it.s["ux"]
    sig_c = np.zeros(p.m)
    sig_c[p.I_l] += it.lam["lA"] / it.s["lA"]
    sig_c[p.I_u] += it.lam["uA"] / it.s["uA"]
    K2 = okkt.condensed_matrix(p.H, p.A_dense(), sig_b, sig_c)
    assert np.max(np.abs(K1 - K2)) <= 1e-13 * np.max(np.abs(K1))
    # diag identity e_j^T K e_j and the colsq formula
    dj = okkt.jacobi_diag(p.H, p.A_dense(), sig_b, sig_c)
    assert np.max(np.abs(dj - np.diag(K1))) <= 1e-13 * np.max(np.abs(dj))
    v = np.random.default_rng(0).normal(size=p.n)
    assert np.max(np.abs(okkt.condensed_apply(p.H, p.A_dense(), sig_b, sig_c, v) - K1 @ v)) <= 1e-12 * np.max(np.abs(K1 @ v))


# ---------------------------------------------------------------- whole-IPM pins
def _active_set_case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 5))
    m = int(rng.integers(0, 4))
    return random_small_qp(n, m, seed, density=0.8)


@pytest.mark.parametrize("block", range(4))
def test_ipm_matches_active_set_bruteforce(block):
    """100 seeded tiny QPs: the oracle IPM matches brute-force active-set
    enumeration (|dx|_inf <= 1e-5, relative objective <= 1e-8)."""
    for seed in range(25 * block, 25 * block + 25):
        q = _active_set_case(seed)
        p = Problem.from_data(q)
        best = solve_active_set(p.H, p.g, p.A_dense(), p.l, p.u, p.xl, p.xu)
        assert best is not None, seed
        res = solve(p)
        assert res.status == "converged", seed
        assert np.max(np.abs(res.x - best[0])) <= 1e-5, seed
        assert abs(res.obj - best[1]) <= 1e-8 * max(1.0, abs(best[1])), seed


@pytest.mark.parametrize("seed", range(10))
def test_ipm_matches_planted_optimum_C1(seed):
    """Planted KKT point (closed form at any size, D5): x within 1e-6 relative,
    objective within 1e-8 relative (north_star tolerances)."""
    q = config("C1", seed)
    p = Problem.from_data(q)
    res = solve(p)
    assert res.status == "converged"
    assert np.max(np.abs(res.x - q.x_star)) <= 1e-6 * max(1.0, np.max(np.abs(q.x_star)))
    assert abs(res.obj - q.f_star) <= 1e-8 * abs(q.f_star)
    lam = full_multipliers(p, res.it)
    for f, ref in (("lA", q.lam_lA), ("uA", q.lam_uA), ("lx", q.lam_lx), ("ux", q.lam_ux)):
        assert np.max(np.abs(lam[f] - ref), initial=0.0) <= 1e-6


def test_ipm_planted_medium():
    q = planted_qp(400, 120, density=0.05, rank=32, seed=3, rows="vmat", var="box")
    p = Problem.from_data(q)
    res = solve(p)
    assert res.status == "converged"
    assert np.max(np.abs(res.x - q.x_star)) <= 1e-6 * np.max(np.abs(q.x_star))
    assert abs(res.obj - q.f_star) <= 1e-8 * abs(q.f_star)


def test_ipm_no_bounds_closed_form():
    """R13: no finite bound -> one exact Newton step gives x = -H^-1 g."""
    q = planted_qp(30, 0, rank=30, seed=5, var="none")
    p = Problem.from_data(q)
    res = solve(p)
    assert res.iters == 1 and res.status == "converged"
    x_cf = np.linalg.solve(p.H, -p.g)
    assert np.max(np.abs(res.x - x_cf)) <= 1e-12 * max(1.0, np.max(np.abs(x_cf)))


def test_ipm_invariants_and_certificate():
    """Alg. 1 semantics: interior preserved, mu decreases exactly by 10x at
    each update, return implies ||r||_inf < mu <= mu_tol; KKT certificate holds."""
    q = config("C1", 11)
    p = Problem.from_data(q)
    opt = Options()
    it0 = initial_point(p, opt)
    res = solve(p, opt)
    mus = [it0.mu] + [t["mu"] for t in res.trace]
    for a, b in zip(mus, mus[1:]):
        assert b == a or b == a / 10.0
    for t in res.trace:
        assert 0 < t["ax"] <= 1 and 0 < t["al"] <= 1
    for f in FAMILIES:
        assert np.all(res.it.s[f] > 0) and np.all(res.it.lam[f] > 0)
    assert res.it.mu <= opt.mu_tol and res.trace[-1]["kkt"] < res.it.mu
    lam = full_multipliers(p, res.it)
    cert = okkt.kkt_certificate(p.H, p.g, p.A_dense(), p.l, p.u, p.xl, p.xu, res.x, lam["lA"], lam["uA"], lam["lx"], lam["ux"])
    assert cert["stationarity"] < 1e-7 and cert["infeasibility"] < 1e-7
    assert cert["min_multiplier"] == 0.0 and cert["complementarity"] < 1e-7


@pytest.mark.parametrize("seed", range(5))
def test_mehrotra_matches_planted(seed):
    q = config("C1", seed)
    p = Problem.from_data(q)
    res = solve(p, Options(predictor_corrector=True))
    assert res.status == "converged"
    assert np.max(np.abs(res.x - q.x_star)) <= 1e-6 * max(1.0, np.max(np.abs(q.x_star)))
    assert abs(res.obj - q.f_star) <= 1e-8 * abs(q.f_star)


def test_mehrotra_matches_active_set():
    for seed in range(20):
        q = _active_set_case(500 + seed)
        p = Problem.from_data(q)
        best = solve_active_set(p.H, p.g, p.A_dense(), p.l, p.u, p.xl, p.xu)
        res = solve(p, Options(predictor_corrector=True))
        assert res.status == "converged", seed
        assert np.max(np.abs(res.x - best[0])) <= 1e-5, seed


def test_warm_start_reaches_planted_optimum():
    """R15: a warm start from a nearby problem's solution converges to the planted
    optimum of the new problem."""
    q0 = config("C1", 20)
    q1 = config("C1", 20)
    q1.g = q1.g + 0.01 * np.random.default_rng(1).normal(size=q1.n)   # perturbed linear term
    p0 = Problem.from_data(q0)
    r0 = solve(p0)
    p1 = Problem.from_data(q1)
    cold = solve(p1)
    warm = solve(p1, start=warm_start_point(p1, r0.x, r0.it.lam, Options()))
    assert warm.status == "converged" and cold.status == "converged"
    assert np.max(np.abs(warm.x - cold.x)) <= 1e-6
    best = np.max(np.abs(warm.x - cold.x))
    assert best <= 1e-6


# ---------------------------------------------------------------- R15 / R18 / a11 hand pins
def test_warm_start_point_hand_values():
    """R15 (SURVEY §8(c) point 15; the paper only names warm starting), values worked by
    hand for theta = 1e-3 on a 3-variable, 1-row problem:
      x_prev = (0, 5, 3.5), boxes [0,1], [0,0.002], (-inf,3]:
        margins min(theta, (xu-xl)/4) = 1e-3, 5e-4, theta (one-sided)  ->  x0 = (1e-3, 1.5e-3, 2.999)
      s = max(gap(x0), theta): s_lA = max(1e-3+1.5e-3-0.5, theta) = 1e-3; s_lx = (1e-3, 1.5e-3);
        s_ux = (0.999, max(5e-4, theta) = 1e-3, max(1e-3, theta) = 1e-3)
      lam = max(lam_prev, theta): lA 0.25; lx (2, 1e-3); ux (1e-3, 0.5, 1e-3)
      mu0 = 0.1 * sum(lam s) / 6 = 0.1 * 0.0037515 / 6 = 6.2525e-5."""
    p = Problem(H=np.eye(3), g=np.zeros(3), A=np.array([[1.0, 1.0, 0.0]]), l=np.array([0.5]),
                u=np.array([np.inf]), xl=np.array([0.0, 0.0, -np.inf]), xu=np.array([1.0, 0.002, 3.0]))
    lam = {"lA": np.array([0.25]), "uA": np.zeros(0), "lx": np.array([2.0, 0.0]), "ux": np.array([0.0, 0.5, 0.0])}
    w = warm_start_point(p, np.array([0.0, 5.0, 3.5]), lam, Options(warm_shift=1e-3))
    np.testing.assert_allclose(w.x, [1e-3, 1.5e-3, 2.999], rtol=0, atol=1e-15)
    np.testing.assert_allclose(w.s["lA"], [1e-3], rtol=0, atol=1e-15)
    np.testing.assert_allclose(w.s["lx"], [1e-3, 1.5e-3], rtol=0, atol=1e-15)
    np.testing.assert_allclose(w.s["ux"], [0.999, 1e-3, 1e-3], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(w.lam["lA"], [0.25])
    np.testing.assert_array_equal(w.lam["lx"], [2.0, 1e-3])
    np.testing.assert_array_equal(w.lam["ux"], [1e-3, 0.5, 1e-3])
    assert abs(w.mu - 6.2525e-5) <= 1e-18


def test_mehrotra_hand_values():
    """R18 worked by hand on min 1/2 x^2 - x/2, x >= 0 at x = s = lam = 1:
      affine (r_c = lam s = 1): r_H = x + g - lam = -0.5, Q = 1 + lam/s = 2, r1 = 0.5 - 1 = -0.5,
        dx = -0.25, ds = -0.25, dlam = -(1 - 0.25) = -0.75; alpha (tau = 1) = 1 for both;
        mu = 1, mu_aff = (1 - 0.75)(1 - 0.25) = 0.1875, sigma = 0.1875^3 = 27/4096
      corrector r_c = lam s + dlam_aff ds_aff - sigma mu = 1 + 0.1875 - 27/4096 = 1.180908203125
        r1 = 0.5 - 1.180908203125, dx = r1 / 2 = -0.3404541015625, dlam = -(r_c + dx) = -0.8404541015625.
    Squaring sigma instead of cubing it, or dropping the dlam_aff o ds_aff term, changes dx."""
    from oracle.ipm import _mehrotra
    e = np.zeros(0)
    p = Problem(H=np.array([[1.0]]), g=np.array([-0.5]), A=np.zeros((0, 1)), l=e, u=e, xl=np.array([0.0]),
                xu=np.array([np.inf]))
    it = Iterate(np.array([1.0]), {"lA": e, "uA": e, "lx": np.array([1.0]), "ux": e},
                 {"lA": e, "uA": e, "lx": np.array([1.0]), "ux": e}, 0.5)
    dx, ds, dl, smu = _mehrotra(p, it, Options(predictor_corrector=True))
    assert smu == 27.0 / 4096.0
    assert abs(dx[0] - (-0.3404541015625)) <= 1e-15
    assert abs(ds["lx"][0] - (-0.3404541015625)) <= 1e-15
    assert abs(dl["lx"][0] - (-0.8404541015625)) <= 1e-15


def test_rank2_update_spec_hand_case_and_secant():
    """a11 / oracle.bfgs: SPEC S:380 hand case (H = I, s = e1, y = 2 e1 -> diag(2, 1, 1)), the
    secant equation H+ s = y and preserved positive definiteness on a random SPD H."""
    from oracle.bfgs import bfgs_terms, rank2_update
    H = np.eye(3)
    s = np.array([1.0, 0.0, 0.0])
    Hp = rank2_update(H, *bfgs_terms(H, s, 2.0 * s))
    np.testing.assert_array_equal(Hp, np.diag([2.0, 1.0, 1.0]))
    rng = np.random.default_rng(11)
    M = rng.normal(size=(30, 30))
    H = M @ M.T + 30 * np.eye(30)
    s = rng.normal(size=30)
    y = H @ s + 0.3 * rng.normal(size=30)
    assert y @ s > 0
    Hp = rank2_update(H, *bfgs_terms(H, s, y))
    np.testing.assert_allclose(Hp @ s, y, rtol=0, atol=1e-11 * np.abs(y).max())
    assert np.linalg.eigvalsh(Hp).min() > 0
    # y = H s (already consistent): H+ acts identically to H on s
    Hq = rank2_update(H, *bfgs_terms(H, s, H @ s))
    np.testing.assert_allclose(Hq @ s, H @ s, rtol=1e-12)


# ---------------------------------------------------------------- oracle.pcg (textbook Jacobi PCG)
def _spd(n, seed, cond=50.0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    return (Q * np.geomspace(1.0, cond, n)) @ Q.T


def test_pcg_dense_spd_matches_cholesky():
    """dense SPD 30x30 against a Cholesky solve (scipy cho_solve)."""
    import scipy.linalg as sla
    from oracle.pcg import pcg
    K = _spd(30, 1)
    b = np.random.default_rng(2).normal(size=30)
    res = pcg(lambda v: K @ v, 1.0 / np.diag(K), b, rtol=1e-13)
    x_ref = sla.cho_solve(sla.cho_factor(K), b)
    assert not res.breakdown and res.iters <= 3 * 30   # finite precision: a few more than n
    np.testing.assert_allclose(res.x, x_ref, rtol=0, atol=1e-10 * np.abs(x_ref).max())


def test_pcg_identity_and_exact_jacobi_one_iteration():
    """K = I and K diagonal with the exact Jacobi preconditioner converge in 1 iteration."""
    from oracle.pcg import pcg
    b = np.random.default_rng(3).normal(size=17)
    res = pcg(lambda v: v, np.ones(17), b, rtol=1e-14)
    assert res.iters == 1 and np.array_equal(res.x, b)
    d = np.random.default_rng(4).uniform(0.5, 4.0, 17)
    res = pcg(lambda v: d * v, 1.0 / d, b, rtol=1e-14)
    assert res.iters == 1
    np.testing.assert_allclose(res.x, b / d, rtol=1e-15)


def test_pcg_conjugacy_and_finite_termination():
    """CG theory: successive directions are K-conjugate (p_i^T K p_j = 0, i != j), and in exact
    arithmetic CG terminates in <= n steps (here n = 8: residual at rounding level after 8)."""
    from oracle.pcg import pcg
    K = _spd(8, 5, cond=20.0)
    b = np.random.default_rng(6).normal(size=8)
    Minv = 1.0 / np.diag(K)
    res = pcg(lambda v: K @ v, Minv, b, maxit=8, keep_directions=True)
    P = np.array(res.directions)
    G = P @ K @ P.T
    off = G - np.diag(np.diag(G))
    assert np.abs(off).max() <= 1e-10 * np.abs(np.diag(G)).max()
    assert np.linalg.norm(res.r) <= 1e-10 * np.linalg.norm(b)
    # one hand-checkable iteration: x1 = alpha0 z0 with alpha0 = (r0,z0)/(K z0, z0)
    r1 = pcg(lambda v: K @ v, Minv, b, maxit=1)
    z0 = Minv * b
    assert abs(r1.alpha - (b @ z0) / (z0 @ K @ z0)) <= 1e-15 * abs(r1.alpha)
    np.testing.assert_allclose(r1.x, r1.alpha * z0, rtol=1e-15)


def test_pcg_on_condensed_operator_matches_condensed_cholesky():
    """The oracle PCG on K = H + Sigma_b + A^T Sigma_c A (oracle.kkt.condensed_apply) reaches the
    Cholesky solution of oracle.kkt.condensed_matrix."""
    from oracle.pcg import pcg
    q = config("C1", 3)
    rng = np.random.default_rng(7)
    A = q.A_scipy().toarray()
    sb = rng.uniform(0.0, 3.0, q.n)
    sc = 10.0 ** rng.uniform(-2, 2, q.m)
    b = rng.normal(size=q.n)
    K = okkt.condensed_matrix(q.H, A, sb, sc)
    res = pcg(lambda v: okkt.condensed_apply(q.H, A, sb, sc, v), 1.0 / okkt.jacobi_diag(q.H, A, sb, sc), b,
              rtol=1e-13)
    np.testing.assert_allclose(res.x, np.linalg.solve(K, b), rtol=0, atol=1e-9 * np.abs(res.x).max())
