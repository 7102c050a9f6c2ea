"""Pins of the SQP oracle (oracle/sqp.py) against things other than itself:
closed forms, the textbook dense BFGS recursion, finite differences, a known analytic
minimum (Rosenbrock), and scipy's SLSQP on the same small dose NLP."""
import numpy as np
import pytest
import scipy.optimize as so
import scipy.sparse as sp

from gen.dose_nlp import dose_nlp, nlp_config
from oracle.sqp import Bfgs, SqpOptions, bfgs_update, dose_gradient, dose_h0, dose_objective, sqp_dose, sqp_solve


def test_dose_gradient_matches_central_differences():
    q = nlp_config("S1", 3)
    x = q.x0 + 0.1 * np.random.default_rng(0).normal(size=q.n)
    g = dose_gradient(q, x)
    h = 1e-6
    fd = np.array([(dose_objective(q, x + h * e) - dose_objective(q, x - h * e)) / (2 * h) for e in np.eye(q.n)])
    assert np.max(np.abs(g - fd)) <= 1e-6 * max(1.0, np.max(np.abs(g)))


def test_h0_is_gauss_newton_diagonal():
    q = nlp_config("S1", 1)
    Dd = q.D_scipy().toarray()
    assert np.allclose(dose_h0(q), np.einsum("ij,i,ij->j", Dd, q.w, Dd) + 1e-3, rtol=1e-14, atol=0)


def test_bfgs_1d_secant_hand_case():
    """H = I, s = e1, y = 2 e1 -> H+ = diag(2, 1, ...)."""
    B = Bfgs.diagonal(np.ones(4))
    ok, theta, *_ = bfgs_update(B, np.eye(4)[0], 2 * np.eye(4)[0])
    assert ok and theta == 1.0
    assert np.allclose(B.dense(), np.diag([2.0, 1, 1, 1]), atol=1e-15)


def test_compact_bfgs_equals_dense_recursion_and_secant():
    """10 updates from a random SPD sequence: the compact form equals the textbook dense
    recursion B+ = B - B s s^T B / s^T B s + y y^T / y^T s (to 1e-10), and B+ s = y."""
    rng = np.random.default_rng(5)
    n = 30
    h0 = rng.uniform(0.5, 2.0, n)
    B = Bfgs.diagonal(h0)
    Bd = np.diag(h0)
    for _ in range(10):
        M = rng.normal(size=(n, n))
        M = M @ M.T + n * np.eye(n)
        s = rng.normal(size=n)
        y = M @ s
        ok, theta, *_ = bfgs_update(B, s, y)
        assert ok and theta == 1.0
        Bs = Bd @ s
        Bd = Bd - np.outer(Bs, Bs) / (s @ Bs) + np.outer(y, y) / (y @ s)
        assert np.linalg.norm(B.apply(s) - y) <= 1e-10 * np.linalg.norm(y)
    assert np.max(np.abs(B.dense() - Bd)) <= 1e-10 * np.max(np.abs(Bd))
    assert B.U.shape == (n, 20)                      # U is n x 2k (R16)
    assert np.all(np.linalg.eigvalsh(B.dense()) > 0)


def test_powell_damping_keeps_curvature():
    """s^T y < 0.2 s^T B s: theta makes y~^T s = 0.2 s^T B s exactly, B+ stays SPD."""
    rng = np.random.default_rng(2)
    n = 12
    B = Bfgs.diagonal(np.ones(n))
    s = rng.normal(size=n)
    y = -0.5 * s                                      # negative curvature
    ok, theta, Bs, a, yt, b = bfgs_update(B, s, y)
    assert ok and 0.0 < theta < 1.0
    assert abs(yt @ s - 0.2 * (s @ s)) <= 1e-12 * (s @ s)
    assert np.all(np.linalg.eigvalsh(B.dense()) > 0)


def test_rosenbrock_known_minimum():
    """Rosenbrock, -5 <= x <= 5, no linear rows -> (1, 1), f ~ 0."""
    f = lambda x: 100.0 * (x[1] - x[0] ** 2) ** 2 + (1.0 - x[0]) ** 2
    g = lambda x: np.array([-400.0 * x[0] * (x[1] - x[0] ** 2) - 2.0 * (1.0 - x[0]), 200.0 * (x[1] - x[0] ** 2)])
    A = sp.csr_matrix((0, 2))
    r = sqp_solve(f, g, np.ones(2), A, np.zeros(0), np.zeros(0), np.full(2, -5.0), np.full(2, 5.0),
                  np.array([-1.2, 1.0]), SqpOptions(max_iter=200, tol_d=1e-10))
    assert r.status == "converged"
    assert np.max(np.abs(r.x - 1.0)) <= 1e-5 and r.f <= 1e-10


def test_convex_qp_posed_as_nlp():
    """kappa = 0: f is the quadratic 1/2 ||W^1/2 (D x - p)||^2, so the NLP is the QP with
    H = D^T W D, g = -D^T W p; SQP must reach that QP's solution."""
    from oracle.ipm import Problem, solve
    q = dose_nlp(30, 60, 5, 10, density=0.3, seed=4)
    q.kappa[:] = 0.0
    r = sqp_dose(q, SqpOptions(max_iter=300, tol_d=1e-7))
    assert r.status == "converged"
    Dd = q.D_scipy().toarray()
    H = Dd.T @ (q.w[:, None] * Dd)
    ref = solve(Problem(H=H, g=-Dd.T @ (q.w * q.p), A=q.A_scipy(), l=q.l, u=q.u, xl=q.xl, xu=q.xu))
    assert np.max(np.abs(r.x - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x)))


@pytest.mark.parametrize("seed", range(3))
def test_dose_nlp_matches_slsqp_and_descends(seed):
    q = nlp_config("S1", seed)
    r = sqp_dose(q, SqpOptions(max_iter=200, tol_d=1e-7))
    assert r.status == "converged"
    fs = [t["f"] for t in r.trace]
    assert all(b <= a + 1e-14 * abs(a) for a, b in zip(fs, fs[1:]))      # merit nonincreasing
    Ad = q.A_scipy().toarray()
    cons = []
    for i in range(q.m):
        if np.isfinite(q.l[i]):
            cons.append(dict(type="ineq", fun=lambda x, i=i: Ad[i] @ x - q.l[i], jac=lambda x, i=i: Ad[i]))
        if np.isfinite(q.u[i]):
            cons.append(dict(type="ineq", fun=lambda x, i=i: q.u[i] - Ad[i] @ x, jac=lambda x, i=i: -Ad[i]))
    ref = so.minimize(lambda x: dose_objective(q, x), q.x0, jac=lambda x: dose_gradient(q, x), method="SLSQP",
                      bounds=list(zip(q.xl, q.xu)), constraints=cons, options=dict(ftol=1e-15, maxiter=2000))
    assert ref.success
    # the IPM stops at mu_tol = 1e-8 (R6): active variables sit O(mu) inside their bounds, so f
    # carries an O(||grad f||_1 mu) offset -> 1e-7 relative
    assert abs(r.f - ref.fun) <= 1e-7 * abs(ref.fun)
    assert np.max(np.abs(r.x - ref.x)) <= 1e-4 * max(1.0, np.max(np.abs(ref.x)))
