"""Generator checks: planted KKT point, exact dyadic H, paper-shaped splits."""
import json
import os

import numpy as np

from gen.planted import VMAT_LOWER_FRACTION, config, dense_hessian, hessian_rows, planted_qp
from oracle import kkt as okkt

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_hand_examples.json")))


def test_planted_point_is_kkt():
    for seed in range(3):
        q = config("C1", seed)
        H = q.H
        A = q.A_dense()
        c = okkt.kkt_certificate(H, q.g, A, q.l, q.u, q.xl, q.xu, q.x_star, q.lam_lA, q.lam_uA, q.lam_lx, q.lam_ux)
        assert c["stationarity"] < 1e-12
        assert c["infeasibility"] < 1e-12
        assert c["min_multiplier"] == 0.0
        assert c["complementarity"] < 1e-12
        assert abs(0.5 * q.x_star @ H @ q.x_star + q.g @ q.x_star - q.f_star) < 1e-12 * abs(q.f_star)


def test_hessian_exact_and_order_independent():
    """D5: H entries are exact dyadics, so any summation order gives identical bits."""
    q = planted_qp(300, 0, rank=64, seed=2)
    H1 = dense_hessian(q.d, q.U, q.w)
    # reversed-order accumulation, one rank-1 term at a time
    H2 = np.zeros_like(H1)
    for r in reversed(range(q.U.shape[1])):
        H2 += q.w[r] * np.outer(q.U[:, r], q.U[:, r])
    H2[np.diag_indices_from(H2)] += q.d
    assert np.array_equal(H1, H2)
    assert np.array_equal(hessian_rows(q.d, q.U, q.w, 17, 93), H1[17:93])
    assert np.array_equal(H1, H1.T)
    assert np.linalg.eigvalsh(H1).min() > 0.99


def test_vmat_split_and_shapes():
    q = planted_qp(2000, 1000, density=0.01, seed=1, rows="vmat")
    nl = int(np.isfinite(q.l).sum())
    nu = int(np.isfinite(q.u).sum())
    assert nl + nu == 1000 and not np.any(np.isfinite(q.l) & np.isfinite(q.u))
    assert nl == round(VMAT_LOWER_FRACTION * 1000)
    g = GOLD["vmat_split"]
    assert abs(VMAT_LOWER_FRACTION - g["lower_rows"] / (g["lower_rows"] + g["upper_rows"])) < 1e-15
    # CSR invariants
    for i in range(q.m):
        c = q.A_col[q.A_rowptr[i]:q.A_rowptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    assert q.nnz == 1000 * 20


def test_generator_is_pure():
    a = config("C1", 4)
    b = config("C1", 4)
    for f in ("g", "A_val", "l", "u", "xl", "xu", "x_star"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_c4_sequence_stays_planted():
    """after every BFGS rank-2 update of H, the random walk of x* (5 % active-set
    flips) re-plants the row bounds and g_k, so x*_k is the exact optimum of each QP of the sequence — checked by the oracle
    (x* and f*_k within its duality-gap error)."""
    from gen.sqp_sequence import sqp_sequence
    from oracle.bfgs import rank2_update
    from oracle.ipm import Problem, solve
    q = planted_qp(300, 80, density=0.05, rank=16, seed=3, rows="vmat", var="box")
    ups = sqp_sequence(q, 4, seed=0)
    H = q.H.copy()
    for up in ups:
        H = rank2_update(H, up.u, up.alpha, up.v, up.beta)
        r = solve(Problem(H=H, g=up.g.copy(), A=q.A_scipy(), l=up.l, u=up.ub, xl=q.xl, xu=q.xu))
        assert r.status == "converged"
        assert np.max(np.abs(r.x - up.x_star)) <= 1e-6
        assert abs(r.obj - up.f_star) <= 1e-8 * abs(up.f_star)
