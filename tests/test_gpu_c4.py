"""C4 (SQP sequence): rank-2 quasi-Newton Hessian updates in place on the borrowed H,
new linear terms and warm starts, GPU vs oracle."""
import numpy as np
import pytest
import torch

from gen.planted import planted_qp
from gen.sqp_sequence import sqp_sequence
from oracle.bfgs import rank2_update
from gen.torch_io import problem_tensors
from oracle.ipm import Options, Problem, solve, warm_start_point

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def test_rank2_update_secant_equation():
    """BFGS update with u = H s, alpha = -1/s^T H s, v = y, beta = 1/y^T s gives H+ s = y
    (secant equation) and H = I, s = e1, y = 2 e1 -> diag(2, 1, ...)."""
    from paper_2405_03584_b200 import QP
    q = planted_qp(700, 50, density=0.05, rank=16, seed=3)
    t = problem_tensors(q, DEV)
    qp = QP(device=DEV, **t)
    rng = np.random.default_rng(0)
    s = rng.normal(size=q.n)
    y = s * (1.0 + rng.uniform(size=q.n))
    u = q.H @ s
    qp.update_hessian_rank2(u, -1.0 / (s @ u), y, 1.0 / (y @ s))
    zero_b, zero_c = np.zeros(q.n), np.zeros(q.m)
    Hs = qp.op_apply(zero_b, zero_c, s).cpu().numpy()
    assert np.linalg.norm(Hs - y) <= 1e-12 * np.linalg.norm(y)
    Hd = t["H"][:, :q.n]
    assert torch.equal(Hd, Hd.T)                       # update keeps H bitwise symmetric
    # S:380 hand case
    q2 = planted_qp(8, 0, rank=1, seed=0)
    q2.U[:] = 0.0
    q2.d[:] = 1.0
    q2._H = None
    t2 = problem_tensors(q2, DEV)
    qp2 = QP(device=DEV, **t2)
    e1 = np.zeros(8)
    e1[0] = 1.0
    qp2.update_hessian_rank2(e1, -1.0, 2 * e1, 0.5)
    assert np.array_equal(t2["H"][:, :8].cpu().numpy(), np.diag([2.0] + [1.0] * 7))
    d = qp2.op_diag(np.zeros(8), np.zeros(0)).cpu().numpy()
    assert np.array_equal(d, np.array([2.0] + [1.0] * 7))   # cached diag(H) follows the update


@pytest.mark.parametrize("seed", [0, 1])
def test_sqp_sequence_warm_start_matches_oracle(seed):
    from paper_2405_03584_b200 import QP
    q = planted_qp(1000, 250, density=0.02, rank=32, seed=30 + seed, rows="vmat", var="box")
    ups = sqp_sequence(q, K=4, seed=seed)
    t = problem_tensors(q, DEV)
    qp = QP(device=DEV, **t)
    assert qp.solve() == "ok"
    H = q.H.copy()
    p = Problem.from_data(q, H=H)
    ref = solve(p)
    for k, up in enumerate(ups):
        qp.update_hessian_rank2(up.u, up.alpha, up.v, up.beta)
        qp.set_linear_term(up.g)
        qp.set_bounds(up.l, up.ub, q.xl, q.xu)
        qp.warm_start()
        assert qp.solve() == "ok"
        sol = qp.solution()
        st = qp.stats()
        H = rank2_update(H, up.u, up.alpha, up.v, up.beta)
        p = Problem(H=H, g=up.g.copy(), A=q.A_scipy(), l=up.l, u=up.ub, xl=q.xl, xu=q.xu)
        ref = solve(p, Options(), start=warm_start_point(p, ref.x, ref.it.lam, Options()))
        assert ref.status == "converged"
        x = sol["x"].cpu().numpy()
        assert np.max(np.abs(x - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x))), k
        assert abs(sol["obj"] - ref.obj) <= 1e-8 * max(1.0, abs(ref.obj)), k
        assert abs(st["ipm_iters"] - ref.iters) <= 2, (k, st["ipm_iters"], ref.iters)


def test_set_bounds_validation():
    """ipm_set_bounds: new values accepted; a change of which bounds are finite, NaN or l >= u
    rejected with nothing changed (include/ipm.h)."""
    from paper_2405_03584_b200 import QP
    from paper_2405_03584_b200._lib import IpmError
    q = planted_qp(400, 100, density=0.05, rank=16, seed=5, rows="vmat", var="box")
    qp = QP(device=DEV, **problem_tensors(q, DEV))
    assert qp.solve() == "ok"
    l2, u2 = q.l - 0.01 * np.isfinite(q.l), q.u + 0.01 * np.isfinite(q.u)
    qp.set_bounds(l2, u2, q.xl, q.xu)
    ref = solve(Problem(H=q.H, g=q.g, A=q.A_scipy(), l=l2, u=u2, xl=q.xl, xu=q.xu))
    assert qp.solve() == "ok"
    assert np.max(np.abs(qp.solution()["x"].cpu().numpy() - ref.x)) <= 1e-6
    bad = l2.copy()
    bad[np.flatnonzero(np.isfinite(bad))[0]] = -np.inf
    with pytest.raises(IpmError):
        qp.set_bounds(bad, u2, q.xl, q.xu)
    bad = q.xu.copy()
    bad[0] = q.xl[0]
    with pytest.raises(IpmError):
        qp.set_bounds(l2, u2, q.xl, bad)
