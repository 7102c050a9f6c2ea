"""NEXT-1: the paper's matrix-free compact quasi-Newton Hessian H = diag(h0) + U diag(w) U^T
(eq:bfgs_hessian), applied as h0 o p + U (w o (U^T p)) without assembling H.
Parity against the oracle on the assembled dense H (the generator's factors ARE such a form)."""
import numpy as np
import pytest
import torch

from gen.planted import planted_qp
from gen.torch_io import problem_tensors
from oracle import kkt as okkt
from oracle.ipm import Problem, solve

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def _compact_qp(q, extra_cols=0, **opts):
    from paper_2405_03584_b200 import QP
    t = problem_tensors(q, DEV)
    t["H"] = None
    k = q.U.shape[1]
    U = np.zeros((q.n, k + extra_cols))
    U[:, :k] = q.U
    return QP(device=DEV, compact=dict(h0=q.d, U=U, w=q.w, k=k), **t, **opts)


@pytest.mark.parametrize("n,m,r", [(1, 1, 1), (300, 40, 17), (2000, 500, 198), (5001, 0, 300)])
def test_compact_apply_and_diag(n, m, r):
    q = planted_qp(n, m, density=min(1.0, 0.02 + 2.0 / n), rank=r, seed=n + r, rows="mixed" if m else "vmat",
                   var="mixed")
    qp = _compact_qp(q)
    assert qp.info()["ncb"] == 1
    rng = np.random.default_rng(3)
    sb, sc, v = rng.uniform(0, 3, q.n), 10 ** rng.uniform(-3, 3, q.m), rng.normal(size=q.n)
    y = qp.op_apply(sb, sc, v).cpu().numpy()
    yref = okkt.condensed_apply(q.H, q.A_dense(), sb, sc, v, dtype=np.longdouble).astype(np.float64)
    assert np.linalg.norm(y - yref) <= 1e-12 * np.linalg.norm(yref)
    d = qp.op_diag(sb, sc).cpu().numpy()
    assert np.max(np.abs(d - okkt.jacobi_diag(q.H, q.A_dense(), sb, sc)) / d) <= 1e-13


@pytest.mark.parametrize("n,m,r", [(1500, 300, 40), (120, 30, 9)])
def test_compact_ipm_matches_oracle(n, m, r):
    """(120, 30): n below the single-CTA PCG threshold, which needs the dense H and must not
    be chosen for a compact Hessian (regression: it read H = NULL)."""
    q = planted_qp(n, m, density=0.02 if n > 1000 else 0.15, rank=r, seed=17, rows="vmat", var="box")
    qp = _compact_qp(q)
    assert qp.solve() == "ok"
    ref = solve(Problem.from_data(q))
    x = qp.solution()["x"].cpu().numpy()
    st = qp.stats()
    assert np.max(np.abs(x - ref.x)) <= 1e-6 * np.max(np.abs(ref.x))
    assert abs(st["obj"] - ref.obj) <= 1e-8 * abs(ref.obj)
    assert abs(st["ipm_iters"] - ref.iters) <= 2


def test_compact_rank2_append_secant():
    """The rank-2 update appends (u, v) as two new columns; H+ s = y."""
    q = planted_qp(800, 60, density=0.05, rank=12, seed=4)
    qp = _compact_qp(q, extra_cols=4)
    rng = np.random.default_rng(1)
    s = rng.normal(size=q.n)
    y = s * (1.0 + rng.uniform(size=q.n))
    u = q.H @ s
    qp.update_hessian_rank2(u, -1.0 / (s @ u), y, 1.0 / (y @ s))
    Hs = qp.op_apply(np.zeros(q.n), np.zeros(q.m), s).cpu().numpy()
    assert np.linalg.norm(Hs - y) <= 1e-12 * np.linalg.norm(y)
    qp.update_hessian_rank2(u, 0.0, y, 0.0)
    from paper_2405_03584_b200 import _lib
    with pytest.raises(_lib.IpmError, match="full"):
        qp.update_hessian_rank2(u, 0.0, y, 0.0)
