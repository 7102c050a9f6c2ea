"""NEXT-2: PCG on the doubly augmented system eq:2x2_augmented instead of
the condensed Schur system (D1).  Unknowns (dx, dlam_lA, dlam_uA); the operator is applied as
H v + Sigma_b v + A^T (2 Sigma_c A v + v_l - v_u) on the top block and +-A v + D v_lam on the
middle block, never assembled.  Parity: one Newton step against the oracle's exact solve of
the same 2x2 system (oracle.newton.doubly_augmented_solve), and whole IPM solves against the
oracle's Alg. 1."""
import numpy as np
import pytest
import torch

from gen.planted import config, planted_qp
from gen.torch_io import problem_tensors
from oracle.ipm import Options, Problem, full_multipliers, initial_point, recover_step, reduced_system, \
    residuals, solve, max_step, FAMILIES
from oracle.newton import doubly_augmented_solve

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def _qp(q, **opts):
    from paper_2405_03584_b200 import QP
    return QP(device=DEV, **problem_tensors(q, DEV), **opts)


def _oracle_aug_step(q):
    """Alg. 1 lines 2-7 once from the R5 starting point, direction from the exact solve of
    eq:2x2_augmented (not the condensed Cholesky the oracle's solve() uses)."""
    p = Problem.from_data(q)
    opt = Options()
    it = initial_point(p, opt)
    r = residuals(p, it)
    Q, B, D, r1, r2 = reduced_system(p, it, r)
    dx, dlam, _ = doubly_augmented_solve(Q, B, D, r1, r2)
    ds, dl = recover_step(p, it, r, dx, dlam)
    ax, al = max_step(it.s, ds, opt.tau), max_step(it.lam, dl, opt.tau)
    x1 = it.x + ax * dx
    lam1 = {f: it.lam[f] + al * dl[f] for f in FAMILIES}
    it1 = it.copy()
    it1.x, it1.lam = x1, lam1
    return p, it, it1


@pytest.mark.parametrize("n,m,rows,var", [(600, 200, "mixed", "mixed"), (300, 1500, "vmat", "box"),
                                          (1100, 90, "upper", "none")])
def test_one_augmented_newton_step_matches_oracle(n, m, rows, var):
    q = planted_qp(n, m, density=0.03, rank=32, seed=n + m, rows=rows, var=var)
    p, it0, it1 = _oracle_aug_step(q)
    qp = _qp(q, pcg_system=1, max_ipm_iter=1)
    qp.solve()
    x, s, lam, _ = qp.get_iterate()
    x = x.cpu().numpy()
    # D6 stops PCG at rtol <= 1e-6 of ||rhs||: the step agrees to that order
    step = np.linalg.norm(it1.x - it0.x)
    assert np.linalg.norm(x - it1.x) <= 1e-4 * step
    full = full_multipliers(p, it1)
    for f in ("lA", "uA", "lx", "ux"):
        got = lam[f].cpu().numpy()
        assert np.linalg.norm(got - full[f]) <= 1e-4 * max(1.0, np.linalg.norm(full[f])), f


@pytest.mark.parametrize("seed", range(4))
def test_augmented_ipm_C1_matches_oracle(seed):
    q = config("C1", seed)
    qp = _qp(q, pcg_system=1)
    assert qp.solve() == "ok"
    ref = solve(Problem.from_data(q))
    x = qp.solution()["x"].cpu().numpy()
    assert np.max(np.abs(x - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x)))
    assert abs(qp.stats()["obj"] - ref.obj) <= 1e-8 * max(1.0, abs(ref.obj))
    assert abs(qp.stats()["ipm_iters"] - ref.iters) <= 2


@pytest.mark.parametrize("n,m,rows,var", [(1200, 400, "vmat", "box"), (900, 300, "mixed", "mixed")])
def test_augmented_ipm_medium_matches_oracle_and_condensed(n, m, rows, var):
    q = planted_qp(n, m, density=0.02, rank=48, seed=7, rows=rows, var=var)
    a = _qp(q, pcg_system=1)
    c = _qp(q)
    assert a.solve() == "ok" and c.solve() == "ok"
    ref = solve(Problem.from_data(q))
    xa = a.solution()["x"].cpu().numpy()
    assert np.max(np.abs(xa - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x)))
    assert abs(a.stats()["obj"] - ref.obj) <= 1e-8 * max(1.0, abs(ref.obj))
    assert abs(a.stats()["ipm_iters"] - ref.iters) <= 2
    print(f"\nPCG iterations n={n} m={m}: augmented {a.stats()['pcg_iters_total']} "
          f"condensed {c.stats()['pcg_iters_total']}")


def test_augmented_deterministic_and_graph_equals_host_loop():
    q = planted_qp(700, 150, density=0.03, rank=32, seed=12, rows="mixed", var="mixed")
    a = _qp(q, pcg_system=1, use_graph=1)
    b = _qp(q, pcg_system=1, use_graph=0)
    a.solve()
    x1 = a.solution()["x"].clone()
    a.solve()
    b.solve()
    assert torch.equal(x1, a.solution()["x"]) and torch.equal(x1, b.solution()["x"])


def test_augmented_without_rows_is_condensed():
    """m = 0: eq:2x2_augmented has no middle block, the option is a no-op (bitwise)."""
    q = planted_qp(500, 0, rank=20, seed=3, var="box")
    a, c = _qp(q, pcg_system=1), _qp(q)
    a.solve()
    c.solve()
    assert torch.equal(a.solution()["x"], c.solution()["x"])


def test_augmented_rejections():
    from paper_2405_03584_b200 import _lib
    q = config("C1", 0)
    a = _qp(q, pcg_system=1)
    with pytest.raises(_lib.IpmError, match="condensed"):
        a.pcg(np.ones(q.n), np.ones(q.m), np.ones(q.n), 1e-8)
    with pytest.raises(_lib.IpmError, match="pcg_system"):
        _qp(q, pcg_system=2)
