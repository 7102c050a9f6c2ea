"""NEXT-4: the closed-loop SQP driver (include/sqp.h) against the SQP oracle (oracle/sqp.py)
on the same seeded dose-like NLPs (gen/dose_nlp.py).  Each QP subproblem is solved by the
GPU IPM (PCG directions) on the GPU side and by the exact-Cholesky oracle IPM on the CPU
side, so trajectories agree to the QP solve accuracy, and the limits to the SQP tolerance."""
import numpy as np
import pytest
import torch

from gen.dose_nlp import dose_nlp, nlp_config
from oracle.sqp import SqpOptions, dose_gradient, dose_objective, sqp_dose

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def _sqp(q, **kw):
    from paper_2405_03584_b200 import SQP
    return SQP.from_nlp(q, device=DEV, **kw)


@pytest.mark.parametrize("n,nd,kd,m", [(40, 80, 6, 12), (3000, 9000, 40, 800), (1, 1, 1, 0)])
def test_objective_and_gradient_match_oracle(n, nd, kd, m):
    q = dose_nlp(n, nd, kd, m, density=min(1.0, 0.02 + 2.0 / n), seed=n)
    s = _sqp(q)
    rng = np.random.default_rng(1)
    for x in (q.x0, q.xu * rng.uniform(size=n)):
        f, g = s.eval(x)
        fr, gr = dose_objective(q, x), dose_gradient(q, x)
        assert abs(f - fr) <= 1e-13 * abs(fr)
        assert np.linalg.norm(g.cpu().numpy() - gr) <= 1e-13 * max(1e-300, np.linalg.norm(gr))


@pytest.mark.parametrize("hess_kind", [0, 1])
@pytest.mark.parametrize("seed", range(3))
def test_sqp_matches_oracle(seed, hess_kind):
    q = nlp_config("S1", seed)
    ref = sqp_dose(q, SqpOptions(max_iter=200))
    s = _sqp(q, hess_kind=hess_kind, max_iter=200)
    assert s.solve(q.x0) == "ok" and ref.status == "converged"
    x = s.x().cpu().numpy()
    st, tr = s.stats(), s.trace()
    assert np.max(np.abs(x - ref.x)) <= 1e-5 * max(1.0, np.max(np.abs(ref.x)))
    assert abs(st["f"] - ref.f) <= 1e-7 * abs(ref.f)
    # the first steps follow the oracle's trajectory (same QPs up to the PCG tolerance)
    for a, b in zip(tr[:3], ref.trace[:3]):
        assert abs(a["f"] - b["f"]) <= 1e-7 * abs(b["f"])
        assert a["step"] == b["step"]
    assert abs(st["iters"] - ref.iters) <= max(3, ref.iters // 4)


def test_dense_and_compact_hessians_agree():
    q = dose_nlp(600, 1500, 30, 150, density=0.03, seed=9)
    a = _sqp(q, hess_kind=0, max_iter=60)
    b = _sqp(q, hess_kind=1, max_iter=60)
    a.solve(q.x0)
    b.solve(q.x0)
    xa, xb = a.x().cpu().numpy(), b.x().cpu().numpy()
    assert np.max(np.abs(xa - xb)) <= 1e-5 * max(1.0, np.max(np.abs(xa)))
    assert b.trace()[-1]["ncols"] == 2 * sum(r["updated"] for r in b.trace())


def test_warm_started_subproblems_reach_the_same_optimum():
    q = nlp_config("S1", 5)
    ref = sqp_dose(q, SqpOptions(max_iter=200))
    s = _sqp(q, warm_start=1, max_iter=200)
    assert s.solve(q.x0) == "ok"
    assert np.max(np.abs(s.x().cpu().numpy() - ref.x)) <= 1e-5 * max(1.0, np.max(np.abs(ref.x)))


def test_convex_qp_posed_as_nlp_reaches_qp_solution():
    from oracle.ipm import Problem, solve
    q = dose_nlp(30, 60, 5, 10, density=0.3, seed=4)
    q.kappa[:] = 0.0
    s = _sqp(q, max_iter=300, tol_d=1e-7)
    assert s.solve(q.x0) == "ok"
    Dd = q.D_scipy().toarray()
    ref = solve(Problem(H=Dd.T @ (q.w[:, None] * Dd), g=-Dd.T @ (q.w * q.p), A=q.A_scipy(), l=q.l, u=q.u,
                        xl=q.xl, xu=q.xu))
    assert np.max(np.abs(s.x().cpu().numpy() - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x)))


def test_repeat_solve_bitwise_and_merit_descends():
    q = dose_nlp(500, 1200, 24, 100, density=0.03, seed=2)
    s = _sqp(q, max_iter=40)
    s.solve(q.x0)
    x1, t1 = s.x().clone(), s.trace()
    s.solve(q.x0)
    untimed = lambda tr: [{k: v for k, v in r.items() if not k.endswith("_ms")} for r in tr]  # noqa: E731
    assert torch.equal(x1, s.x()) and untimed(t1) == untimed(s.trace())
    fs = [r["f"] for r in t1]
    assert all(b <= a for a, b in zip(fs, fs[1:]))


def test_invalid_inputs_rejected():
    from paper_2405_03584_b200 import _lib
    q = nlp_config("S1", 0)
    s = _sqp(q)
    with pytest.raises(_lib.IpmError, match="x0 violates"):
        s.solve(q.xu * 1.5)
    bad = nlp_config("S1", 0)
    bad.w[3] = 0.0
    with pytest.raises(_lib.IpmError, match="w must be"):
        _sqp(bad)
    with pytest.raises(_lib.IpmError, match="options"):
        _sqp(q, powell=1.5)
