"""GPU vs oracle below the whole-solve level (SURVEY.md §8(c) "replay parity"), and the
error paths of ipm_solve.

* PCG-mode operator parity: ``ipm_pcg_iterate`` runs exactly k iterations of the PCG the solve
  runs (single-CTA loop for n <= 256, else the captured graph: SYMV in PCG mode with the fused
  p^T (H + Sigma_b) p, the SpMV / SpMV^T side branch, the fused cooperative update) and is
  compared element by element with ``oracle.pcg.pcg`` — the textbook recurrence on
  K = H + Sigma_b + A^T Sigma_c A evaluated from its definition (oracle.kkt).
* Per-IPM-iteration replay: the oracle's iterate k is put into the GPU with ipm_set_iterate,
  the GPU takes ONE Algorithm-1 iteration with its PCG at rtol 1e-12, and the new iterate is
  compared with the oracle's exact (Cholesky) step from the same iterate.
  This isolates the kernels from trajectory drift.
"""
import numpy as np
import pytest
import torch

from gen.planted import config, planted_qp
from gen.torch_io import problem_tensors
from oracle import kkt as okkt
from oracle.ipm import FAMILIES, Options, Problem, max_step, newton_direction, residuals, solve
from oracle.pcg import pcg as oracle_pcg

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def _qp(q, **opts):
    from paper_2405_03584_b200 import QP
    return QP(device=DEV, **problem_tensors(q, DEV), **opts)


def _problem(name):
    if name == "C1":
        return config("C1", 0)
    if name == "medium":
        return planted_qp(1200, 400, density=0.03, rank=48, seed=4, rows="mixed", var="mixed")
    if name == "vmat3000":
        return planted_qp(3000, 1500, density=0.02, rank=64, seed=2, rows="vmat", var="box")
    return config(name, 0)


# ---------------------------------------------------------------- PCG-mode operator parity
@pytest.mark.parametrize("name,ks", [("C1", (1, 2, 5)), ("medium", (1, 2, 5)), ("vmat3000", (1, 4)), ("C3", (1, 3))])
def test_pcg_iterate_matches_oracle_pcg(name, ks):
    q = _problem(name)
    qp = _qp(q)
    rng = np.random.default_rng(17)
    sb = rng.uniform(0.0, 3.0, q.n)
    sc = 10.0 ** rng.uniform(-2, 2, q.m)
    b = rng.normal(size=q.n)
    A = q.A_scipy()
    H = q.H
    rows = np.arange(q.n)
    apply_K = lambda v: okkt.condensed_apply_rows(H, rows, A, sb, sc, v)   # noqa: E731
    Minv = 1.0 / (np.diag(H) + sb + (A.multiply(A)).T @ sc)
    for k in ks:
        ref = oracle_pcg(apply_K, Minv, b, maxit=k)
        out = qp.pcg_iterate(sb, sc, b, k)
        assert not ref.breakdown and ref.iters == k
        # k iterations amplify rounding only mildly: element-wise within 1e-11 of each vector's scale
        for key, refv in (("x", ref.x), ("r", ref.r), ("z", ref.z), ("p", ref.p)):
            g = out[key].cpu().numpy()
            err = np.max(np.abs(g - refv)) / np.max(np.abs(refv))
            assert err <= 1e-11, (name, k, key, err)
        for key, refs in (("rho", ref.rho), ("pKp", ref.pKp), ("alpha", ref.alpha)):
            assert abs(out[key] - refs) <= 1e-11 * abs(refs), (name, k, key, out[key], refs)
        assert abs(out["rr"] - float(ref.r @ ref.r)) <= 1e-10 * float(ref.r @ ref.r)


def test_pcg_iterate_deterministic_and_consistent_with_pcg_solve():
    q = _problem("vmat3000")
    qp = _qp(q)
    rng = np.random.default_rng(5)
    sb, sc, b = rng.uniform(0.0, 3.0, q.n), 10.0 ** rng.uniform(-2, 2, q.m), rng.normal(size=q.n)
    a = qp.pcg_iterate(sb, sc, b, 7)
    c = qp.pcg_iterate(sb, sc, b, 7)
    for key in ("x", "r", "z", "p"):
        assert torch.equal(a[key], c[key])
    assert a["rho"] == c["rho"] and a["pKp"] == c["pKp"]


# ---------------------------------------------------------------- per-IPM-iteration replay
def _full(p, it):
    """Oracle compact iterate -> the ABI's masked full-length families (0 where absent)."""
    idx = {"lA": p.I_l, "uA": p.I_u, "lx": p.J_l, "ux": p.J_u}
    s, lam = {}, {}
    for f in FAMILIES:
        ln = p.m if f.endswith("A") else p.n
        s[f] = np.zeros(ln)
        lam[f] = np.zeros(ln)
        s[f][idx[f]] = it.s[f]
        lam[f][idx[f]] = it.lam[f]
    return s, lam


def _oracle_step(p, it, opt):
    from oracle.ipm import condensed_solve, recover_step, reduced_system
    r = residuals(p, it)
    Q, B, D, r1, r2 = reduced_system(p, it, r)
    dx, dlamA, (K, rhs, _) = condensed_solve(Q, B, D, r1, r2)
    ds, dl = recover_step(p, it, r, dx, dlamA)
    ax = max_step(it.s, ds, opt.tau)
    al = max_step(it.lam, dl, opt.tau)
    nx = it.copy()
    nx.x = it.x + ax * dx
    for f in FAMILIES:
        nx.s[f] = it.s[f] + ax * ds[f]
        nx.lam[f] = it.lam[f] + al * dl[f]
    return nx, dx, ax, al, K, rhs


@pytest.mark.parametrize("name,k", [("C1", 0), ("C1", 3), ("C1", 7), ("medium", 0), ("medium", 4),
                                    ("vmat3000", 2), ("C3", 0)])
def test_replay_one_ipm_iteration(name, k):
    q = _problem(name)
    p = Problem.from_data(q)
    opt = Options()
    if k > 0:
        it = solve(p, Options(max_iter=k)).it
    else:
        from oracle.ipm import initial_point
        it = initial_point(p, opt)
    nx, dx_or, ax, al, K, rhs = _oracle_step(p, it, opt)
    # the GPU at PCG rtol 1e-12 (schedule pinned to the floor) takes one Alg. 1 iteration
    qp = _qp(q, max_ipm_iter=1, pcg_rtol_max=1e-12, pcg_rtol_floor=1e-12, trace=1)
    s, lam = _full(p, it)
    qp.set_iterate(it.x, s, lam, it.mu)
    assert qp.solve() in ("ok", "not_converged")
    tr = qp.trace()[0]
    assert tr["pcg_relres"] <= 1e-12 * 1.0000001
    assert abs(tr["alpha_x"] - ax) <= 1e-9 and abs(tr["alpha_lam"] - al) <= 1e-9, (tr, ax, al)
    x, s_g, l_g, _ = qp.get_iterate()
    x_new = x.cpu().numpy()
    dx_gpu = (x_new - it.x) / tr["alpha_x"]
    # reconstructing dx from the iterate difference costs ~1 ulp of |x| per entry
    dx_rec = np.finfo(float).eps * (np.abs(it.x) + np.abs(x_new)) / tr["alpha_x"]
    # (1) the GPU direction solves the ORACLE's condensed system (its Sigma's, RHS, K assembled
    #     densely from the definition) to the PCG tolerance: pins a4, a5 and a6 together
    # (the GPU's own relres <= 1e-12 is on its K, formed in another order: the two K's differ by
    #  rounding, bounded by a few ulps of |K| |dx| — the fp64 backward-error term)
    #  and the two right-hand sides differ by the rounding of r_H = Hx + g - A^T lam - ..., whose
    #  terms cancel near convergence: bounded by a few ulps of their magnitudes)
    res = np.linalg.norm(K @ dx_gpu - rhs) / np.linalg.norm(rhs)
    back = np.linalg.norm(np.abs(K) @ np.abs(dx_gpu)) / np.linalg.norm(rhs)
    lam = _full(p, it)[1]
    Aa = abs(q.A_scipy())
    mag = (np.abs(q.H) @ np.abs(it.x) + np.abs(q.g) + Aa.T @ (lam["lA"] + lam["uA"]) + lam["lx"] + lam["ux"])
    back_rhs = np.linalg.norm(mag) / np.linalg.norm(rhs)
    back_rec = np.linalg.norm(np.abs(K) @ dx_rec) / np.linalg.norm(rhs)
    assert res <= 1.0000001e-12 + 64 * np.finfo(float).eps * (back + back_rhs) + 2 * back_rec, \
        (name, k, res, back, back_rhs, back_rec)
    # (2) and it equals the Cholesky direction within the conditioning of the Jacobi-scaled K
    dm = 1.0 / np.sqrt(np.diag(K))
    kappa = np.linalg.cond(K * dm[:, None] * dm[None, :]) if q.n <= 3000 else 1e3
    err = np.max(np.abs(dx_gpu - dx_or)) / np.max(np.abs(dx_or))
    assert err <= max(1e-9, 10.0 * kappa * 1e-12) + 2 * np.max(dx_rec) / np.max(np.abs(dx_or)), (name, k, err, kappa)
    # (3) recovery / step lengths / update: every family's change matches the oracle's step
    s_or, l_or = _full(p, nx)
    s0, l0 = _full(p, it)
    tol = max(1e-8, 100.0 * kappa * 1e-12)
    for f in FAMILIES:
        for gv, ov, base in ((s_g[f].cpu().numpy(), s_or[f], s0[f]), (l_g[f].cpu().numpy(), l_or[f], l0[f])):
            if ov.size == 0:
                continue
            d_or = ov - base
            scale = max(np.max(np.abs(d_or)), 1e-300)
            e = np.max(np.abs((gv - base) - d_or)) / scale
            assert e <= tol, (name, k, f, e, kappa)


# ---------------------------------------------------------------- error paths
def test_not_converged_keeps_best_iterate():
    q = config("C1", 0)
    # PCG at rtol 1e-12 so the two inexact directions stay within 1e-8 of the oracle's exact ones
    qp = _qp(q, max_ipm_iter=2, pcg_rtol_max=1e-12, pcg_rtol_floor=1e-12)
    assert qp.solve() == "not_converged"
    st = qp.stats()
    assert st["status"] == "not_converged" and st["ipm_iters"] == 2
    sol = qp.solution()
    x = sol["x"].cpu().numpy()
    assert np.all(np.isfinite(x)) and np.isfinite(sol["obj"])
    # the retrievable iterate is the one two oracle iterations produce (same trajectory)
    ref = solve(Problem.from_data(q), Options(max_iter=2))
    assert ref.status == "not_converged"
    assert np.max(np.abs(x - ref.x)) <= 1e-8 * max(1.0, np.max(np.abs(ref.x)))


@pytest.mark.parametrize("n", [50, 300])
def test_pcg_breakdown_on_indefinite_H(n):
    """H = -5 I makes K = H + Sigma_b negative definite at the initial point (Sigma_b = 2 on a
    two-sided box): the first p^T K p < 0 is a breakdown, on both PCG paths
    (single CTA for n <= 256, the graph otherwise)."""
    from paper_2405_03584_b200 import QP
    from paper_2405_03584_b200._lib import IpmError
    H = -5.0 * torch.eye(n, dtype=torch.float64, device=DEV)
    e = torch.zeros(0, dtype=torch.float64, device=DEV)
    qp = QP(H, torch.ones(n, dtype=torch.float64, device=DEV), torch.zeros(1, dtype=torch.int64, device=DEV),
            torch.zeros(0, dtype=torch.int32, device=DEV), e, e, e,
            torch.zeros(n, dtype=torch.float64, device=DEV), torch.ones(n, dtype=torch.float64, device=DEV) * 2,
            device=DEV)
    with pytest.raises(IpmError) as ei:
        qp.solve()
    assert "PCG_BREAKDOWN" in str(ei.value) or "breakdown" in str(ei.value).lower()
    assert qp.solve(raise_on_error=False) == "pcg_breakdown"
    assert qp.stats()["status"] == "pcg_breakdown"


def test_nonfinite_starting_iterate():
    q = config("C1", 1)
    p = Problem.from_data(q)
    from oracle.ipm import initial_point
    it = initial_point(p, Options())
    it.x[3] = np.nan
    qp = _qp(q)
    s, lam = _full(p, it)
    qp.set_iterate(it.x, s, lam, it.mu)
    assert qp.solve(raise_on_error=False) == "nonfinite"
    assert qp.stats()["status"] == "nonfinite"
    # the context stays usable: a cold solve afterwards converges
    assert qp.solve() == "ok"
