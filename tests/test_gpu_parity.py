"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Tolerances are north_star's: operator apply <= 1e-12 relative (fp64),
final x <= 1e-6 relative, objective <= 1e-8 relative, IPM iterations within +-2."""
import numpy as np
import pytest
import torch

from gen.planted import config, planted_qp, random_small_qp
from gen.torch_io import device_hessian, problem_tensors
from oracle import kkt as okkt
from oracle.ipm import Options, Problem, full_multipliers, solve

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def _qp(q, **opts):
    from paper_2405_03584_b200 import QP
    return QP(device=DEV, **problem_tensors(q, DEV), **opts)


def _rand_sigmas(q, seed, dyadic=False):
    rng = np.random.default_rng(seed)
    if dyadic:
        sb = rng.integers(0, 64, size=q.n) / 16.0
        sc = rng.integers(0, 64, size=q.m) / 16.0
        v = rng.integers(-64, 64, size=q.n) / 8.0
    else:
        sb = rng.uniform(0.0, 3.0, size=q.n)
        sc = 10.0 ** rng.uniform(-3, 3, size=q.m)
        v = rng.normal(size=q.n)
    return sb, sc, v


# ---------------------------------------------------------------- operator apply / diag
@pytest.mark.parametrize("n,m,dens", [(50, 20, 0.3), (1, 1, 1.0), (1025, 300, 0.02), (3001, 0, 0.0),
                                      (2049, 700, 0.01), (4100, 1500, 0.05)])
def test_op_apply_matches_oracle(n, m, dens):
    q = planted_qp(n, m, density=dens, rank=min(64, n), seed=n + m, rows="mixed" if m else "vmat",
                   var="mixed")
    qp = _qp(q)
    sb, sc, v = _rand_sigmas(q, 1)
    y = qp.op_apply(sb, sc, v).cpu().numpy()
    A = q.A_dense()
    yref = okkt.condensed_apply(q.H, A, sb, sc, v, dtype=np.longdouble)
    err = np.linalg.norm((y - yref).astype(np.float64)) / np.linalg.norm(yref.astype(np.float64))
    assert err <= 1e-12, err
    d = qp.op_diag(sb, sc).cpu().numpy()
    dref = okkt.jacobi_diag(q.H, A, sb, sc)
    assert np.max(np.abs(d - dref) / np.abs(dref)) <= 1e-13


def test_op_apply_bit_exact_on_dyadic_inputs():
    """Every product and partial sum exact in fp64 -> GPU == numpy bit for bit, whatever the
    summation order (SURVEY.md §8(c) 'Operator apply')."""
    q = planted_qp(1500, 400, density=0.02, rank=32, seed=9, rows="mixed")
    q.A_val = np.round(q.A_val * 16) / 16.0
    qp = _qp(q)
    sb, sc, v = _rand_sigmas(q, 2, dyadic=True)
    y = qp.op_apply(sb, sc, v).cpu().numpy()
    yref = okkt.condensed_apply(q.H, q.A_dense(), sb, sc, v)
    assert np.array_equal(y, yref)


@pytest.mark.parametrize("n", [777, 2048, 3071])
def test_gemv_kernels_agree_bitwise(n):
    """LDG-tile and TMA-bulk GEMV variants accumulate every (row, column block) partial in
    the same lane order, so K v is bit-identical between them."""
    q = planted_qp(n, 200, density=0.02, rank=32, seed=n, rows="mixed")
    a = _qp(q, gemv_kernel=1)
    b = _qp(q, gemv_kernel=2)
    sb, sc, v = _rand_sigmas(q, 3)
    ya = a.op_apply(sb, sc, v)
    yb = b.op_apply(sb, sc, v)
    assert torch.equal(ya, yb)
    yref = okkt.condensed_apply(q.H, q.A_dense(), sb, sc, v, dtype=np.longdouble).astype(np.float64)
    assert np.linalg.norm(yb.cpu().numpy() - yref) <= 1e-12 * np.linalg.norm(yref)


@pytest.mark.parametrize("n,m", [(1, 1), (255, 30), (256, 0), (300, 0), (700, 50), (1000, 200), (2049, 500),
                                 (5003, 300), (12000, 0)])
def test_symmetric_gemv_matches_oracle(n, m):
    """gemv_kernel=3 reads only the upper block triangle of the (exactly symmetric) H."""
    q = planted_qp(n, m, density=min(1.0, 0.02 + 2.0 / n), rank=min(48, n), seed=n + 3 * m,
                   rows="mixed" if m else "vmat", var="mixed")
    qp = _qp(q, gemv_kernel=3)
    sb, sc, v = _rand_sigmas(q, 4)
    y = qp.op_apply(sb, sc, v).cpu().numpy()
    yref = okkt.condensed_apply(q.H, q.A_dense(), sb, sc, v, dtype=np.longdouble).astype(np.float64)
    assert np.linalg.norm(y - yref) <= 1e-12 * np.linalg.norm(yref)
    # and it is the auto choice for a symmetric H
    assert _qp(q).profile("gemv", 1) > 0


def test_symmetric_gemv_rejected_for_asymmetric_H():
    from paper_2405_03584_b200 import QP, _lib
    q = planted_qp(300, 20, density=0.05, rank=16, seed=1)
    t = problem_tensors(q, DEV)
    t["H"][3, 7] += 1e-3          # H != H^T
    with pytest.raises(_lib.IpmError, match="symmetric"):
        QP(device=DEV, gemv_kernel=3, **t)
    qp = QP(device=DEV, **t)      # auto falls back to the full GEMV and stays exact
    sb, sc, v = _rand_sigmas(q, 1)
    H = t["H"][:, :q.n].cpu().numpy()
    yref = okkt.condensed_apply(H, q.A_dense(), sb, sc, v, dtype=np.longdouble).astype(np.float64)
    y = qp.op_apply(sb, sc, v).cpu().numpy()
    assert np.linalg.norm(y - yref) <= 1e-12 * np.linalg.norm(yref)


@pytest.mark.parametrize("gk", [1, 2, 3])
def test_ipm_both_gemv_kernels(gk):
    q = planted_qp(1500, 300, density=0.02, rank=32, seed=11, rows="vmat", var="box")
    _check_against_oracle(q, dict(gemv_kernel=gk))


def test_device_hessian_bitwise_equals_numpy():
    q = planted_qp(777, 0, rank=64, seed=4)
    H, ldh = device_hessian(q, DEV)
    assert np.array_equal(H[:, :q.n].cpu().numpy(), q.H)


# ---------------------------------------------------------------- PCG
def test_pcg_identity_and_jacobi_exact():
    """K = I converges in 1 iteration; diagonal K with Jacobi in 1."""
    n = 64
    d = np.zeros(n)
    q = planted_qp(n, 0, rank=1, seed=0)
    q.U[:] = 0.0
    q.d[:] = 1.0
    q._H = None
    qp = _qp(q)
    rhs = np.random.default_rng(0).normal(size=n)
    x, it = qp.pcg(np.zeros(n), np.zeros(0), rhs, 1e-12)
    assert it == 1 and np.allclose(x.cpu().numpy(), rhs, rtol=0, atol=1e-14)
    x, it = qp.pcg(np.arange(1.0, n + 1) - 1.0, np.zeros(0), rhs, 1e-12)   # K = diag(1..n)
    assert it == 1
    assert np.max(np.abs(x.cpu().numpy() - rhs / np.arange(1.0, n + 1))) <= 1e-14


@pytest.mark.parametrize("seed", range(3))
def test_pcg_solves_condensed_system(seed):
    q = planted_qp(800, 300, density=0.03, rank=48, seed=seed, rows="mixed", var="mixed")
    qp = _qp(q)
    sb, sc, _ = _rand_sigmas(q, seed)
    sc = np.minimum(sc, 10.0)
    K = okkt.condensed_matrix(q.H, q.A_dense(), sb, sc)
    rhs = np.random.default_rng(seed).normal(size=q.n)
    x, it = qp.pcg(sb, sc, rhs, 1e-10)
    x = x.cpu().numpy()
    assert np.linalg.norm(rhs - K @ x) <= 1.0000001e-10 * np.linalg.norm(rhs)
    xref = np.linalg.solve(K, rhs)
    assert np.max(np.abs(x - xref)) <= 1e-6 * np.max(np.abs(xref))


def test_pcg_deterministic():
    q = planted_qp(2000, 500, density=0.02, rank=32, seed=3)
    qp = _qp(q)
    sb, sc, _ = _rand_sigmas(q, 5)
    rhs = np.random.default_rng(1).normal(size=q.n)
    x1, i1 = qp.pcg(sb, sc, rhs, 1e-9)
    x2, i2 = qp.pcg(sb, sc, rhs, 1e-9)
    assert i1 == i2 and torch.equal(x1, x2)


# ---------------------------------------------------------------- whole IPM vs oracle
def _check_against_oracle(q, opts_gpu=None, opts_or=None, xtol=1e-6, ftol=1e-8, ittol=2):
    qp = _qp(q, **(opts_gpu or {}))
    status = qp.solve()
    sol = qp.solution()
    st = qp.stats()
    ref = solve(Problem.from_data(q), opts_or or Options())
    x = sol["x"].cpu().numpy()
    assert status == "ok" and ref.status == "converged", (status, st)
    assert np.max(np.abs(x - ref.x)) <= xtol * max(1.0, np.max(np.abs(ref.x))), np.max(np.abs(x - ref.x))
    assert abs(sol["obj"] - ref.obj) <= ftol * max(1.0, abs(ref.obj))
    assert abs(st["ipm_iters"] - ref.iters) <= ittol, (st["ipm_iters"], ref.iters)
    return qp, sol, st, ref


@pytest.mark.parametrize("seed", range(8))
def test_ipm_C1_matches_oracle(seed):
    q = config("C1", seed)
    _, sol, _, _ = _check_against_oracle(q)
    assert np.max(np.abs(sol["x"].cpu().numpy() - q.x_star)) <= 1e-6 * np.max(np.abs(q.x_star))


@pytest.mark.parametrize("seed", range(4))
def test_ipm_random_small_matches_oracle(seed):
    q = random_small_qp(12, 8, seed, density=0.5)
    _check_against_oracle(q)


@pytest.mark.parametrize("seed", range(3))
def test_ipm_mehrotra_matches_oracle(seed):
    q = config("C1", seed)
    _check_against_oracle(q, dict(predictor_corrector=1), Options(predictor_corrector=True))


def test_ipm_medium_planted_and_oracle():
    q = planted_qp(1200, 400, density=0.02, rank=48, seed=7, rows="vmat", var="box")
    qp, sol, st, ref = _check_against_oracle(q)
    assert abs(sol["obj"] - q.f_star) <= 1e-8 * abs(q.f_star)


def test_ipm_box_only_and_odd_n():
    q = planted_qp(1537, 0, rank=40, seed=2, var="box")
    _check_against_oracle(q)


def test_ipm_no_bounds_one_step():
    q = planted_qp(300, 0, rank=50, seed=1, var="none")
    qp = _qp(q)
    assert qp.solve() == "ok"
    assert qp.stats()["ipm_iters"] == 1
    x = qp.solution()["x"].cpu().numpy()
    xcf = np.linalg.solve(q.H, -q.g)
    assert np.max(np.abs(x - xcf)) <= 1e-9 * np.max(np.abs(xcf))


def test_ipm_vmat_ratio_more_rows_than_variables():
    """VMAT H&N has ~5 linear constraints per variable (Table 1): m > n."""
    q = planted_qp(300, 1500, density=0.05, rank=32, seed=13, rows="vmat", var="box")
    _check_against_oracle(q)


def test_ipm_empty_rows_and_single_variable():
    q = planted_qp(40, 12, density=0.1, rank=8, seed=3, rows="mixed", var="mixed")
    # empty the CSR rows 2 and 7 (their bounds stay valid: 0 in [l, u] is not required,
    # an empty row is a constant 0 <= u or l <= 0 constraint -> drop its bounds)
    keep = np.ones(q.nnz, bool)
    for i in (2, 7):
        keep[q.A_rowptr[i]:q.A_rowptr[i + 1]] = False
        q.l[i], q.u[i] = -np.inf, np.inf
    lens = np.diff(q.A_rowptr).copy()
    lens[[2, 7]] = 0
    q.A_col, q.A_val = q.A_col[keep], q.A_val[keep]
    q.A_rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    _check_against_oracle(q, ftol=1e-8)
    q1 = planted_qp(1, 1, density=1.0, rank=1, seed=2, rows="upper", var="box")
    _check_against_oracle(q1)


def test_ipm_deterministic_bitwise():
    q = planted_qp(900, 300, density=0.03, rank=32, seed=5, rows="mixed", var="mixed")
    qp = _qp(q, trace=1)
    qp.solve()
    x1 = qp.solution()["x"].clone()
    t1 = qp.trace()
    qp.solve()
    x2 = qp.solution()["x"].clone()
    assert torch.equal(x1, x2) and t1 == qp.trace()


def test_host_loop_fallback_equals_graph():
    """The CUDA-graph PCG (device WHILE node) and the host-driven loop launch the same kernels
    in the same order: bitwise identical (n > 256, so the single-CTA path is not used)."""
    q = planted_qp(700, 150, density=0.03, rank=32, seed=12, rows="mixed", var="mixed")
    a = _qp(q, use_graph=1)
    b = _qp(q, use_graph=0)
    a.solve()
    b.solve()
    assert torch.equal(a.solution()["x"], b.solution()["x"])


@pytest.mark.parametrize("shape", ["C1", "h_global", "t_global"])
def test_single_cta_pcg_small_n(shape):
    """n <= 256: the whole PCG loop in one CTA (launch-latency path) agrees with the
    multi-kernel host loop to rounding and with the oracle — with everything staged in shared
    memory (C1), with H read from global memory (n = 200: 320 KB > the 200 KB budget) and with
    t and A in global memory (n = 64, m = 30000)."""
    if shape == "C1":
        q = config("C1", 6)
    elif shape == "h_global":
        q = planted_qp(200, 50, density=0.1, rank=64, seed=6, rows="mixed", var="mixed")
    else:   # m >> n: no well-posed planted QP, so only the PCG hook runs on it
        q = planted_qp(64, 30000, density=0.05, rank=32, seed=7, rows="mixed", var="mixed")
    a = _qp(q)               # single-CTA PCG
    b = _qp(q, use_graph=0)  # multi-kernel loop
    if shape != "t_global":
        assert a.solve() == "ok" and b.solve() == "ok"
        xa, xb = a.solution()["x"].cpu().numpy(), b.solution()["x"].cpu().numpy()
        assert np.max(np.abs(xa - xb)) <= 1e-9 * max(1.0, np.max(np.abs(xb)))
        assert abs(a.stats()["ipm_iters"] - b.stats()["ipm_iters"]) <= 1
    sb, sc, _ = _rand_sigmas(q, 9)
    sc = np.minimum(sc, 10.0)
    K = okkt.condensed_matrix(q.H, q.A_dense(), sb, sc)
    rhs = np.random.default_rng(2).normal(size=q.n)
    x, it = a.pcg(sb, sc, rhs, 1e-11)
    assert np.linalg.norm(rhs - K @ x.cpu().numpy()) <= 1.0000001e-11 * np.linalg.norm(rhs)
    xb_, itb = b.pcg(sb, sc, rhs, 1e-11)
    assert np.max(np.abs(x.cpu().numpy() - xb_.cpu().numpy())) <= 1e-8 * np.max(np.abs(xb_.cpu().numpy()))
    # the k-step recurrence of the single-CTA loop against the textbook PCG (oracle.pcg)
    from oracle.pcg import pcg as oracle_pcg
    ref = oracle_pcg(lambda v: K @ v, 1.0 / np.diag(K), rhs, maxit=4)
    out = a.pcg_iterate(sb, sc, rhs, 4)
    assert np.max(np.abs(out["x"].cpu().numpy() - ref.x)) <= 1e-11 * np.max(np.abs(ref.x))


# ---------------------------------------------------------------- validation / errors
def test_invalid_inputs_rejected():
    from paper_2405_03584_b200 import QP, _lib
    q = config("C1", 0)
    t = problem_tensors(q, DEV)
    bad = dict(t)
    col = t["A_col"].clone()
    col[1], col[0] = col[0].item(), col[1].item()   # unsorted row
    bad["A_col"] = col
    with pytest.raises(_lib.IpmError, match="strictly increasing"):
        QP(device=DEV, **bad)
    bad = dict(t)
    l = t["l"].clone()
    i = int(torch.nonzero(torch.isfinite(t["l"]) & torch.isfinite(t["u"]))[0])
    l[i] = t["u"][i]
    bad["l"] = l
    with pytest.raises(_lib.IpmError, match="lower < upper"):
        QP(device=DEV, **bad)
    bad = dict(t)
    H = t["H"].clone()
    H[3, 7] = float("nan")
    bad["H"] = H
    with pytest.raises(_lib.IpmError, match="non-finite"):
        QP(device=DEV, **bad)


@pytest.mark.parametrize("n,m", [(300, 0), (2049, 500), (12000, 0)])
def test_symmetric_gemv_interleaved_order(n, m, monkeypatch):
    """IPM_SYM_ORDER=1: the same tiles in an interleaved per-CTA order (and so different carry
    splits) — K v still matches the longdouble reference, and bitwise on dyadic inputs."""
    monkeypatch.setenv("IPM_SYM_ORDER", "1")
    q = planted_qp(n, m, density=min(1.0, 0.02 + 2.0 / n), rank=min(48, n), seed=n + 3 * m,
                   rows="mixed" if m else "vmat", var="mixed")
    if m:
        q.A_val = np.round(q.A_val * 16) / 16.0
    qp = _qp(q, gemv_kernel=3)
    sb, sc, v = _rand_sigmas(q, 4)
    y = qp.op_apply(sb, sc, v).cpu().numpy()
    yref = okkt.condensed_apply(q.H, q.A_dense(), sb, sc, v, dtype=np.longdouble).astype(np.float64)
    assert np.linalg.norm(y - yref) <= 1e-12 * np.linalg.norm(yref)
    sb, sc, v = _rand_sigmas(q, 5, dyadic=True)
    assert np.array_equal(qp.op_apply(sb, sc, v).cpu().numpy(), okkt.condensed_apply(q.H, q.A_dense(), sb, sc, v))


@pytest.mark.parametrize("seed", range(4))
def test_one_warp_ipm_matches_multi_kernel_path(seed):
    """n, m <= 64: the whole Algorithm 1 loop runs in one warp (tiny.cu).  It follows the
    multi-kernel path's formulas and stopping rules, so against that path (use_graph=0 keeps the
    tiny problem on it) the IPM count, the trace, x and the objective agree to rounding; the
    oracle comparison of the same problems is test_ipm_C1_matches_oracle."""
    q = config("C1", seed)
    a = _qp(q, trace=1)                 # one-warp path
    b = _qp(q, trace=1, use_graph=0)    # per-kernel host loop
    assert a.solve() == "ok" and b.solve() == "ok"
    sa, sb_ = a.stats(), b.stats()
    assert sa["ipm_iters"] == sb_["ipm_iters"]
    assert abs(sa["pcg_iters_total"] - sb_["pcg_iters_total"]) <= 0.2 * sb_["pcg_iters_total"]
    assert sa["t_pcg_ms"] > 0.0 and sa["t_pcg_ms"] <= sa["t_solve_ms"]
    xa, xb = a.solution()["x"].cpu().numpy(), b.solution()["x"].cpu().numpy()
    assert np.max(np.abs(xa - xb)) <= 1e-9 * max(1.0, np.max(np.abs(xb)))
    assert abs(sa["obj"] - sb_["obj"]) <= 1e-12 * abs(sb_["obj"])
    ta, tb = a.trace(), b.trace()
    assert len(ta) == len(tb) == sa["ipm_iters"]
    for ra, rb in zip(ta, tb):
        assert ra["it"] == rb["it"] and ra["mu"] == rb["mu"]
        # intermediate iterates carry the PCG tolerance of their iteration (rtol up to 1e-6, D6)
        assert abs(ra["obj"] - rb["obj"]) <= 1e-5 * max(1.0, abs(rb["obj"]))
    # a second solve from the stored state (warm start is the multi-kernel path's) still works
    a.warm_start()
    assert a.solve() == "ok"


def test_one_warp_ipm_iteration_limit():
    """max_ipm_iter reached on the one-warp path: IPM_NOT_CONVERGED with the iterate kept."""
    q = config("C1", 0)
    a = _qp(q, max_ipm_iter=3, trace=1)
    assert a.solve(raise_on_error=False) == "not_converged"
    s = a.stats()
    assert s["ipm_iters"] == 3 and len(a.trace()) == 3 and np.all(np.isfinite(a.solution()["x"].cpu().numpy()))
