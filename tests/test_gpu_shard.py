"""Row-sharded path on one GPU: P virtual ranks as P contexts of an
in-process group (comm_kind 2), each on its own stream and host thread.  The kernels,
partition, allgathers and rank-ordered combines are exactly the multi-GPU path's; only the
allgather transport differs from NCCL."""
import numpy as np
import pytest
import torch

from gen.planted import config, planted_qp
from gen.torch_io import device_hessian, problem_tensors
from oracle import kkt as okkt
from oracle.ipm import Problem, solve

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def _sharded(q, P, H=None, **opts):
    from paper_2405_03584_b200 import QP
    from paper_2405_03584_b200.dist import LocalGroup, partition
    t = problem_tensors(q, DEV) if H is None else dict(problem_tensors(q, DEV), H=H)
    grp = LocalGroup(P)
    fns = []
    for r, (b, e) in enumerate(partition(q.n, P)):
        tr = dict(t)
        tr["H"] = t["H"][b:e].contiguous()
        fns.append(lambda r=r, tr=tr: QP(device=DEV, stream=torch.cuda.Stream(DEV), shard=grp.shard(r), **tr, **opts))
    # ipm_create is collective when sharded (the symmetry certificate is exchanged): every
    # rank's context is created concurrently, as separate processes would under NCCL
    return grp, grp.run(fns)


def _solve_all(grp, qps):
    st = grp.run([q.solve for q in qps])
    xs = [q.solution()["x"] for q in qps]
    torch.cuda.synchronize()
    return st, torch.cat(xs).cpu().numpy(), [q.stats() for q in qps]


def test_sharded_p1_is_bitwise_the_unsharded_path():
    """P = 1 through the sharded code path (allgathers + k_xcombine) reproduces the
    one-GPU path bit for bit (the combine applies the same epilogue in the same order)."""
    from paper_2405_03584_b200 import QP
    q = planted_qp(900, 250, density=0.03, rank=32, seed=8, rows="mixed", var="mixed")
    a = QP(device=DEV, gemv_kernel=2, **problem_tensors(q, DEV))   # the sharded path's GEMV
    a.solve()
    grp, qps = _sharded(q, 1, gemv_kernel=2)
    st, x, stats = _solve_all(grp, qps)
    assert st == ["ok"]
    assert np.array_equal(a.solution()["x"].cpu().numpy(), x)
    assert stats[0]["ipm_iters"] == a.stats()["ipm_iters"]
    assert stats[0]["pcg_iters_total"] == a.stats()["pcg_iters_total"]


def test_nccl_transport_single_rank():
    """The NCCL backend (dlopen'd libnccl, ncclCommInitRank, ncclAllGather) with one rank runs
    the sharded path and reproduces the unsharded solve bitwise."""
    from paper_2405_03584_b200 import QP
    from paper_2405_03584_b200.dist import nccl_shard, nccl_unique_id
    q = planted_qp(600, 150, density=0.03, rank=32, seed=21, rows="mixed", var="mixed")   # n > kSmallN
    t = problem_tensors(q, DEV)
    a = QP(device=DEV, gemv_kernel=2, **t)
    a.solve()
    b = QP(device=DEV, gemv_kernel=2, shard=nccl_shard(0, 1, nccl_unique_id()), **t)
    assert b.info()["sharded"] == 1
    assert b.solve() == "ok"
    assert torch.equal(a.solution()["x"], b.solution()["x"])


@pytest.mark.parametrize("P", [2, 3, 4])
def test_sharded_matches_oracle(P):
    q = planted_qp(1001, 300, density=0.02, rank=32, seed=40 + P, rows="vmat", var="box")
    grp, qps = _sharded(q, P)
    st, x, stats = _solve_all(grp, qps)
    assert st == ["ok"] * P
    ref = solve(Problem.from_data(q))
    assert np.max(np.abs(x - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x)))
    objs = {s["obj"] for s in stats}
    assert len(objs) == 1                                  # every rank holds the same combined scalars
    assert abs(stats[0]["obj"] - ref.obj) <= 1e-8 * abs(ref.obj)
    assert len({s["ipm_iters"] for s in stats}) == 1
    assert abs(stats[0]["ipm_iters"] - ref.iters) <= 2
    assert abs(stats[0]["obj"] - q.f_star) <= 1e-8 * abs(q.f_star)


def test_sharded_bitwise_reproducible():
    q = config("C1", 5)
    runs = []
    for _ in range(2):
        grp, qps = _sharded(q, 2, trace=1)
        st, x, stats = _solve_all(grp, qps)
        runs.append((x, [qq.trace() for qq in qps]))
    assert np.array_equal(runs[0][0], runs[1][0]) and runs[0][1] == runs[1][1]


def test_sharded_op_apply_rows():
    q = planted_qp(777, 200, density=0.03, rank=32, seed=2, rows="mixed")
    grp, qps = _sharded(q, 3)
    rng = np.random.default_rng(0)
    sb, sc, v = rng.uniform(0, 2, q.n), 10 ** rng.uniform(-2, 2, q.m), rng.normal(size=q.n)
    from paper_2405_03584_b200.dist import partition
    ys = grp.run([lambda r=r, qq=qq: qq.op_apply(sb[slice(*partition(q.n, 3)[r])], sc, v)
                  for r, qq in enumerate(qps)])
    y = torch.cat(ys).cpu().numpy()
    yref = okkt.condensed_apply(q.H, q.A_dense(), sb, sc, v, dtype=np.longdouble).astype(np.float64)
    assert np.linalg.norm(y - yref) <= 1e-12 * np.linalg.norm(yref)


@pytest.mark.parametrize("n,P", [(1000, 2), (1200, 3), (1000, 4), (2600, 5)])
def test_sharded_symmetric_op_apply(n, P):
    """Row-sharded symmetric GEMV (each rank reads ~n^2/(2P) entries of its row block; the
    column parts of other ranks' rows are exchanged): K v matches a longdouble reference."""
    q = planted_qp(n, 300, density=0.02, rank=32, seed=n + P, rows="mixed")
    grp, qps = _sharded(q, P)
    assert all(qq.info()["gemv_kernel"] == 3 for qq in qps)          # chunk even: symmetric path
    rng = np.random.default_rng(P)
    sb, sc, v = rng.uniform(0, 2, q.n), 10 ** rng.uniform(-2, 2, q.m), rng.normal(size=q.n)
    from paper_2405_03584_b200.dist import partition
    ys = grp.run([lambda r=r, qq=qq: qq.op_apply(sb[slice(*partition(q.n, P)[r])], sc, v)
                  for r, qq in enumerate(qps)])
    y = torch.cat(ys).cpu().numpy()
    yref = okkt.condensed_apply(q.H, q.A_dense(), sb, sc, v, dtype=np.longdouble).astype(np.float64)
    assert np.linalg.norm(y - yref) <= 1e-12 * np.linalg.norm(yref)


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_symmetric_matches_oracle_and_is_reproducible(P):
    q = planted_qp(1000, 300, density=0.02, rank=32, seed=60 + P, rows="vmat", var="box")
    runs = []
    for _ in range(2):
        grp, qps = _sharded(q, P)
        assert all(qq.info()["gemv_kernel"] == 3 for qq in qps)
        runs.append(_solve_all(grp, qps))
    (st, x, stats), (_, x2, _) = runs
    assert st == ["ok"] * P and np.array_equal(x, x2)
    ref = solve(Problem.from_data(q))
    assert np.max(np.abs(x - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x)))
    assert len({s["obj"] for s in stats}) == 1
    assert abs(stats[0]["obj"] - ref.obj) <= 1e-8 * abs(ref.obj)
    assert abs(stats[0]["ipm_iters"] - ref.iters) <= 2


def test_sharded_asymmetric_H_falls_back_on_every_rank():
    """One off-diagonal entry changed on ONE side (rank 1's rows only): the exchanged hash
    certificate fails on every rank, so all ranks take the full GEMV (auto) and
    gemv_kernel=3 is refused; the full GEMV stays exact for the stored (asymmetric) H."""
    from paper_2405_03584_b200 import _lib
    q = planted_qp(1000, 100, density=0.02, rank=16, seed=3)
    H = problem_tensors(q, DEV)["H"].clone()
    H[700, 10] += 1e-3                      # row 700 belongs to rank 1 of 2; H[10, 700] unchanged
    grp, qps = _sharded(q, 2, H=H)
    assert all(qq.info()["gemv_kernel"] != 3 for qq in qps)
    rng = np.random.default_rng(0)
    sb, sc, v = rng.uniform(0, 2, q.n), 10 ** rng.uniform(-2, 2, q.m), rng.normal(size=q.n)
    from paper_2405_03584_b200.dist import partition
    ys = grp.run([lambda r=r, qq=qq: qq.op_apply(sb[slice(*partition(q.n, 2)[r])], sc, v)
                  for r, qq in enumerate(qps)])
    Hn = H[:, :q.n].cpu().numpy()
    yref = okkt.condensed_apply(Hn, q.A_dense(), sb, sc, v, dtype=np.longdouble).astype(np.float64)
    assert np.linalg.norm(torch.cat(ys).cpu().numpy() - yref) <= 1e-12 * np.linalg.norm(yref)
    with pytest.raises(_lib.IpmError, match="symmetric"):
        _sharded(q, 2, H=H, gemv_kernel=3)


@pytest.mark.parametrize("P", [2, 3])
def test_a_row_split_spmv(P):
    """north_star's A-row partition (opt.a_row_split, default with the peer data plane): each rank
    forms t = Sigma_c o (A p) for its own rows of A and the slices are allgathered over peer
    memory on the SpMV side branch.  Same solution as the replicated SpMV (a_row_split = 0) up to
    the rounding of the S_c sum, and bitwise reproducible at fixed P."""
    q = planted_qp(1200, 500, density=0.02, rank=32, seed=60 + P, rows="vmat", var="box")
    grp, qps = _sharded(q, P)
    st, x, stats = _solve_all(grp, qps)
    st2, x2, _ = _solve_all(grp, qps)
    assert st == ["ok"] * P and np.array_equal(x, x2)
    grp_r, qps_r = _sharded(q, P, a_row_split=0)
    st_r, x_r, stats_r = _solve_all(grp_r, qps_r)
    assert st_r == ["ok"] * P
    assert np.max(np.abs(x - x_r)) <= 1e-7 * max(1.0, np.max(np.abs(x_r)))
    assert abs(stats[0]["ipm_iters"] - stats_r[0]["ipm_iters"]) <= 1
    ref = solve(Problem.from_data(q))
    assert np.max(np.abs(x - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x)))


@pytest.mark.parametrize("P", [2, 3])
def test_single_reduction_pcg(P):
    """Chronopoulos-Gear single-reduction PCG (opt.pcg_single_reduction, SURVEY NEXT-3's sharded
    variant): one scalar exchange per iteration.  Its k-step iterates equal the textbook PCG's
    (oracle.pcg) to rounding, and the IPM solve matches the oracle."""
    from oracle.pcg import pcg as oracle_pcg
    from paper_2405_03584_b200.dist import partition
    q = planted_qp(1200, 400, density=0.02, rank=32, seed=70 + P, rows="vmat", var="box")
    grp, qps = _sharded(q, P, pcg_single_reduction=1)
    rng = np.random.default_rng(3)
    sb, sc, b = rng.uniform(0.0, 3.0, q.n), 10.0 ** rng.uniform(-2, 2, q.m), rng.normal(size=q.n)
    parts = partition(q.n, P)
    A = q.A_scipy()
    K_apply = lambda v: q.H @ v + sb * v + A.T @ (sc * (A @ v))   # noqa: E731
    Minv = 1.0 / (np.diag(q.H) + sb + (A.multiply(A)).T @ sc)
    for k in (1, 3, 6):
        outs = grp.run([lambda qq=qq, r=r: qq.pcg_iterate(sb[parts[r][0]:parts[r][1]], sc,
                                                          b[parts[r][0]:parts[r][1]], k)
                        for r, qq in enumerate(qps)])
        ref = oracle_pcg(K_apply, Minv, b, maxit=k)
        for key, refv in (("x", ref.x), ("r", ref.r), ("p", ref.p)):
            g = np.concatenate([o[key].cpu().numpy() for o in outs])
            assert np.max(np.abs(g - refv)) <= 1e-10 * np.max(np.abs(refv)), (P, k, key)
        assert abs(outs[0]["alpha"] - ref.alpha) <= 1e-10 * abs(ref.alpha)
    st, x, stats = _solve_all(grp, qps)
    assert st == ["ok"] * P and len({s["obj"] for s in stats}) == 1
    ref = solve(Problem.from_data(q))
    assert np.max(np.abs(x - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x)))
    assert abs(stats[0]["ipm_iters"] - ref.iters) <= 2
