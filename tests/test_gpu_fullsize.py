"""Parity at BASELINE.json's full C3 size, in the configuration bench.py times (auto kernel
selection = symmetric GEMV, CUDA-graph PCG): sampled operator rows computed one by one on the
host, and the whole QP against the planted optimum and the oracle's stored IPM count
(tests/golden/oracle_counts.json, written by scripts/oracle_reference_counts.py)."""
import json
import os

import numpy as np
import pytest
import torch

from gen.planted import config, hessian_rows
from gen.torch_io import problem_tensors

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


@pytest.fixture(scope="module")
def c3():
    from paper_2405_03584_b200 import QP
    q = config("C3", 0)
    t = problem_tensors(q, DEV)
    qp = QP(device=DEV, **t)
    yield q, qp
    qp.close()


def test_c3_operator_rows_sampled(c3):
    q, qp = c3
    assert qp.info()["gemv_kernel"] == 3            # the benchmarked configuration
    rng = np.random.default_rng(11)
    sb = rng.uniform(0.0, 3.0, q.n)
    sc = 10.0 ** rng.uniform(-3, 3, q.m)
    v = rng.normal(size=q.n)
    y = qp.op_apply(sb, sc, v).cpu().numpy()
    A = q.A_scipy()
    ATt = A.T @ (sc * (A @ v))
    rows = np.sort(rng.choice(q.n, size=48, replace=False))
    for i in rows:
        Hi = hessian_rows(q.d, q.U, q.w, int(i), int(i) + 1)[0]
        terms = np.concatenate([Hi * v, [sb[i] * v[i], ATt[i]]]).astype(np.longdouble)
        ref = float(terms.sum())
        scale = float(np.abs(Hi * v).sum() + abs(sb[i] * v[i]) + abs(ATt[i]))
        assert abs(y[i] - ref) <= 1e-13 * scale, i


def test_c3_qp_matches_planted_and_oracle_count(c3):
    q, qp = c3
    assert qp.solve() == "ok"
    st = qp.stats()
    x = qp.solution()["x"].cpu().numpy()
    assert np.max(np.abs(x - q.x_star)) <= 1e-6 * np.max(np.abs(q.x_star))
    assert abs(st["obj"] - q.f_star) <= 1e-8 * abs(q.f_star)
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_counts.json")))["C3/seed0"]
    assert abs(st["ipm_iters"] - ref["ipm_iters"]) <= 2
    assert abs(st["obj"] - ref["obj"]) <= 1e-8 * abs(ref["obj"])
