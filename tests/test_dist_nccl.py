"""NCCL-bootstrapped row-sharded solves on separate GPUs (comm_kind 1, one process per GPU
under torchrun; the per-iteration data plane is peer memory over NVLink, peer.cu).  Skipped
below 2 GPUs — every gpurun lease and the round-end driver have one GPU; the same code path is
exercised on one GPU by test_dist_peer.py (IPC between processes) and test_gpu_shard.py."""
import os
import sys

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from test_dist_peer import run_workers  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_nccl_sharded_matches_oracle_and_repeats(nproc, tmp_path):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    from gen.planted import planted_qp
    from oracle.ipm import Problem, solve
    res = run_workers(nproc, "nccl", tmp_path / "r.json", ["--nvars", "2000", "--mrows", "500", "--seed", "45"])
    r0, r1 = res["runs"]
    assert r0["status"] == ["ok"] * nproc and len(set(r0["obj"])) == 1
    assert r0["x"] == r1["x"] and r0["pcg_iters"] == r1["pcg_iters"]      # bitwise at fixed P
    q = planted_qp(2000, 500, density=0.02, rank=32, seed=45, rows="vmat", var="box")
    ref = solve(Problem.from_data(q))
    x = np.array(r0["x"])
    assert np.max(np.abs(x - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x)))
    assert abs(r0["obj"][0] - ref.obj) <= 1e-8 * abs(ref.obj)
    assert abs(r0["ipm_iters"][0] - ref.iters) <= 2
