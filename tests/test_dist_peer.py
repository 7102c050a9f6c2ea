"""Multi-PROCESS row-sharded solves through the peer-memory data plane.

* Two processes sharing cuda:0, bootstrapped over a gloo process group (comm_kind 3): every
  exchange of the PCG loop is a CUDA-IPC store into the other process's workspace plus a flag
  (peer.cu) — the same code path separate GPUs take over NVLink.  The result must equal the
  in-process two-rank group's bit for bit (same kernels, same fixed-order combines), match the
  oracle, and repeat bitwise.
* test_dist_nccl.py covers NCCL-bootstrapped ranks on separate GPUs (skipped below 2 GPUs).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_workers(nproc, mode, out, extra=(), timeout=600):
    env = dict(os.environ, IPM_PEER_TIMEOUT_S=os.environ.get("IPM_PEER_TIMEOUT_S", "60"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "dist_worker.py"),
           "--mode", mode, "--out", str(out), *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    return json.load(open(out))


def test_two_processes_share_one_gpu_over_ipc(tmp_path):
    from gen.planted import planted_qp
    from gen.torch_io import problem_tensors
    from oracle.ipm import Problem, solve
    from paper_2405_03584_b200 import QP
    from paper_2405_03584_b200.dist import LocalGroup, partition
    res = run_workers(2, "host", tmp_path / "r.json", ["--same-gpu", "--nvars", "600", "--mrows", "150", "--seed", "44"])
    assert res["ws"] == 2 and res["sharded"] == 1
    r0, r1 = res["runs"]
    assert r0["status"] == ["ok", "ok"]
    assert len(set(r0["obj"])) == 1                          # identical combined scalars on both ranks
    x = np.array(r0["x"])
    assert np.array_equal(x, np.array(r1["x"])) and r0["pcg_iters"] == r1["pcg_iters"]   # bitwise repeat
    # the in-process two-rank group (raw pointers instead of IPC) computes the same bits
    dev = torch.device("cuda", 0)
    q = planted_qp(600, 150, density=0.02, rank=32, seed=44, rows="vmat", var="box")
    t = problem_tensors(q, dev)
    grp = LocalGroup(2)
    fns = []
    for r, (b, e) in enumerate(partition(q.n, 2)):
        tr = dict(t)
        tr["H"] = t["H"][b:e].contiguous()
        fns.append(lambda r=r, tr=tr: QP(device=dev, stream=torch.cuda.Stream(dev), shard=grp.shard(r), **tr))
    qps = grp.run(fns)
    grp.run([qq.solve for qq in qps])
    xin = torch.cat([qq.solution()["x"] for qq in qps]).cpu().numpy()
    assert np.array_equal(x, xin)
    assert r0["ipm_iters"][0] == qps[0].stats()["ipm_iters"]
    ref = solve(Problem.from_data(q))
    assert np.max(np.abs(x - ref.x)) <= 1e-6 * max(1.0, np.max(np.abs(ref.x)))
    assert abs(r0["obj"][0] - ref.obj) <= 1e-8 * abs(ref.obj)
