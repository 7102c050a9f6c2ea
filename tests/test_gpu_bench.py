"""bench.py (our arm) keeps the driver's JSON-line contract: one line on rank 0 with the metric,
the roofline and cpu_baseline objects, e2e through host buffers, a launch count and the clocks
line — and it finishes inside the driver's budget at the driver's own flags (--steps 20
--warmup 5).  The default workload is C5 (80 GB H); these tests run the same code path on C3
(3.2 GB H, the multi-CTA operator kernels the roofline times live) and on C1 (the single-CTA
PCG), so they take seconds to a minute."""
import json
import os
import subprocess
import sys
import time

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks")


def _run(*extra, timeout=900):
    t0 = time.time()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *extra], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    wall = time.time() - t0
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0]), wall


def test_bench_driver_flags_c3_within_budget():
    d, wall = _run("--workload", "C3", "--steps", "20", "--warmup", "5", "--no-extra")
    # C3 is 25x smaller than C5 in H bytes; the same flags must stay far inside the driver's 1800 s
    assert wall < 300, wall
    for k in KEYS:
        assert k in d, k
    assert d["unit"] == "PCG it/s" and d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 5
    assert d["dtype"] == "f64" and d["config"]["workload"] == "C3" and d["status"] == ["not_converged"]
    assert len(d["pcg_iters_per_step"]) == 1          # identical work in every step (deterministic)
    assert d["pcg_iters_job"] == 20 * d["pcg_iters_per_step"][0]
    assert abs(d["ms_per_step"] * 20 / 1e3 - d["pcg_iters_job"] / d["value"]) < 1e-6 * d["ms_per_step"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9 and rf["launches_timed"] >= 20
    assert rf["timing"].startswith("live") and 0 < rf["share_of_step"] < 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 8 * 20000 and e["d2h_bytes_per_step"] == 8 * 20000
    assert d["gpu_launches"] > 0
    assert d["clocks"]["samples"] >= 0


def test_bench_c1_single_cta_path():
    d, _ = _run("--workload", "C1", "--steps", "3", "--warmup", "3", "--no-extra", "--no-cpu-baseline")
    assert d["value"] > 0 and d["roofline"]["launches_timed"] == 0 and d["cpu_baseline"] is None


def test_bench_two_ranks_sharded_same_gpu():
    """The N > 1 branch of bench.py (torchrun, barriers, max over ranks, the row-sharded QP with
    the peer data plane, e2e) on one GPU: two processes share cuda:0 (--same-gpu: gloo bootstrap,
    CUDA IPC exchanges), C3 forced sharded."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, IPM_PEER_TIMEOUT_S="60")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--same-gpu", "--workload", "C3", "--shard", "--steps", "1", "--warmup", "1",
                        "--no-extra", "--no-cpu-baseline"], capture_output=True, text=True, timeout=1200, cwd=ROOT,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["parallelism"].startswith("row-sharded")
    assert len(d["pcg_iters_per_step"]) == 1 and abs(d["pcg_iters_per_step"][0] - 67) <= 2   # one GPU: 67
