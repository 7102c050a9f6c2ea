"""Per-PCG-iteration time of the tiny-problem PCG kernels (k_pcg_warp for n <= 64, else
k_pcg_small): ipm_pcg_iterate with k = 100 and k = 1000 on the C1 operator, wall time around
synchronised calls, (T1000 - T100) / 900.  IPM_PCG_WARP=0 forces k_pcg_small."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen.planted import config  # noqa: E402
from gen.torch_io import problem_tensors  # noqa: E402
from paper_2405_03584_b200 import QP  # noqa: E402

dev = torch.device("cuda", 0)
q = config(sys.argv[1] if len(sys.argv) > 1 else "C1", 0)
qp = QP(device=dev, **problem_tensors(q, dev))
rng = np.random.default_rng(0)
sb = torch.from_numpy(rng.uniform(0.0, 3.0, q.n)).to(dev)
sc = torch.from_numpy(10.0 ** rng.uniform(-2, 2, q.m)).to(dev)
b = torch.from_numpy(rng.normal(size=q.n)).to(dev)


def t(k, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        qp.pcg_iterate(sb, sc, b, k)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


t(10)
t100, t1000 = t(40), t(340)
print(json.dumps({"workload": q.n, "IPM_PCG_WARP": os.environ.get("IPM_PCG_WARP", "1"),
                  "us_per_pcg_iter": (t1000 - t100) / 300 * 1e6, "t40_ms": t100 * 1e3, "t340_ms": t1000 * 1e3}))
qp.solve()
ts, tp, tw = [], [], []
for _ in range(5):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    qp.solve()
    tw.append((time.perf_counter() - w0) * 1e3)
    ts.append(qp.stats()["t_solve_ms"])
    tp.append(qp.stats()["t_pcg_ms"])
print(json.dumps({"qp_solve_ms_median": sorted(ts)[2], "t_pcg_ms_median": sorted(tp)[2],
                  "wall_ms_median": sorted(tw)[2], "ipm_iters": qp.stats()["ipm_iters"],
                  "pcg_iters": qp.stats()["pcg_iters_total"], "IPM_TINY": os.environ.get("IPM_TINY", "1")}))
