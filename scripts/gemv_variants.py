"""Time the three GEMV variants (LDG tiles, TMA-bulk, symmetric TMA-bulk) on a workload."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP
wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
q = config(wl, 0)
t = problem_tensors(q, torch.device("cuda", 0))
n = q.n
for gk in (1, 2, 3):
    qp = QP(device="cuda:0", gemv_kernel=gk, **t)
    ms = qp.profile("gemv", 20)
    it = qp.profile("pcg_iter", 20)
    full = 8.0 * n * n
    print(json.dumps({"workload": wl, "gemv_kernel": gk, "gemv_ms": ms, "pcg_iter_ms": it,
                      "effective_GBps(8n^2/t)": full / ms / 1e6,
                      "streamed_GBps": (full if gk < 3 else 4.0 * n * n + 4.0 * n * 256) / ms / 1e6}), flush=True)
    qp.close()
