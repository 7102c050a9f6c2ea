"""Experiment: SYMV time vs tile order (IPM_SYM_ORDER: 0 row-major contiguous ranges, 1
interleaved across CTAs) on a workload; prints one JSON line per setting (separate processes)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen.planted import config
from gen.torch_io import device_hessian, problem_tensors
from paper_2405_03584_b200 import QP
wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
q = config(wl, 0)
dev = torch.device("cuda", 0)
H, ldh = device_hessian(q, dev)
t = problem_tensors(q, dev, H=H, ldh=ldh)
qp = QP(device=dev, max_ipm_iter=1, pcg_max_iter=20 if wl != "C5" else 3, **t)
qp.solve()
g = qp.profile("gemv", 10 if wl == "C5" else 30)
it = qp.profile("pcg_iter", 5 if wl == "C5" else 30)
n = q.n
nb = (n + 255) // 256
sizes = [min(256, n - i * 256) for i in range(nb)]
tri = 8.0 * sum(sizes[i] * sizes[j] for i in range(nb) for j in range(i, nb))
print(json.dumps({"workload": wl, "order": os.environ.get("IPM_SYM_ORDER", "0"), "gemv_ms": g, "pcg_iter_ms": it,
                  "streamed_GBps": tri / g / 1e6}), flush=True)
