"""C5 full solve on ONE B200 (n = 100 000, m = 20 000, H = 80 GB): the QP to convergence,
checked against its planted optimum (x*, f*).  Run with IPM_DEBUG=1 to stream per-IPM-iteration
progress lines (mu, KKT residual, PCG iterations) to stderr."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from gen.planted import config
from gen.torch_io import device_hessian, problem_tensors
from paper_2405_03584_b200 import QP
dev = torch.device("cuda", 0)
q = config("C5", 0)
H, ldh = device_hessian(q, dev)
t = problem_tensors(q, dev, H=H, ldh=ldh)
qp = QP(device=dev, trace=1, **t)
t0 = time.time()
st = qp.solve()
s = qp.stats()
x = qp.solution()["x"].cpu().numpy()
print(json.dumps({"workload": "C5", "status": st, "wall_s": time.time() - t0, **s,
                  "max_err_x_planted": float(np.abs(x - q.x_star).max()),
                  "rel_err_f_planted": abs(s["obj"] - q.f_star) / abs(q.f_star)}), flush=True)
for r in qp.trace():
    print(json.dumps(r), flush=True)
