"""Proton-H&N-shaped QP with the paper's compact quasi-Newton Hessian (Table 1 / P:294):
n = 77373 variables, bound constraints only, U with 2k = 198 columns (SQP iteration 99).
Times the two skinny passes (the paper's Table 2 'gemv transpose' U^T x and 'gemv' U v) as one
compact operator apply, and a full QP solve."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from gen.planted import planted_qp
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP

n, k = int(os.environ.get("PROTON_N", 77373)), int(os.environ.get("PROTON_K", 198))
q = planted_qp(n, 0, rank=k, seed=0, var="box", name="proton-hn")
dev = torch.device("cuda", 0)
t = problem_tensors(q, dev, H=torch.zeros(2, dtype=torch.float64, device=dev), ldh=n)
t["H"] = None
qp = QP(device=dev, compact=dict(h0=q.d, U=q.U, w=q.w, k=k), **t)
ms = qp.profile("gemv", 50)
bytes_ = 2 * 8.0 * n * k + 8.0 * 3 * n
print(json.dumps({"workload": "proton-hn compact", "n": n, "2k": k, "op_apply_ms": ms,
                  "GBps_two_passes": bytes_ / ms / 1e6,
                  "paper_table2_us": {"rtx4080 gemv+gemvT": 189.12 + 199.36, "a100 gemv+gemvT": 111.39 + 103.78}}),
      flush=True)
st = qp.solve()
s = qp.stats()
x = qp.solution()["x"].cpu().numpy()
print(json.dumps({"status": st, "qp_solve_s": s["t_solve_ms"] / 1e3, "ipm": s["ipm_iters"], "pcg": s["pcg_iters_total"],
                  "x_err_planted": float(np.max(np.abs(x - q.x_star))), "obj_rel": abs(s["obj"] - q.f_star) / abs(q.f_star)}),
      flush=True)
