"""C5 time to solution on ONE B200 (n = 100 000, m = 20 000, H = 80 GB fp64): Algorithm 1 to
convergence, one IPM iteration per ipm_solve call (max_ipm_iter = 1, the iterate and mu carried
over with ipm_get_iterate / ipm_set_iterate — exactly the trajectory of one long solve, since
every step is deterministic), so every IPM iteration is logged (flushed) as it completes and a
run cut off by a time limit still leaves its record.  Checked against the planted optimum.

  python scripts/c5_solve.py OUT.jsonl [--workload C5] [--max-hours 2]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen.planted import config  # noqa: E402
from gen.torch_io import device_hessian, problem_tensors  # noqa: E402
from paper_2405_03584_b200 import QP  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--workload", default="C5")
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--max-hours", type=float, default=2.0)
a = ap.parse_args()
dev = torch.device("cuda", 0)
log = open(a.out, "a")


def emit(d):
    log.write(json.dumps(d) + "\n")
    log.flush()


t_wall = time.time()
q = config(a.workload, a.seed)
H, ldh = device_hessian(q, dev)
t = problem_tensors(q, dev, H=H, ldh=ldh)
qp = QP(device=dev, max_ipm_iter=1, **t)
emit({"stage": "setup", "workload": a.workload, "n": q.n, "m": q.m, "nnz": q.nnz, "setup_s": time.time() - t_wall,
      "gemv_kernel": qp.info()["gemv_kernel"]})
total_ms = pcg_ms = 0.0
pcg_total = 0
status = "not_converged"
k = 0
for k in range(1, 101):
    if k > 1:
        qp.set_iterate(x, s, lam, mu)
    st = qp.solve()
    s_ = qp.stats()
    x, s, lam, mu = qp.get_iterate()
    total_ms += s_["t_solve_ms"]
    pcg_ms += s_["t_pcg_ms"]
    pcg_total += s_["pcg_iters_total"]
    emit({"it": k, "pcg_iters": s_["pcg_iters_total"], "pcg_total": pcg_total, "t_iter_s": s_["t_solve_ms"] / 1e3,
          "t_total_s": total_ms / 1e3, "mu_next": mu, "kkt_inf": s_["kkt_inf"], "obj": s_["obj"],
          "stalls": s_["pcg_stalls"], "status": st})
    if st == "ok":
        status = "converged"
        break
    if time.time() - t_wall > a.max_hours * 3600:
        status = "time_limit"
        break
xs = x.cpu().numpy()
emit({"stage": "result", "workload": a.workload, "status": status, "ipm_iters": k, "pcg_iters_total": pcg_total,
      "qp_solve_s": total_ms / 1e3, "t_pcg_s": pcg_ms / 1e3,
      "pcg_it_per_s": pcg_total / (pcg_ms * 1e-3) if pcg_ms > 0 else None,
      "max_err_x_planted": float(np.abs(xs - q.x_star).max()),
      "rel_err_f_planted": abs(s_["obj"] - q.f_star) / abs(q.f_star)})
