"""PCG tolerance schedules vs IPM-iteration parity (reading R11: the paper states no CG
tolerance).  For each problem: the oracle's IPM count (exact Cholesky directions) and, per
schedule, the GPU IPM count, total PCG iterations, |x - x_oracle| and the relative objective
error.  One JSON line per (problem, schedule)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from gen.planted import config, planted_qp, random_small_qp
from gen.torch_io import problem_tensors
from oracle.ipm import Problem, solve
from paper_2405_03584_b200 import QP

SCHED = {
    "D6 (default)": {},
    "D6' factor 1e-2, floor 1e-10, max 1e-4": dict(pcg_rtol_mu_factor=1e-2, pcg_rtol_floor=1e-10, pcg_rtol_max=1e-4),
    "SPEC S:238": dict(pcg_schedule=1),
}
probs = [(f"C1/s{s}", config("C1", s)) for s in range(8)]
probs += [(f"rand12x8/s{s}", random_small_qp(12, 8, s, density=0.5)) for s in range(4)]
probs += [("vmat300x1500", planted_qp(300, 1500, density=0.05, rank=32, seed=13, rows="vmat", var="box")),
          ("medium1200x400", planted_qp(1200, 400, density=0.02, rank=48, seed=7, rows="vmat", var="box"))]
if "--c3" in sys.argv:
    probs.append(("C3", config("C3", 0)))
dev = torch.device("cuda", 0)
oracle_counts = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "oracle_counts.json")))
for name, q in probs:
    if name == "C3":
        oi, ox, of = oracle_counts["C3/seed0"]["ipm_iters"], q.x_star, oracle_counts["C3/seed0"]["obj"]
    else:
        r = solve(Problem.from_data(q))
        oi, ox, of = r.iters, r.x, r.obj
    t = problem_tensors(q, dev)
    for sname, opts in SCHED.items():
        if name == "C3" and sname.startswith("SPEC"):
            continue
        qp = QP(device=dev, max_ipm_iter=60, **t, **opts)
        st = qp.solve(raise_on_error=False)
        s = qp.stats()
        x = qp.solution()["x"].cpu().numpy()
        print(json.dumps({"problem": name, "schedule": sname, "status": st, "oracle_ipm": oi, "gpu_ipm": s["ipm_iters"],
                          "pcg_total": s["pcg_iters_total"],
                          "x_err": float(np.max(np.abs(x - ox)) / max(1.0, np.max(np.abs(ox)))),
                          "obj_rel": abs(s["obj"] - of) / max(1.0, abs(of))}), flush=True)
        qp.close()
