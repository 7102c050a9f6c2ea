"""C4: an SQP-like sequence of K QPs at C3 size (BASELINE.json configs[3]): rank-2 BFGS updates
of the resident H (ipm_update_hessian_rank2), a new linear term, and a warm start (R15) before
every solve; aggregated QP time excludes the Hessian updates, as the paper measures.
Every QP gets the next planted sub-problem of gen/sqp_sequence.py (x* random walk with 5 % active-set
flips: new g, new row bounds through ipm_set_bounds).  Each QP's record is flushed as it completes.
Usage: python scripts/c4_sequence.py [K=30] [--cold] [--n N --m M] [--out FILE]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from gen.planted import config
from gen.sqp_sequence import sqp_sequence
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP

ap = argparse.ArgumentParser()
ap.add_argument("K", type=int, nargs="?", default=30)
ap.add_argument("--cold", action="store_true")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--m", type=int, default=None)
ap.add_argument("--out", default=None)
a = ap.parse_args()
kw = {}
if a.n:
    kw["n"] = a.n
if a.m is not None:
    kw["m"] = a.m
q = config("C3", 0, **kw)
ups = sqp_sequence(q, a.K, seed=0)
dev = torch.device("cuda", 0)
qp = QP(device=dev, **problem_tensors(q, dev))
tot_ms, rows = 0.0, []
for k in range(a.K):
    if k > 0:
        up = ups[k - 1]
        qp.update_hessian_rank2(up.u, up.alpha, up.v, up.beta)
        qp.set_linear_term(up.g)
        qp.set_bounds(up.l, up.ub, q.xl, q.xu)
        if not a.cold:
            qp.warm_start()
    st = qp.solve()
    s = qp.stats()
    tot_ms += s["t_solve_ms"]
    fstar = q.f_star if k == 0 else ups[k - 1].f_star
    xstar = q.x_star if k == 0 else ups[k - 1].x_star
    x = qp.solution()["x"].cpu().numpy()
    rec = {"qp": k, "status": st, "t_solve_s": s["t_solve_ms"] / 1e3, "ipm": s["ipm_iters"],
           "pcg": s["pcg_iters_total"], "obj": s["obj"], "rel_err_f_planted": abs(s["obj"] - fstar) / abs(fstar),
           "max_err_x_planted": float(abs(x - xstar).max())}
    rows.append(rec)
    print(json.dumps(rec), flush=True)
    if a.out:
        with open(a.out, "a") as fo:
            fo.write(json.dumps(rec) + "\n")
print(json.dumps({"summary": "C4", "K": a.K, "mode": "cold" if a.cold else "warm", "n": q.n, "m": q.m,
                  "aggregate_qp_time_s": tot_ms / 1e3, "mean_qp_time_s": tot_ms / 1e3 / a.K,
                  "ipm_total": sum(r["ipm"] for r in rows), "pcg_total": sum(r["pcg"] for r in rows)}), flush=True)
