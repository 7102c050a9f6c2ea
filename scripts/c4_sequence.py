"""C4: an SQP-like sequence of K QPs at C3 size (BASELINE.json configs[3]): rank-2 BFGS updates
of the resident H (ipm_update_hessian_rank2), a new linear term and new row bounds
(ipm_set_linear_term, ipm_set_bounds) and a warm start (R15) before every solve; aggregated QP
time excludes the Hessian updates, as the paper measures.  Every QP is the next planted
sub-problem of gen/sqp_sequence.py (x* random walk with 5 % active-set flips), so each solution
is checked against its exact optimum.

Each QP's record is appended to --out as it completes, and the solution that warm-starts the next
QP is checkpointed (--ckpt, npz), so a sequence longer than one GPU lease runs as several calls:
  python scripts/c4_sequence.py 30 --out r.jsonl --ckpt c.npz [--resume prev.npz] [--max-minutes 50]
--resume rebuilds H_k on the device by replaying the rank-2 updates 1..k (deterministic: the same
bits as the uninterrupted sequence) and warm-starts from the checkpointed solution.
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
from gen.sqp_sequence import sqp_sequence  # noqa: E402
from gen.torch_io import problem_tensors  # noqa: E402
from paper_2405_03584_b200 import QP  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("K", type=int, nargs="?", default=30)
ap.add_argument("--cold", action="store_true")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--m", type=int, default=None)
ap.add_argument("--out", default=None)
ap.add_argument("--ckpt", default=None)
ap.add_argument("--resume", default=None)
ap.add_argument("--max-minutes", type=float, default=1e9)
ap.add_argument("--stop-after", type=int, default=None, help="stop before QP k (resume testing)")
ap.add_argument("--warm-shift", type=float, default=None, help="R15 theta (ipm_options.warm_shift)")
a = ap.parse_args()
t_wall = time.time()
kw = {}
if a.n:
    kw["n"] = a.n
if a.m is not None:
    kw["m"] = a.m
q = config("C3", 0, **kw)
ups = sqp_sequence(q, a.K, seed=0)
dev = torch.device("cuda", 0)
qp = QP(device=dev, **problem_tensors(q, dev), **({"warm_shift": a.warm_shift} if a.warm_shift is not None else {}))
k0 = 0
if a.resume:
    ck = np.load(a.resume)
    k0 = int(ck["next_qp"])
    for up in ups[:k0 - 1]:                       # H_{k0-1}: replay the updates (same bits)
        qp.update_hessian_rank2(up.u, up.alpha, up.v, up.beta)
    fam = ("lA", "uA", "lx", "ux")
    qp.set_iterate(ck["x"], {f: ck["s_" + f] for f in fam}, {f: ck["lam_" + f] for f in fam}, float(ck["mu"]))


def emit(rec):
    print(json.dumps(rec), flush=True)
    if a.out:
        with open(a.out, "a") as fo:
            fo.write(json.dumps(rec) + "\n")


for k in range(k0, a.K):
    if time.time() - t_wall > a.max_minutes * 60 or (a.stop_after is not None and k >= a.stop_after):
        emit({"stop": "time_limit", "next_qp": k})
        break
    if k > 0:
        up = ups[k - 1]
        qp.update_hessian_rank2(up.u, up.alpha, up.v, up.beta)
        qp.set_linear_term(up.g)
        qp.set_bounds(up.l, up.ub, q.xl, q.xu)
        if not a.cold:
            qp.warm_start()
    st = qp.solve()
    s = qp.stats()
    fstar = q.f_star if k == 0 else ups[k - 1].f_star
    xstar = q.x_star if k == 0 else ups[k - 1].x_star
    x = qp.solution()["x"].cpu().numpy()
    emit({"qp": k, "mode": "cold" if a.cold else "warm", "theta": a.warm_shift, "status": st, "t_solve_s": s["t_solve_ms"] / 1e3,
          "ipm": s["ipm_iters"], "pcg": s["pcg_iters_total"], "obj": s["obj"],
          "rel_err_f_planted": abs(s["obj"] - fstar) / abs(fstar), "max_err_x_planted": float(abs(x - xstar).max())})
    if a.ckpt:
        xi, si, li, mu = qp.get_iterate()
        np.savez(a.ckpt, next_qp=k + 1, x=xi.cpu().numpy(), mu=mu,
                 **{"s_" + f: si[f].cpu().numpy() for f in si}, **{"lam_" + f: li[f].cpu().numpy() for f in li})
