"""Closed-loop SQP on a paper-shaped dose NLP; prints one JSON line per SQP
iteration and a summary (aggregate QP time = the paper's Fig. 3 quantity).
Usage: python scripts/sqp_run.py S-proton|S-vmat|S-c4 [--iters K] [--hess 0|1] [--warm]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from gen.dose_nlp import nlp_config
from paper_2405_03584_b200 import SQP

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--iters", type=int, default=None)
ap.add_argument("--hess", type=int, default=None)
ap.add_argument("--warm", action="store_true")
ap.add_argument("--tol", type=float, default=1e-6)
a = ap.parse_args()
defaults = {"S-proton": (100, 1), "S-vmat": (33, 1), "S-c4": (30, 0), "S1": (50, 1)}
K, hk = defaults[a.config]
K = a.iters or K
hk = hk if a.hess is None else a.hess
t0 = time.time()
q = nlp_config(a.config, 0)
tgen = time.time() - t0
dev = torch.device("cuda", 0)
t0 = time.time()
s = SQP.from_nlp(q, device=dev, hess_kind=hk, max_iter=K, max_cols=2 * K, warm_start=int(a.warm), tol_d=a.tol)
torch.cuda.synchronize()
tcreate = time.time() - t0
t0 = time.time()
st = s.solve(q.x0)
wall = time.time() - t0
for r in s.trace():
    print(json.dumps(r), flush=True)
S = s.stats()
print(json.dumps({"summary": a.config, "n": q.n, "m": q.m, "nd": q.nd, "D_nnz": q.D_nnz, "hess_kind": hk,
                  "warm": a.warm, "status": st, "sqp_iters": S["iters"], "f": S["f"],
                  "aggregate_qp_time_s": S["t_qp_ms"] / 1e3, "sqp_device_time_s": S["t_total_ms"] / 1e3,
                  "wall_s": wall, "ipm_iters_total": S["ipm_iters_total"], "pcg_iters_total": S["pcg_iters_total"],
                  "backtracks": S["backtracks"], "updates_skipped": S["updates_skipped"],
                  "gen_s": tgen, "create_s": tcreate, "kernel_launches": s.kernel_launches()}), flush=True)
