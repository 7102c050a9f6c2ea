"""Short, bounded run of the hot path for ncu: one IPM iteration of WORKLOAD with the PCG
capped at PCG_ITERS iterations (steady-state kernel mix), then 3 isolated PCG GEMVs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP
wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 30
gk = int(sys.argv[3]) if len(sys.argv) > 3 else 0
q = config(wl, 0)
t = problem_tensors(q, torch.device("cuda", 0))
qp = QP(device="cuda:0", max_ipm_iter=1, pcg_max_iter=its, gemv_kernel=gk, use_graph=int(os.environ.get("USE_GRAPH", "0")), **t)
qp.solve()
print("gemv ms", qp.profile("gemv", 3), flush=True)
print(qp.stats(), flush=True)
