"""Experiment: keep a share of H's upper block triangle L2-resident (evict_last TMA policy on
the leading tiles of each CTA's range, IPM_SYM_KEEP_MB) and time the PCG SYMV on C3."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP
q = config(sys.argv[1] if len(sys.argv) > 1 else "C3", 0)
t = problem_tensors(q, torch.device("cuda", 0))
for mb in [0, 16, 32, 48, 64, 80, 96, 112]:
    os.environ["IPM_SYM_KEEP_MB"] = str(mb)
    qp = QP(device="cuda:0", max_ipm_iter=1, pcg_max_iter=20, **t)
    qp.solve()
    g = qp.profile("gemv", 30)
    it = qp.profile("pcg_iter", 30)
    print(json.dumps({"keep_mb": mb, "gemv_ms": g, "pcg_iter_ms": it}), flush=True)
    qp.close()
