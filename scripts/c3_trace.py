"""One C3 solve with the per-IPM-iteration trace: PCG iterations, restarts and relative
residuals per IPM iteration (where the PCG count comes from)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP
q = config(sys.argv[1] if len(sys.argv) > 1 else "C3", 0)
qp = QP(device="cuda:0", trace=1, **problem_tensors(q, torch.device("cuda", 0)))
qp.solve()
print(json.dumps(qp.stats()))
for r in qp.trace():
    print(json.dumps(r))
