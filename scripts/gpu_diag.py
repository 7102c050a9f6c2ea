"""Bounded GPU diagnostic: stage by stage on C1 (IPM_DEBUG=2 syncs after every stage)."""
import faulthandler, os, sys, time
faulthandler.dump_traceback_later(40, exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("IPM_DEBUG", "2")
import numpy as np
import torch
print("torch", torch.__version__, torch.cuda.get_device_name(0), flush=True)
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP
q = config("C1", 0)
t = problem_tensors(q, torch.device("cuda", 0))
ug = int(sys.argv[1]) if len(sys.argv) > 1 else 0
gk = int(sys.argv[2]) if len(sys.argv) > 2 else 1
qp = QP(device="cuda:0", use_graph=ug, gemv_kernel=gk, **t)
print("created", flush=True)
sb = np.ones(q.n); sc = np.ones(q.m); v = np.ones(q.n)
y = qp.op_apply(sb, sc, v); torch.cuda.synchronize(); print("op_apply ok", float(y.sum()), flush=True)
x, it = qp.pcg(sb, sc, v, 1e-10); print("pcg ok", it, flush=True)
print("status", qp.solve(), qp.stats(), flush=True)
