"""Bounded GPU diagnostic: create + solve C1 with the host-loop PCG and the graph PCG."""
import faulthandler, os, sys, time
faulthandler.dump_traceback_later(100, exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("IPM_DEBUG", "1")
import torch
print("torch", torch.__version__, torch.cuda.get_device_name(0), flush=True)
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP
q = config("C1", 0)
t = problem_tensors(q, torch.device("cuda", 0))
for ug in [int(a) for a in sys.argv[1:]] or [0, 1]:
    t0 = time.time()
    qp = QP(device="cuda:0", use_graph=ug, **t)
    print("created", ug, time.time() - t0, flush=True)
    print("status", qp.solve(), qp.stats(), time.time() - t0, flush=True)
