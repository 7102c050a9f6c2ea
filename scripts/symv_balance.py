"""Experiment: symmetric GEMV streaming rate vs tile balance (ntiles = nb(nb+1)/2 over 148 CTAs).
n = 28416 gives nb = 111, 6216 tiles = 42 per CTA exactly; others leave a partial last wave."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP
for n in [int(a) for a in sys.argv[1:]] or [20000, 28160, 28416, 18944, 19200]:
    q = config("C2", 0, n=n, rank=16)
    t = problem_tensors(q, torch.device("cuda", 0))
    qp = QP(device="cuda:0", max_ipm_iter=1, pcg_max_iter=5, **t)
    qp.solve()
    g = qp.profile("gemv", 20)
    nb = (n + 255) // 256
    sizes = [min(256, n - i * 256) for i in range(nb)]
    tri = sum(sizes[i] * sizes[j] for i in range(nb) for j in range(i, nb))
    print(json.dumps({"n": n, "nb": nb, "tiles": nb * (nb + 1) // 2, "tiles_per_cta": nb * (nb + 1) / 2 / 148,
                      "gemv_ms": g, "GBps": 8.0 * tri / g / 1e6}), flush=True)
    qp.close()
    del t, qp
    torch.cuda.empty_cache()
