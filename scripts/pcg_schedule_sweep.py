"""C3 (or other) solve with per-IPM-iteration trace under several PCG tolerance options."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP
wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
variants = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [{}]
q = config(wl, 0)
t = problem_tensors(q, torch.device("cuda", 0))
for v in variants:
    qp = QP(device="cuda:0", trace=1, **t, **v)
    t0 = time.time()
    st = qp.solve()
    s = qp.stats()
    x = qp.solution()["x"].cpu().numpy()
    err = float(abs(x - q.x_star).max() / abs(q.x_star).max())
    print(json.dumps({"variant": v, "status": st, "ipm": s["ipm_iters"], "pcg_total": s["pcg_iters_total"],
                      "restarts": s["pcg_restarts"], "stalls": s["pcg_stalls"], "t_s": time.time() - t0,
                      "xerr_planted": err, "obj_rel": abs(s["obj"] - q.f_star) / abs(q.f_star),
                      "trace": [(r["it"], r["pcg_iters"], round(r["mu"], 12), r["kkt_inf"], round(r["alpha_x"], 4),
                                 round(r["alpha_lam"], 4), r["pcg_relres"]) for r in qp.trace()]}), flush=True)
    qp.close()
