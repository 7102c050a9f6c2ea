"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck): C1 (single-CTA PCG
k_pcg_small), a 3000-variable VMAT-shaped QP (SYMV mbarrier ring + named barrier, SpMV side
branch, cooperative fused update with its grid barrier, graph WHILE loop), and optionally the
same QP row-sharded over 2 in-process ranks (peer data plane).
  compute-sanitizer --tool racecheck python scripts/sanitize_run.py [--case solve|c1|c1pcg|opapply|pcgiter|sharded]
(C1 solves now run the whole IPM loop in one warp, k_ipm_tiny; c1pcg = the one-warp PCG hooks)"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen.planted import config, planted_qp  # noqa: E402
from gen.torch_io import problem_tensors  # noqa: E402
from paper_2405_03584_b200 import QP  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="solve")
ap.add_argument("--nograph", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
q3 = planted_qp(3000, 1500, density=0.02, rank=64, seed=2, rows="vmat", var="box")
rng = np.random.default_rng(0)
G = dict(use_graph=0) if a.nograph else {}
if a.case in ("solve", "c1"):
    for name, q in (("C1", config("C1", 0)), ("vmat3000", q3))[:1 if a.case == "c1" else 2]:
        qp = QP(device=dev, max_ipm_iter=3, **G, **problem_tensors(q, dev))
        st = qp.solve()
        s = qp.stats()
        print(name, st, s["ipm_iters"], s["pcg_iters_total"], flush=True)
        qp.close()
elif a.case in ("opapply", "pcgiter"):
    qp = QP(device=dev, use_graph=0 if a.nograph else 1, **problem_tensors(q3, dev))
    sb, sc, v = rng.uniform(0, 3, q3.n), 10.0 ** rng.uniform(-2, 2, q3.m), rng.normal(size=q3.n)
    if a.case == "opapply":
        print("opapply", float(qp.op_apply(sb, sc, v).sum()), flush=True)
    else:
        print("pcgiter", qp.pcg_iterate(sb, sc, v, 3)["rho"], flush=True)
elif a.case == "c1pcg":                            # one-warp PCG on the assembled K (k_form_K + k_pcg_warp)
    q = config("C1", 0)
    qp = QP(device=dev, **problem_tensors(q, dev))
    sb, sc, v = rng.uniform(0, 3, q.n), 10.0 ** rng.uniform(-2, 2, q.m), rng.normal(size=q.n)
    print("c1pcg", qp.pcg_iterate(sb, sc, v, 5)["rho"], flush=True)
    x, it = qp.pcg(sb, sc, v, 1e-10)
    print("c1pcg solve", it, flush=True)
elif a.case == "sharded":
    from paper_2405_03584_b200.dist import LocalGroup, partition
    q = planted_qp(1000, 300, density=0.02, rank=32, seed=43, rows="vmat", var="box")
    t = problem_tensors(q, dev, H=torch.from_numpy(np.ascontiguousarray(q.H)).to(dev), ldh=q.n)   # no cuBLAS
    grp = LocalGroup(2)
    fns = []
    for r, (b, e) in enumerate(partition(q.n, 2)):
        tr = dict(t)
        tr["H"] = t["H"][b:e].contiguous()
        fns.append(lambda r=r, tr=tr: QP(device=dev, stream=torch.cuda.Stream(dev), shard=grp.shard(r), max_ipm_iter=2,
                                         **G, **tr))
    qps = grp.run(fns)
    print("sharded", grp.run([qq.solve for qq in qps]), flush=True)
