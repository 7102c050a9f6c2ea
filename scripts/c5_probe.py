"""C5 on ONE B200 (the largest single-GPU case of BASELINE.json: n = 100000, H = 80 GB fp64,
m = 20000, nnz = 2e7): builds H on the device from its exact factors, creates the context,
checks sampled operator rows against host values computed one by one, and times the PCG GEMV
variants and one PCG iteration with CUDA events (ipm_profile).  A full C5 QP solve (hundreds of
thousands of PCG iterations) is out of a bench step's budget; this probe measures the kernels.
Prints one JSON line per measurement."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from gen.planted import config, hessian_rows
from gen.torch_io import device_hessian, problem_tensors
from paper_2405_03584_b200 import QP

dev = torch.device("cuda", 0)
t0 = time.time()
q = config("C5", 0)
print(json.dumps({"stage": "generated", "s": round(time.time() - t0, 1), "nnz": q.nnz}), flush=True)
H, ldh = device_hessian(q, dev)
t = problem_tensors(q, dev, H=H, ldh=ldh)
torch.cuda.synchronize()
print(json.dumps({"stage": "H on device", "s": round(time.time() - t0, 1), "H_GB": H.numel() * 8 / 1e9}), flush=True)
n = q.n
rng = np.random.default_rng(5)
sb = rng.uniform(0.0, 3.0, n)
sc = 10.0 ** rng.uniform(-3, 3, q.m)
v = rng.normal(size=n)
A = q.A_scipy()
ATt = A.T @ (sc * (A @ v))
rows = np.sort(rng.choice(n, size=16, replace=False))
for gk in [int(a) for a in sys.argv[1:]] or [3, 2]:
    qp = QP(device=dev, gemv_kernel=gk, **t)
    y = qp.op_apply(sb, sc, v).cpu().numpy()
    err = 0.0
    for i in rows:
        Hi = hessian_rows(q.d, q.U, q.w, int(i), int(i) + 1)[0]
        ref = float(np.concatenate([Hi * v, [sb[i] * v[i], ATt[i]]]).astype(np.longdouble).sum())
        scale = float(np.abs(Hi * v).sum() + abs(sb[i] * v[i]) + abs(ATt[i]))
        err = max(err, abs(y[i] - ref) / scale)
    gemv = qp.profile("gemv", 5)
    it = qp.profile("pcg_iter", 5)
    info = qp.info()
    if info["gemv_kernel"] == 3:
        nb = (n + 255) // 256          # info["ncb"] also counts the carry slots
        sizes = [min(256, n - i * 256) for i in range(nb)]
        streamed = 8.0 * sum(sizes[i] * sizes[j] for i in range(nb) for j in range(i, nb))
    else:
        streamed = 8.0 * n * n
    print(json.dumps({"workload": "C5", "gemv_kernel": info["gemv_kernel"], "sampled_rel_err": err,
                      "gemv_ms": gemv, "pcg_iter_ms": it, "streamed_GBps": streamed / gemv / 1e6,
                      "dense_equivalent_GBps": 8.0 * n * n / gemv / 1e6}), flush=True)
    qp.close()
