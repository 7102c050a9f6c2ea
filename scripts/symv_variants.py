"""Experiment: time the PCG SYMV / PCG iteration of diagnostic builds of libipm (build.py
--variant=...) on a workload, one child process per variant (IPM_LIB selects the build).
  python scripts/symv_variants.py C5 "" nc nocol env:IPM_SYMV_LDG=1 ...
("" = the production build; env:K=V,... = the production build with environment switches)
Prints one JSON line per variant."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys
sys.path.insert(0, ROOT)
import torch
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP
wl, var = sys.argv[1], sys.argv[2]
q = config(wl, 0)
t = problem_tensors(q, torch.device("cuda", 0))
qp = QP(device="cuda:0", max_ipm_iter=1, pcg_max_iter=3, **t)
qp.solve(raise_on_error=False)
n = q.n
nb = (n + 255) // 256
sizes = [min(256, n - i * 256) for i in range(nb)]
streamed = 8.0 * sum(sizes[i] * sizes[j] for i in range(nb) for j in range(i, nb))
import hashlib, numpy as np
rng = np.random.default_rng(1)
y = qp.op_apply(rng.uniform(0, 3, n), 10.0 ** rng.uniform(-2, 2, q.m), rng.normal(size=n)).cpu().numpy()
digest = hashlib.sha1(y.tobytes()).hexdigest()[:12]
np.save("/tmp/symv_y_" + (var or "prod").replace(":", "_").replace("=", "_").replace(",", "_") + ".npy", y)
reps = 5 if n > 50000 else 20
g = qp.profile("gemv", reps)
sp = qp.profile("spmv", reps)
it = qp.profile("pcg_iter", reps)
print(json.dumps({"variant": var or "prod", "workload": wl, "gemv_ms": g, "spmv_ms": sp, "pcg_iter_ms": it,
                  "streamed_GBps": streamed / g / 1e6, "y_sha1": digest}), flush=True)
'''.replace("ROOT", repr(ROOT))

wl = sys.argv[1]
for var in sys.argv[2:]:
    env = dict(os.environ)
    if var.startswith("env:"):                      # production build with environment switches
        for kv in var[4:].split(","):
            k, v = kv.split("=")
            env[k] = v
    elif var:
        subprocess.run([sys.executable, os.path.join(ROOT, "paper_2405_03584_b200", "build.py"), f"--variant={var}"],
                       check=True, capture_output=True)
        env["IPM_LIB"] = os.path.join(ROOT, "paper_2405_03584_b200", f"libipm_{var}.so")
    r = subprocess.run([sys.executable, "-c", CHILD, wl, var], env=env, capture_output=True, text=True)
    line = r.stdout.strip()
    if line.startswith("{"):
        import numpy as np
        d = json.loads(line)
        ref = "/tmp/symv_y_prod.npy"
        if var and os.path.exists(ref):
            y0, y1 = np.load(ref), np.load("/tmp/symv_y_" + var.replace(":", "_").replace("=", "_").replace(",", "_") + ".npy")
            d["max_rel_diff_vs_prod"] = float(np.max(np.abs(y1 - y0)) / np.max(np.abs(y0)))
        line = json.dumps(d)
    print(line or r.stderr[-1500:], flush=True)
