"""Run the CPU oracle (oracle/ only) to completion on a bench workload and store its IPM
iteration count and objective in tests/golden/oracle_counts.json.

bench.py's reference / cpu_baseline legs time a BOUNDED sample (one IPM iteration) of
the oracle and scale it to a QP solve time with this stored count.  The GPU parity
tests also compare the GPU's IPM iteration count against it (north_star: +-2).
Usage: python scripts/oracle_reference_counts.py C3 [seed]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from gen.planted import config  # noqa: E402
from oracle.ipm import Options, Problem, solve  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
q = config(name, seed)
p = Problem.from_data(q)
t0 = time.time()
res = solve(p, Options())
dt = time.time() - t0
path = os.path.join(ROOT, "tests", "golden", "oracle_counts.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[f"{name}/seed{seed}"] = {
    "status": res.status, "ipm_iters": res.iters, "obj": res.obj, "f_star_planted": q.f_star,
    "x_err_vs_planted": float(abs(res.x - q.x_star).max()), "seconds": round(dt, 1),
    "cores": os.cpu_count(), "written_by": "scripts/oracle_reference_counts.py (oracle/ only)",
}
json.dump(data, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps(data[f"{name}/seed{seed}"]))
