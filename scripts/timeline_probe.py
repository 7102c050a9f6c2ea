"""Diagnostic: per-iteration kernel timeline of the captured PCG loop (libipm_tl.so, built with
`python paper_2405_03584_b200/build.py --timeline`).  Prints, relative to each iteration's SYMV
start (us): spmv [start, end], spmvT [start, end], symv end, update start, update barrier, and the
gap from the update barrier to the next iteration's SYMV start."""
import ctypes as C, json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("IPM_LIB", os.path.join(ROOT, "paper_2405_03584_b200", "libipm_tl.so"))
sys.path.insert(0, ROOT)
import torch
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP, _lib
wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
q = config(wl, 0)
t = problem_tensors(q, torch.device("cuda", 0))
qp = QP(device="cuda:0", max_ipm_iter=1, pcg_max_iter=60, **t)
qp.solve()
buf = (C.c_ulonglong * (64 * 16))()
_lib.lib.ipm_debug_timeline.argtypes = [C.c_void_p, C.c_void_p]
_lib.lib.ipm_debug_timeline(qp.ctx, buf)
recs = [[buf[i * 16 + k] for k in range(16)] for i in range(60)]
rows = []
for i in range(5, 58):
    r, nx = recs[i], recs[i + 1]
    s0 = r[4]
    rel = lambda v: (v - s0) / 1e3 if v else None  # noqa: E731
    rows.append({"spmv": [rel(r[0]), rel(r[1])], "spmvT": [rel(r[2]), rel(r[3])], "symv_end": rel(r[5]),
                 "upd_start": rel(r[6]), "upd_last_cta_start": rel(r[8]), "upd_rows_done": rel(r[9]),
                 "upd_last_arrival": rel(r[10]), "upd_barrier": rel(r[7]), "next_symv": rel(nx[4])})
for r in rows[:3]:
    print(json.dumps(r))
def med(f):
    v = [f(r) for r in rows if f(r) is not None]
    return statistics.median(v) if v else None
print(json.dumps({"workload": wl, "median_us": {
    "spmv_start": med(lambda r: r["spmv"][0]), "spmv_end": med(lambda r: r["spmv"][1]),
    "spmvT_start": med(lambda r: r["spmvT"][0]), "spmvT_end": med(lambda r: r["spmvT"][1]),
    "symv_end": med(lambda r: r["symv_end"]), "upd_start": med(lambda r: r["upd_start"]),
    "upd_last_cta_start": med(lambda r: r["upd_last_cta_start"]), "upd_rows_done": med(lambda r: r["upd_rows_done"]),
    "upd_last_arrival": med(lambda r: r["upd_last_arrival"]),
    "upd_barrier": med(lambda r: r["upd_barrier"]), "next_symv_start": med(lambda r: r["next_symv"])}}))
