"""Time the PCG GEMV and one full PCG iteration (stream-launched) on a workload; used to compare
update-kernel group sizes (IPM_UPD_G) and L2 residency settings across processes."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen.planted import config
from gen.torch_io import problem_tensors
from paper_2405_03584_b200 import QP
wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
torch.cuda.init()
if os.environ.get("PERSIST_MB"):
    import glob
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
    rt = ctypes.CDLL(cands[0])
    rc = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(int(float(os.environ["PERSIST_MB"]) * 1048576)))
    print("persist limit rc", rc, file=sys.stderr)
q = config(wl, 0)
t = problem_tensors(q, torch.device("cuda", 0))
qp = QP(device="cuda:0", max_ipm_iter=1, pcg_max_iter=20, **t)
qp.solve()
res = {"workload": wl, "upd_g": os.environ.get("IPM_UPD_G"), "unroll": os.environ.get("IPM_UNROLL"), "keep_mb": os.environ.get("IPM_SYM_KEEP_MB"),
       "persist_mb": os.environ.get("PERSIST_MB"), "gemv_ms": qp.profile("gemv", 30),
       "spmv_ms": qp.profile("spmv", 30) if q.m else None, "pcg_iter_ms": qp.profile("pcg_iter", 30)}
qg = QP(device="cuda:0", max_ipm_iter=1, pcg_max_iter=300, **t)   # captured-graph PCG iterations
qg.solve()
qg.solve()
sg = qg.stats()
res["graph_pcg_iter_ms"] = sg["t_pcg_ms"] / max(1, sg["pcg_iters_total"])
qg.close()
if os.environ.get("PROBE_QP", "1") == "0":
    print(json.dumps(res), flush=True)
    sys.exit(0)
qp2 = QP(device="cuda:0", **t)
qp2.solve()
ts = []
for _ in range(3):
    qp2.solve()
    ts.append(qp2.stats()["t_solve_ms"])
kt = qp2.kernel_timer()
res["qp_ms"] = sorted(ts)[1]
res["pcg_iters"] = qp2.stats()["pcg_iters_total"]
res["live_gemv_ms"] = kt[0] / max(1, kt[1])
print(json.dumps(res), flush=True)
