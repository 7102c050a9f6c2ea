#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric) — one JSON line on rank 0.

Workload (default): C5, the largest single-GPU configuration of BASELINE.json (n = 100000,
m = 20000, 1 % dense A, dense fp64 H = 80 GB), on which north_star states the roofline target.

A *step* is one pass of the whole hot path over the workload: ONE iteration of Algorithm 1
 from the cold start, i.e. `ipm_solve` with max_ipm_iter = 1 — initial point and
mu0 (a1), residuals (a2), the KKT norm / objective (a3), Sigma_b, Sigma_c and the Jacobi
diagonal (a4), the condensed right-hand side (a5), the PCG solve of K dx = rhs to its D6
tolerance (a6: SYMV + SpMV + SpMV^T + fused update per PCG iteration), the recovery of the full
step (a8), the fraction-to-boundary step lengths (a9) and the update (a10), then the final
residuals.  Every step does identical work (same start, deterministic kernels), so a whole
QP (≈10^5-10^6 PCG iterations at C5, hours) is not the timing unit — SURVEY §8(d), VERDICT r1.

  value = PCG iterations per second over the whole job (all ranks), inputs resident in HBM
  (the PCG is >90 % of QP runtime; QP time = PCG iterations / value).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5] [--impl ours|reference]

N > 1: C5 is row-sharded over the N GPUs (ONE QP, NCCL allgathers inside libipm, "strong");
C1-C3 run as N replicas (rank r solves seed + r, no collective, "weak").  --impl reference
times the CPU oracle (oracle/) as it stands on the host cores on a bounded sample of the same
workload (see OracleSample).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QP solve time (s) & PCG it/s at 1/2/4/8 B200; op-apply HBM GB/s vs peak"
UNIT = "PCG it/s"
STEP = ("one Algorithm-1 IPM iteration from the cold start (ipm_solve, max_ipm_iter = 1): initial point, "
        "residuals, Sigma/Jacobi, condensed RHS, PCG to the D6 tolerance, recovery, step lengths, update")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _l2_note(n: int) -> str:
    """How the timed steps relate to the 126 MB L2 (no flush between steps in any case)."""
    tri = 4.0 * n * (n + 256)          # upper block triangle incl. diagonal blocks (kSymB = 256)
    if 8 * n * n > 400e6:
        return f"inputs larger than L2 (H {8 * n * n / 1e9:.1f} GB >> 126 MB), no flush"
    if tri <= 100 * 1048576:           # libipm's evict_last threshold (ipm_api.cu, sym_keep)
        return (f"H {8 * n * n / 1e6:.3g} MB; its {tri / 1e6:.3g} MB upper triangle is L2-resident across PCG "
                "iterations by design (evict_last, IPM_SYM_KEEP_MB); no flush between steps")
    return f"H {8 * n * n / 1e6:.3g} MB vs 126 MB L2, no flush"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cores():
    return int(os.environ.get("OPENBLAS_NUM_THREADS", "0")) or os.cpu_count()


# ----------------------------------------------------------------------------- oracle
class OracleSample:
    """A bounded sample of one PCG iteration of the workload, computed by the CPU oracle as it
    stands: ``oracle.kkt.condensed_apply_rows`` — K v from its definition,
    t = Sigma_c o (A v), A^T t over the full A, and the H part for a slab of R rows of the
    workload's H (built on the host from the generator's exact factors).  One PCG iteration is
    one K apply plus O(n) vector work (H is 99.8 % of its bytes at C5), so
        seconds per PCG iteration ~= t(A part) + (n / R) * t(H slab)
    with both terms timed separately (the A part via an empty row set)."""

    def __init__(self, workload: str, seed: int, rows: int = 2048):
        import numpy as np
        from gen.planted import config, hessian_rows
        self.q = q = config(workload, seed)
        self.n = q.n
        self.R = min(rows, q.n)
        rng = np.random.default_rng(seed + 7)
        self.v = rng.normal(size=q.n)
        self.sig_b = rng.uniform(0.0, 3.0, q.n)
        self.sig_c = 10.0 ** rng.uniform(-3, 3, q.m)
        self.A = q.A_scipy()
        r0 = (q.n - self.R) // 2
        self.rows = np.arange(r0, r0 + self.R)
        self.H_rows = hessian_rows(q.d, q.U, q.w, r0, r0 + self.R)
        self.H_none = self.H_rows[:0]

    def _apply(self, H_rows, rows):
        from oracle.kkt import condensed_apply_rows
        t0 = time.perf_counter()
        condensed_apply_rows(H_rows, rows, self.A, self.sig_b, self.sig_c, self.v)
        return time.perf_counter() - t0

    def step(self):
        """One timed sample: (seconds measured, extrapolated seconds per PCG iteration)."""
        ta = self._apply(self.H_none, self.rows[:0])
        ts = self._apply(self.H_rows, self.rows)
        th = max(ts - ta, 0.0)
        return ta + ts, ta + th * self.n / self.R

    def describe(self, reps):
        return (f"oracle.kkt.condensed_apply_rows (numpy/scipy, fp64) on the {self.q.n}-variable workload: "
                f"full A / A^T part + an {self.R}-row slab of H ({8 * self.R * self.q.n / 1e9:.2f} GB), "
                f"median of {reps}; per PCG iteration = t_A + (n/R) t_Hslab (one K apply; vector work O(n) "
                f"neglected); OPENBLAS threads = {_cores()}")


def run_reference(args):
    """The reference arm of this tier: the CPU oracle, as it stands, on the host cores."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    t_setup = time.perf_counter()
    smp = OracleSample(args.workload, args.seed)
    t_setup = time.perf_counter() - t_setup
    for _ in range(args.warmup):          # untimed warm-up samples (page-in, BLAS thread pools)
        smp.step()
    meas, per_it = [], []
    for _ in range(args.steps):
        a, b = smp.step()
        meas.append(a)
        per_it.append(b)
    t_it = statistics.median(per_it)
    value = 1.0 / t_it
    sample = smp.describe(len(per_it))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.mean(meas) * 1e3,          # the unit actually timed (one sample)
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic planted-KKT QP (gen/planted.py, seeded)",
            "config": {"workload": args.workload, "seed": args.seed},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": _cores(), "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "extrapolated_ms_per_pcg_iter": t_it * 1e3, "setup_s": t_setup}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- ours
def _algorithmic_gemv_bytes(qp, info, n, rows, sharded, ws, rank):
    """Bytes one launch of the PCG operator kernel must move."""
    ncb = info["ncb"]
    nrow = rows[1] - rows[0]
    if info["gemv_kernel"] == 3:
        import ctypes as C
        from paper_2405_03584_b200 import _lib
        nt = C.c_int32()
        P, r = (ws, rank) if sharded else (1, 0)
        _lib.ipm_sym_plan(n, P, r, 148, None, 0, C.byref(nt), None, None, None)
        tl = (C.c_int32 * (8 * nt.value))()
        _lib.ipm_sym_plan(n, P, r, 148, tl, nt.value, C.byref(nt), None, None, None)
        elems = sum(tl[8 * t + 1] * tl[8 * t + 3] for t in range(nt.value))
        slots = (n + 255) // 256              # every (row, block) slot of ypart is written once
        return (8.0 * elems + 8.0 * n + 8.0 * nrow * slots,
                "k_symv_bulk<1> (symmetric upper-triangle GEMV, 2-D TMA, p^T (H + Sigma_b) p fused)")
    name = ("k_gemv_bulk<1> (TMA-bulk GEMV, p^T H p fused)" if info["gemv_kernel"] == 2
            else "k_gemv_tiles<1,1> (LDG.128 GEMV, p^T H p fused)")
    return 8.0 * nrow * n + 8.0 * n + 8.0 * nrow * ncb, name


def _traffic(workload, kernel):
    tp = os.path.join(ROOT, "profiles", "gemv_traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp)).get(f"{workload}/gemv_kernel{kernel}")
        if tj:
            return tj.get("dram_bytes_per_launch"), tj.get("source")
    return None, None


def _qp_context(wl, seed, dev):
    """Median QP time-to-solution of a smaller BASELINE config (context keys, 1 GPU)."""
    import torch
    from gen.planted import config
    from gen.torch_io import problem_tensors
    from paper_2405_03584_b200 import QP
    qo = config(wl, seed)
    qx = QP(device=dev, **problem_tensors(qo, dev))
    reps = {"C1": 5, "C2": 3}.get(wl, 1)
    if wl in ("C1", "C2"):
        qx.solve()
    ts = []
    for _ in range(reps):
        qx.solve()
        ts.append(qx.stats())
    ts.sort(key=lambda s: s["t_solve_ms"])
    med = ts[len(ts) // 2]
    out = {"qp_solve_s": med["t_solve_ms"] / 1e3, "ipm_iters": med["ipm_iters"], "pcg_iters": med["pcg_iters_total"],
           "pcg_it_per_s": med["pcg_iters_total"] / (med["t_solve_ms"] * 1e-3), "status": med["status"],
           "solves": reps, "gemv_kernel": qx.info()["gemv_kernel"]}
    qx.close()
    del qx
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from gen.planted import CONFIGS, config
    from gen.torch_io import device_hessian, problem_tensors
    from paper_2405_03584_b200 import QP

    ws, rank, local = _dist()
    if args.same_gpu:       # testing the N > 1 paths on one GPU: every rank on cuda:0, gloo bootstrap
        local = 0
    if ws > 1:
        dist.init_process_group("gloo" if args.same_gpu else "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rdev = torch.device("cpu") if args.same_gpu else dev    # device of the cross-rank reductions
    # C5 at N > 1 (or --shard): ONE QP row-sharded over the ranks (NCCL allgathers inside libipm,
    # SURVEY §8(e)), each rank building only its row block of H on its device; otherwise every
    # rank solves its own QP (seed + rank): replicas, no collective on the data path.
    sharded = (ws > 1 and args.workload == "C5") or args.force_shard
    seed = args.seed if sharded else args.seed + rank
    t_gen = time.perf_counter()
    q = config(args.workload, seed)
    n, m, nnz = q.n, q.m, q.nnz
    opts = dict(max_ipm_iter=1, kernel_timer=1)
    if args.host_loop:
        opts["use_graph"] = 0
    rows = (0, n)
    uid_holder = {}
    if sharded:
        from paper_2405_03584_b200.dist import broadcast_unique_id, nccl_shard, nccl_unique_id, partition
        rows = partition(n, ws)[rank]

        def shard():
            if args.same_gpu and ws > 1:
                # processes sharing one GPU cannot form an NCCL communicator: bootstrap the peer
                # data plane over the gloo group instead (comm_kind 3, CUDA IPC between processes)
                from paper_2405_03584_b200.dist import host_shard, torch_allgather_bytes
                uid_holder["s"] = host_shard(rank, ws, torch_allgather_bytes())
                return uid_holder["s"]
            uid = (nccl_unique_id() if ws == 1
                   else broadcast_unique_id(nccl_unique_id, rank, dist.broadcast_object_list))
            uid_holder["s"] = nccl_shard(rank, ws, uid)
            return uid_holder["s"]
    else:
        def shard():
            return None
    Hb, ldh = device_hessian(q, dev, rows=rows)
    t = problem_tensors(q, dev, H=Hb, ldh=ldh)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    t_create = time.perf_counter()
    qp = QP(device=dev, shard=shard(), **opts, **t)
    torch.cuda.synchronize()
    t_create = time.perf_counter() - t_create
    stream = qp.stream

    def barrier():
        if ws > 1:
            dist.barrier()

    for _ in range(args.warmup):
        qp.solve()
    warm_stats = qp.stats()
    barrier()
    clocks = Clocks(local)
    clocks.start()
    stats = []
    launches0 = qp.kernel_launches()
    kt0 = qp.kernel_timer()
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        qp.solve()
        stats.append(qp.stats())
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = qp.kernel_launches() - launches0
    kt1 = qp.kernel_timer()
    kt_ms, kt_n = kt1[0] - kt0[0], kt1[1] - kt0[1]
    t_s = e0.elapsed_time(e1) / 1e3
    pcg_local = sum(s["pcg_iters_total"] for s in stats)
    tt = torch.tensor([t_s], dtype=torch.float64, device=rdev)
    pc = torch.tensor([float(pcg_local)], dtype=torch.float64, device=rdev)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        if not sharded:
            dist.all_reduce(pc, op=dist.ReduceOp.SUM)   # replicas: every rank's PCG iterations count
    t_max = float(tt.item())
    pcg_job = float(pc.item())
    pcg_ms = sum(s["t_pcg_ms"] for s in stats)
    statuses = sorted(set(s["status"] for s in stats))
    pcg_per_step = sorted(set(s["pcg_iters_total"] for s in stats))

    # --- roofline of the dominant kernel (the PCG SYMV / GEMV), timed live on the library stream
    info = qp.info()
    gemv_bytes, kname = _algorithmic_gemv_bytes(qp, info, n, rows, sharded, ws, rank)
    gemv_iso_ms = qp.profile("gemv", reps=5 if n >= 50000 else (10 if n >= 10000 else 50))
    gemv_ms = kt_ms / kt_n if kt_n > 0 else gemv_iso_ms
    peak, peak_src = _peaks()
    achieved = gemv_bytes / (gemv_ms * 1e-3) / 1e9
    traffic, traffic_src = _traffic(args.workload, info["gemv_kernel"])
    if traffic is not None and sharded and ws > 1:
        traffic = None                                   # the committed capture is the P = 1 launch
    qp_stats_last = stats[-1] if stats else warm_stats

    # --- end to end through the public API with HOST buffers --------------------------------
    # The same job from pinned host memory: upload of every problem array (H2D, inside the timed
    # region), ipm_create, then per step the new linear term g from the host (the input an SQP
    # caller supplies per QP) and the step's result x read back to the host.
    Hh = torch.empty((rows[1] - rows[0], ldh), dtype=torch.float64, pin_memory=True)
    Hh.copy_(Hb)
    th = problem_tensors(q, dev, H=Hh, ldh=ldh, host=True)
    g_host = th["g"]
    x_host = torch.empty(rows[1] - rows[0], dtype=torch.float64, pin_memory=True)
    qp.close()
    del qp, t, Hb
    torch.cuda.empty_cache()
    h2d_once = sum(v.numel() * v.element_size() for k, v in th.items() if hasattr(v, "numel"))
    barrier()
    torch.cuda.synchronize()
    a0 = time.perf_counter()
    qp2 = QP(device=dev, shard=shard(), **opts, **th)
    e2e_pcg = 0
    for _ in range(args.steps):
        qp2.set_linear_term(g_host)
        qp2.solve()
        x_host.copy_(qp2.solution()["x"])
        e2e_pcg += qp2.stats()["pcg_iters_total"]
    torch.cuda.synchronize()
    e2e_t = time.perf_counter() - a0
    qp2.close()
    del qp2
    te = torch.tensor([e2e_t], dtype=torch.float64, device=rdev)
    pe = torch.tensor([float(e2e_pcg)], dtype=torch.float64, device=rdev)
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        if not sharded:
            dist.all_reduce(pe, op=dist.ReduceOp.SUM)
    h2d_step = h2d_once / max(1, args.steps) + g_host.numel() * 8
    d2h_step = x_host.numel() * 8
    del Hh, th
    torch.cuda.empty_cache()

    # --- QP time-to-solution on the smaller BASELINE configs (context; 1 GPU) ---------------
    others = {}
    if ws == 1 and not args.no_extra:
        for wl in ("C1", "C2", "C3"):
            if wl != args.workload:
                others[wl] = _qp_context(wl, args.seed, dev)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        smp = OracleSample(args.workload, args.seed)
        smp.step()
        per = [smp.step()[1] for _ in range(3)]
        cpu = {"value": 1.0 / statistics.median(per), "unit": UNIT, "cores": _cores(), "kind": "oracle",
               "sample": smp.describe(len(per))}

    if rank == 0:
        units = "one QP row-sharded" if sharded else (f"{ws} replicas" if ws > 1 else "1 GPU")
        line = {
            "metric": METRIC, "value": pcg_job / t_max, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic planted-KKT QP (gen/planted.py, seeded; random-init dyadic H = diag + U W U^T)",
            "config": {"workload": args.workload, **CONFIGS[args.workload],
                       "seed": args.seed if (sharded or ws == 1) else f"{args.seed}..{args.seed + ws - 1} (one per rank)",
                       "nnz": nnz, "H_bytes": 8 * n * n, "l2": _l2_note(n), "step": STEP,
                       "parallelism": (f"row-sharded H over {ws} GPUs (NCCL allgather)" if sharded
                                       else (f"replicas x{ws}" if ws > 1 else "1 GPU"))},
            "pcg_iters_per_step": pcg_per_step, "pcg_iters_job": int(pcg_job), "job_units": units,
            "pcg_it_per_s_inside_pcg": pcg_local / (pcg_ms * 1e-3) if pcg_ms > 0 else None,
            "status": statuses, "kkt_inf_after_step": qp_stats_last["kkt_inf"],
            "setup_s": {"generate_and_H_on_device": t_gen, "ipm_create": t_create},
            "roofline": {"bound": "hbm", "kernel": kname,
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": gemv_bytes,
                         "dense_equivalent_GBps": 8.0 * (rows[1] - rows[0]) * n / (gemv_ms * 1e-3) / 1e9,
                         "launch_ms": gemv_ms, "launches_timed": int(kt_n), "peak_source": peak_src,
                         "share_of_step": kt_ms / (t_max * 1e3) if kt_n > 0 else None,
                         "isolated_launch_ms": gemv_iso_ms,
                         "timing": ("live: in-kernel %globaltimer (first CTA start to last CTA end) summed over "
                                    "every launch in the timed region, on the library stream (opt.kernel_timer)"
                                    if kt_n > 0 else "CUDA events, back-to-back launches after the timed region "
                                    "(small n: the timed PCG ran in the single-CTA k_pcg_small)")},
            "cpu_baseline": cpu,
            "e2e": {"value": float(pe.item()) / float(te.item()), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d_step), "d2h_bytes_per_step": int(d2h_step),
                    "how": (f"host-pinned inputs: H2D of every problem array ({h2d_once / 1e9:.2f} GB, once) + "
                            f"ipm_create + {args.steps} steps, each with g uploaded from the host "
                            "(ipm_set_linear_term) and x read back; wall clock")},
            "gpu_launches": int(launches), "clocks": clk, "other_workloads": others,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C5", choices=["C1", "C2", "C3", "C5"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", "--force-shard", dest="force_shard", action="store_true",
                    help="row-shard ONE QP over the N ranks (default only for C5 at N > 1) — also at N = 1 (NCCL path)")
    ap.add_argument("--no-extra", action="store_true", help="skip the C1/C2/C3 QP time-to-solution context")
    ap.add_argument("--same-gpu", action="store_true",
                    help="testing only: every rank on cuda:0 (gloo bootstrap, CUDA IPC data plane)")
    ap.add_argument("--host-loop", action="store_true",
                    help="profiling only: drive the PCG from the host (batches of 16) instead of the conditional-"
                         "WHILE graph, whose kernel nodes ncu cannot profile one by one")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
