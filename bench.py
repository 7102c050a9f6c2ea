#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric) — one JSON line on rank 0.

A *step* is one full QP solve (Algorithm 1 to convergence, every §8(a) row: initial point,
residuals, diagonals + Jacobi, RHS, the PCG solve, recovery, step lengths, update) of the
workload, cold-started, with all inputs resident in HBM.  Default workload: C3, the
patient-case-shaped QP (n=20000, m=5000, 1% dense A, dense 3.2 GB H) — see DESIGN.md §7.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3] [--impl ours|reference]

value = QPs solved per second over the whole job (all ranks) = N*K / max-over-ranks time.
N > 1: a workload that fits one GPU (C1-C3) runs as N independent replicas —
rank r solves the QP of seed + r, no data-path collective ("scaling": "weak"); C5 (80 GB H) is
solved as ONE QP row-sharded over the N GPUs (NCCL allgathers inside libipm, "strong").
--shard forces the row-sharded path for any workload (and at N = 1).  --impl reference times
the CPU oracle (oracle/) as it stands on the host cores, on a bounded sample (one IPM iteration
per step) scaled to QP/s.
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
    tri_mb = tri / 1e6
    if 8 * n * n > 400e6:
        return f"inputs larger than L2 (H {8 * n * n / 1e9:.1f} GB >> 126 MB), no flush"
    if tri <= 100 * 1048576:           # libipm's evict_last threshold (ipm_api.cu, sym_keep)
        return (f"H {8 * n * n / 1e6:.3g} MB; its {tri_mb:.3g} MB upper triangle is L2-resident across PCG "
                "iterations by design (evict_last, IPM_SYM_KEEP_MB); no flush between steps")
    return f"H {8 * n * n / 1e6:.3g} MB vs 126 MB L2, no flush"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- oracle
def oracle_sample(workload: str, seed: int, iters: int = 1):
    """Time `iters` IPM iterations of the CPU oracle (as it stands) on the workload and
    return (seconds per IPM iteration, cores, description)."""
    import numpy as np  # noqa: F401
    from gen.planted import config
    from oracle.ipm import Options, Problem, initial_point, max_step, newton_direction, residuals
    q = config(workload, seed)
    p = Problem.from_data(q)
    opt = Options()
    it = initial_point(p, opt)
    r = residuals(p, it)
    t0 = time.perf_counter()
    for _ in range(iters):
        dx, ds, dl = newton_direction(p, it, r)
        ax = max_step(it.s, ds, opt.tau)
        al = max_step(it.lam, dl, opt.tau)
        it.x = it.x + ax * dx
        for f in ds:
            it.s[f] = it.s[f] + ax * ds[f]
            it.lam[f] = it.lam[f] + al * dl[f]
        r = residuals(p, it)
    dt = (time.perf_counter() - t0) / iters
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", "0")) or os.cpu_count()
    return dt, cores


def oracle_ipm_iters(workload: str, seed: int):
    path = os.path.join(ROOT, "tests", "golden", "oracle_counts.json")
    if os.path.exists(path):
        d = json.load(open(path)).get(f"{workload}/seed{seed}")
        if d:
            return int(d["ipm_iters"]), "tests/golden/oracle_counts.json (full oracle run)"
    return None, None


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    n_ipm, src = oracle_ipm_iters(args.workload, args.seed)
    times = []
    for _ in range(args.warmup):          # untimed warm-up samples (page-in, BLAS thread pools)
        oracle_sample(args.workload, args.seed, 1)
    cores = None
    for k in range(args.steps):
        dt, cores = oracle_sample(args.workload, args.seed, 1)
        times.append(dt)
    t_iter = statistics.median(times)
    if n_ipm is None:
        n_ipm, src = 20, "assumed 20 IPM iterations (no stored oracle count)"
    qp_s = t_iter * n_ipm
    sample = (f"1 oracle IPM iteration (dense Cholesky of K, n={args.workload}) per step, median of {len(times)}; "
              f"QP time = {t_iter:.2f} s/iter x {n_ipm} IPM iterations [{src}]")
    line = {"impl": "reference", "metric": METRIC, "value": 1.0 / qp_s, "unit": "QP/s", "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": qp_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (gen/planted.py, seeded)",
            "config": {"workload": args.workload, "seed": args.seed},
            "cpu_baseline": {"value": 1.0 / qp_s, "unit": "QP/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": 1.0 / qp_s, "unit": "QP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "qp_solve_s": qp_s, "oracle_s_per_ipm_iter": t_iter}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    from gen.planted import CONFIGS, config
    from gen.torch_io import problem_tensors
    from paper_2405_03584_b200 import QP

    ws, rank, local = _dist()
    if ws > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # C5 at N > 1 (or --shard): ONE QP row-sharded over the ranks (NCCL allgathers inside libipm,
    # SURVEY §8(e)), each rank building only its row block of H on its device; otherwise every
    # rank solves its own QP (seed + rank): replicas, no collective on the data path.
    sharded = (ws > 1 and args.workload == "C5") or args.force_shard
    q = config(args.workload, args.seed if sharded else args.seed + rank)
    n, m, nnz = q.n, q.m, q.nnz
    extra = {"use_graph": 0} if args.host_loop else {}
    rows = (0, n)
    if sharded:
        from gen.torch_io import device_hessian
        from paper_2405_03584_b200.dist import broadcast_unique_id, nccl_shard, nccl_unique_id, partition
        rows = partition(n, ws)[rank]
        Hb, ldh = device_hessian(q, dev, rows=rows)
        t = problem_tensors(q, dev, H=Hb, ldh=ldh)

        def make_qp(tensors):
            uid = (nccl_unique_id() if ws == 1
                   else broadcast_unique_id(nccl_unique_id, rank, dist.broadcast_object_list))
            return QP(device=dev, shard=nccl_shard(rank, ws, uid), **extra, **tensors)
    else:
        t = problem_tensors(q, dev)

        def make_qp(tensors):
            return QP(device=dev, **extra, **tensors)
    torch.cuda.synchronize()
    qp = make_qp(t)
    stream = qp.stream

    def barrier():
        if ws > 1:
            dist.barrier()

    for _ in range(args.warmup):
        qp.solve()
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
        status = qp.solve()
        stats.append(qp.stats())
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = qp.kernel_launches() - launches0
    kt1 = qp.kernel_timer()
    kt_ms, kt_n = kt1[0] - kt0[0], kt1[1] - kt0[1]
    t_s = e0.elapsed_time(e1) / 1e3
    tt = torch.tensor([t_s], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max = float(tt.item())
    pcg_total = sum(s["pcg_iters_total"] for s in stats)
    pcg_ms = sum(s["t_pcg_ms"] for s in stats)
    ipm_iters = [s["ipm_iters"] for s in stats]
    statuses = sorted(set(s["status"] for s in stats))

    # --- roofline of the dominant kernel (the PCG GEMV), CUDA events on our stream -------
    info = qp.info()
    gemv_iso_ms = qp.profile("gemv", reps=10 if n >= 10000 else 50)
    # live: the dominant kernel's own average launch duration over the timed region
    # (device %globaltimer from its first CTA start to its last CTA end, summed in-kernel)
    gemv_ms = kt_ms / kt_n if kt_n > 0 else gemv_iso_ms
    pcg_iter_ms = qp.profile("pcg_iter", reps=10 if n >= 10000 else 50)
    ncb = info["ncb"]
    if info["gemv_kernel"] == 3:
        # symmetric GEMV: algorithmic bytes = the tiles this rank streams (its share of the upper
        # block triangle, from the library's own work plan) + p + the tile partials
        import ctypes as C
        from paper_2405_03584_b200 import _lib
        nt = C.c_int32()
        _lib.ipm_sym_plan(n, ws if sharded else 1, rank if sharded else 0, 148, None, 0, C.byref(nt), None, None, None)
        tl = (C.c_int32 * (8 * nt.value))()
        _lib.ipm_sym_plan(n, ws if sharded else 1, rank if sharded else 0, 148, tl, nt.value, C.byref(nt), None,
                          None, None)
        elems = sum(tl[8 * t + 1] * tl[8 * t + 3] for t in range(nt.value))
        nrow = rows[1] - rows[0]
        gemv_bytes = 8.0 * elems + 8.0 * n + 8.0 * nrow * ncb
        kname = "k_symv_bulk<1> (symmetric upper-triangle GEMV, 2-D TMA, p^T (H + Sigma_b) p fused)"
    else:
        nrow = rows[1] - rows[0]
        gemv_bytes = 8.0 * nrow * n + 8.0 * n + 8.0 * nrow * ncb   # H (local rows) + p + tile partials
        kname = ("k_gemv_bulk<1> (TMA-bulk GEMV, p^T H p fused)" if info["gemv_kernel"] == 2
                 else "k_gemv_tiles<1,1> (LDG.128 GEMV, p^T H p fused)")
    peak, peak_src = _peaks()
    achieved = gemv_bytes / (gemv_ms * 1e-3) / 1e9
    effective = 8.0 * (rows[1] - rows[0]) * n / (gemv_ms * 1e-3) / 1e9   # dense-H-equivalent rate
    traffic = None
    tp = os.path.join(ROOT, "profiles", "gemv_traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp)).get(f"{args.workload}/gemv_kernel{info['gemv_kernel']}")
        if tj:
            traffic = tj.get("dram_bytes_per_launch")
    iter_bytes = gemv_bytes + 2 * 12.0 * nnz + 8.0 * (m + 1) + 8.0 * (n + 1) + 8.0 * 2 * m + 8.0 * 12 * n

    # --- end to end through the public API with host buffers ----------------------------
    if sharded:
        import numpy as np
        from gen.planted import hessian_rows
        ldh_h = n + (n & 1)
        Hh = np.zeros((rows[1] - rows[0], ldh_h))
        Hh[:, :n] = hessian_rows(q.d, q.U, q.w, rows[0], rows[1])
        th = problem_tensors(q, dev, H=torch.from_numpy(Hh).pin_memory(), ldh=ldh_h, host=True)
    else:
        th = problem_tensors(q, dev, host=True)
    h2d = sum(v.numel() * v.element_size() for k, v in th.items() if hasattr(v, "numel"))
    e2e_times = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        a0 = time.perf_counter()
        qp2 = make_qp(th)                     # H2D of every input (pinned), validation, A^T build
        qp2.solve()
        x_host = qp2.solution()["x"].cpu()   # D2H of the result
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - a0)
        qp2.close()
        del qp2
    e2e_t = sum(e2e_times)
    te = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    d2h = (rows[1] - rows[0]) * 8

    # --- the smaller configs of BASELINE.json, for context (median QP time, 1 GPU) ----------
    others = {}
    if ws == 1 and not args.no_extra:
        for wl, reps in (("C1", 5), ("C2", 3)):
            qo = config(wl, args.seed)
            qx = QP(device=dev, **problem_tensors(qo, dev))
            qx.solve()
            ts = []
            for _ in range(reps):
                qx.solve()
                ts.append(qx.stats())
            ts.sort(key=lambda s: s["t_solve_ms"])
            med = ts[len(ts) // 2]
            others[wl] = {"qp_solve_ms": med["t_solve_ms"], "ipm_iters": med["ipm_iters"],
                          "pcg_iters": med["pcg_iters_total"], "status": med["status"],
                          "gemv_kernel": qx.info()["gemv_kernel"]}
            qx.close()

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        n_ipm, src = oracle_ipm_iters(args.workload, args.seed)
        if n_ipm is None:
            n_ipm, src = int(round(statistics.mean(ipm_iters))), "IPM count of this GPU run (parity +-2)"
        dt, cores = oracle_sample(args.workload, args.seed, 1)
        cpu = {"value": 1.0 / (dt * n_ipm), "unit": "QP/s", "cores": cores, "kind": "oracle",
               "sample": f"1 oracle IPM iteration of {args.workload} seed {args.seed} ({dt:.1f} s, dense Cholesky "
                         f"of K on {cores} host threads) x {n_ipm} IPM iterations [{src}]"}

    if rank == 0:
        qps = (1 if sharded else ws) * args.steps / t_max
        line = {
            "metric": METRIC, "value": qps, "unit": "QP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic planted-KKT QP (gen/planted.py, seeded; random-init dyadic H = diag + U W U^T)",
            "config": {"workload": args.workload, **CONFIGS[args.workload],
                       "seed": args.seed if (sharded or ws == 1) else f"{args.seed}..{args.seed + ws - 1} (one per rank)", "nnz": nnz,
                       "H_bytes": 8 * n * n, "l2": _l2_note(n),
                       "parallelism": (f"row-sharded H over {ws} GPUs (NCCL allgather)" if sharded
                                       else (f"replicas x{ws}" if ws > 1 else "1 GPU"))},
            "qp_solve_s": t_max / args.steps,
            "pcg_it_per_s": pcg_total / (pcg_ms * 1e-3) if pcg_ms > 0 else None,
            "pcg_iters_per_qp": pcg_total / args.steps, "ipm_iters": ipm_iters, "status": statuses,
            "pcg_iter_us_isolated": pcg_iter_ms * 1e3,
            "op_apply_GBps": iter_bytes / (pcg_iter_ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": kname,
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "algorithmic_bytes_per_launch": gemv_bytes,
                         "dense_equivalent_GBps": effective,
                         "launch_ms": gemv_ms, "launches_timed": int(kt_n), "peak_source": peak_src,
                         "share_of_step": kt_ms / (t_max * 1e3) if kt_n > 0 else None,
                         "isolated_launch_ms": gemv_iso_ms,
                         "timing": ("live: in-kernel %globaltimer (first CTA start to last CTA end) summed over "
                                    "every launch in the timed region, on the library stream"
                                    if kt_n > 0 else "CUDA events, back-to-back launches after the timed region (small n: the timed "
                                    "PCG ran in the single-CTA k_pcg_small, not in this kernel)")},
            "cpu_baseline": cpu,
            "e2e": {"value": (1 if sharded else ws) * args.steps / float(te.item()), "unit": "QP/s",
                    "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches), "clocks": clk, "other_workloads": others,
        }
        print(json.dumps(line), flush=True)
    qp.close()
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C3", choices=["C1", "C2", "C3", "C5"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", "--force-shard", dest="force_shard", action="store_true",
                    help="row-shard ONE QP over the N ranks (default only for C5) — also at N = 1 (NCCL path)")
    ap.add_argument("--no-extra", action="store_true", help="skip the C1/C2 context timings")
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
