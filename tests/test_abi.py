"""CPU-only checks of the boundary: libipm.so loads, exports every entry point that
include/ipm.h declares, and the ctypes structs match the header layout."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("ipm.h", "sqp.h")]


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2405_03584_b200 import _lib
    return _lib


def _declared():
    txt = "".join(open(h).read() for h in HEADERS)
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ipm_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported(lib):
    declared = _declared()
    assert "ipm_create" in declared and "ipm_solve" in declared
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ipm_\w+)", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    # the binding wraps exactly the declared API
    assert sorted(lib.EXPORTED) == declared
    # nothing else leaks out of the library (hidden visibility)
    assert exported == set(declared)


def test_options_default_and_abi(lib):
    assert lib.ipm_abi_version() == 1
    o = lib.ipm_options()
    lib.ipm_options_default(C.byref(o))
    assert o.size == C.sizeof(lib.ipm_options)
    assert o.mu_tol == 1e-8 and o.tau == 0.995 and o.mu_divisor == 10.0 and o.max_ipm_iter == 100
    assert o.pcg_rtol_max == 1e-6 and o.pcg_rtol_floor == 1e-12 and o.use_graph == 1


def test_struct_sizes_match_c(lib, tmp_path):
    """Compile a tiny C program against include/ipm.h and compare sizeof/offsetof with ctypes."""
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "ipm.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(ipm_options), sizeof(ipm_problem), sizeof(ipm_stats), sizeof(ipm_trace_rec),'
                   'offsetof(ipm_options, warm_shift), offsetof(ipm_problem, comm_handle_host),'
                   'offsetof(ipm_options, a_row_split), offsetof(ipm_options, kernel_timer),'
                   'sizeof(ipm_host_comm), offsetof(ipm_host_comm, user));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    assert vals == [C.sizeof(lib.ipm_options), C.sizeof(lib.ipm_problem), C.sizeof(lib.ipm_stats),
                    C.sizeof(lib.ipm_trace_rec), lib.ipm_options.warm_shift.offset,
                    lib.ipm_problem.comm_handle_host.offset, lib.ipm_options.a_row_split.offset,
                    lib.ipm_options.kernel_timer.offset, C.sizeof(lib.ipm_host_comm), lib.ipm_host_comm.user.offset]


def test_workspace_size_host_only(lib):
    p = lib.ipm_problem()
    p.n, p.m, p.nnz, p.ldh, p.nranks = 20000, 5000, 10**6, 20000, 1
    nb = C.c_size_t()
    assert lib.ipm_workspace_size(C.byref(p), None, C.byref(nb)) == lib.IPM_OK
    assert nb.value > 20000 * 8 * 30
    p.n = 0
    assert lib.ipm_workspace_size(C.byref(p), None, C.byref(nb)) == lib.IPM_ERR_INVALID
    assert b"bad dimensions" in lib.ipm_last_error(None)


def test_create_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2405_03584_b200 import QP
    import numpy as np
    with pytest.raises(RuntimeError):
        QP(np.eye(2), np.zeros(2), np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0), np.zeros(0),
           np.zeros(0), -np.ones(2), np.ones(2))


def test_partition_validation_before_any_device_work(lib):
    """ipm_create rejects a row block that is not the ceil(n/P) partition (host check, no GPU)."""
    from paper_2405_03584_b200.dist import LocalGroup, partition
    assert partition(10, 3) == [(0, 4), (4, 8), (8, 10)]
    with pytest.raises(ValueError):
        partition(5, 4)          # ceil(5/4)=2 -> ranks 0..2 cover 6 > 5 rows, rank 3 empty
    grp = LocalGroup(3)
    p = lib.ipm_problem()
    p.n, p.m, p.nnz, p.ldh = 10, 0, 0, 10
    dummy = C.c_void_p(16)
    p.H = p.g = p.xl = p.xu = dummy
    p.rank, p.nranks, p.comm_kind, p.comm_handle_host = 1, 3, 2, grp.handle
    p.row_begin, p.row_end = 3, 8
    ctx = C.c_void_p()
    st = lib.ipm_create(C.byref(ctx), C.byref(p), None, None, 0, None)
    assert st == lib.IPM_ERR_INVALID and b"must be [4,8)" in lib.ipm_last_error(None)
    p.comm_kind = 0
    st = lib.ipm_create(C.byref(ctx), C.byref(p), None, None, 0, None)
    assert st == lib.IPM_ERR_INVALID and b"nranks > 1 needs comm_kind" in lib.ipm_last_error(None)
    grp.close()


def test_sqp_struct_sizes_match_c(lib, tmp_path):
    """include/sqp.h structs vs the ctypes mirrors."""
    src = tmp_path / "sq.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "sqp.h"\nint main(){printf("%zu %zu %zu %zu %zu\\n",'
                   'sizeof(ipm_dose_nlp), sizeof(ipm_sqp_options), sizeof(ipm_sqp_stats), sizeof(ipm_sqp_trace_rec),'
                   'offsetof(ipm_sqp_options, h0_floor));return 0;}\n')
    exe = tmp_path / "sq"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    assert vals == [C.sizeof(lib.ipm_dose_nlp), C.sizeof(lib.ipm_sqp_options), C.sizeof(lib.ipm_sqp_stats),
                    C.sizeof(lib.ipm_sqp_trace_rec), lib.ipm_sqp_options.h0_floor.offset]
    o = lib.ipm_sqp_options()
    lib.ipm_sqp_options_default(C.byref(o))
    assert o.size == C.sizeof(lib.ipm_sqp_options) and o.max_iter == 50 and o.tol_d == 1e-6 and o.powell == 0.2


def _sym_plan(lib, n, P, r, grid):
    nt = C.c_int32()
    ldy, ldz = C.c_int32(), C.c_int32()
    assert lib.ipm_sym_plan(n, P, r, grid, None, 0, C.byref(nt), None, None, None) == 0
    tiles = (C.c_int32 * (8 * nt.value))()
    ranges = (C.c_int32 * (5 * grid))()
    assert lib.ipm_sym_plan(n, P, r, grid, tiles, nt.value, C.byref(nt), ranges, C.byref(ldy), C.byref(ldz)) == 0
    import numpy as np
    return (np.array(tiles, dtype=np.int64).reshape(-1, 8), np.array(ranges, dtype=np.int64).reshape(-1, 5),
            ldy.value, ldz.value)


@pytest.mark.parametrize("n,P,grid", [(1000, 1, 148), (1000, 2, 148), (1000, 3, 7), (1000, 4, 148), (777, 5, 31),
                                      (300, 8, 148), (2600, 6, 148), (20000, 1, 148), (100000, 8, 148)])
def test_sym_plan_uses_every_entry_once(lib, n, P, grid):
    """Host-side work plan of the (sharded) symmetric GEMV (NEXT-3 + SURVEY §8(e)): across all
    ranks, every ORDERED entry (i, j) of H enters y = H p exactly once — as a row part of a tile
    holding row i, or as the column part of a tile holding (j, i) — and each rank's strip ranges
    cover its tiles' strips exactly once, in order.  Pinned by counting, no GPU needed."""
    import numpy as np
    chunk = -(-n // P)
    small = n <= 3000
    used = np.zeros((n, n), dtype=np.int32) if small else None
    per_rank = []
    for r in range(P):
        rb = min(r * chunk, n)
        tiles, ranges, ldy, ldz = _sym_plan(lib, n, P, r, grid)
        reads = 0
        for r0, rows, c0, cols, rslot, cmode, cbase, cslot in tiles:
            gi0 = rb + r0
            assert 0 < rows <= 256 and 0 < cols <= 256 and 0 <= c0 and c0 + cols <= n
            reads += rows * cols
            if small:
                used[gi0:gi0 + rows, c0:c0 + cols] += 1                     # row part
                if cmode != 0:
                    used[c0:c0 + cols, gi0:gi0 + rows] += 1                 # column part (H symmetric)
            if cmode == 0:
                assert c0 == gi0 and cols == rows
            if cmode == 1:
                assert rb <= c0 and c0 + cols <= rb + chunk and cbase == c0 - rb
        per_rank.append(reads)
        # ranges: contiguous, in order, covering every strip once
        strips = [(t[1] + 31) // 32 for t in tiles]
        pos = 0
        flat = [(t, s) for t in range(len(tiles)) for s in range(strips[t])]
        for t0, s0, t1, s1, carry in ranges:
            a = flat.index((t0, s0)) if (t0, s0) != (len(tiles), 0) and t0 < len(tiles) else len(flat)
            b = flat.index((t1, s1)) if t1 < len(tiles) else len(flat)
            if t0 == t1 and s0 == s1:
                continue
            assert a == pos
            pos = b
            assert (carry >= 0) == (s0 > 0 and tiles[t0][5] != 0)
        assert pos == len(flat)
    if small:
        assert used.min() == 1 and used.max() == 1
    # balanced: every rank streams about n^2 / (2P) entries
    assert max(per_rank) <= 1.15 * n * n / (2 * P) + 256 * 256 * 4


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the CPU oracle arm) prints one JSON line with the contract's
    keys; runs on CPU (workload C1 keeps it to seconds)."""
    import json
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "C1",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "cpu_baseline",
              "e2e", "config"):
        assert k in d
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"] == "C1"
