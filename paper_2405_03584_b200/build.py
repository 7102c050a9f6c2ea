"""Build libipm.so in-tree for sm_100a (nvcc; no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libipm.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]
SOURCES = ["linalg.cu", "compact.cu", "pcg.cu", "ipmops.cu", "shard.cu", "peer.cu", "comm.cu", "ipm_api.cu",
           "sqp.cu", "tiny.cu"]


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, variant: str = "") -> str:
    """variant "tl": diagnostic build with per-kernel timeline stamps (-DIPM_TIMELINE) into
    libipm_tl.so; loaded only when IPM_LIB points at it (scripts/timeline_probe.py)."""
    lib = LIB if not variant else LIB.replace("libipm.so", f"libipm_{variant}.so")
    extra = {"tl": ["-DIPM_TIMELINE"], "sr16": ["-DIPM_SYM_SR=16", "-DIPM_SYM_STAGES=6"],
             "sr16s4": ["-DIPM_SYM_SR=16", "-DIPM_SYM_STAGES=4"],
             "nc": ["-DIPM_SYM_NOCOMPUTE"], "nocol": ["-DIPM_SYM_NOCOL"],
             "pf1": ["-DIPM_SYM_PF=1"], "pf2": ["-DIPM_SYM_PF=2"], "pf3": ["-DIPM_SYM_PF=3"],
             "pf4": ["-DIPM_SYM_PF=4"], "pf6": ["-DIPM_SYM_PF=6"], "pf3nc": ["-DIPM_SYM_PF=3", "-DIPM_SYM_NOCOMPUTE"],
             "lds4": ["-DIPM_SYM_LDGSTS", "-DIPM_SYM_LOADERS=4"], "lds2": ["-DIPM_SYM_LDGSTS", "-DIPM_SYM_LOADERS=2"],
             "lds6": ["-DIPM_SYM_LDGSTS", "-DIPM_SYM_LOADERS=6"], "lds4nc": ["-DIPM_SYM_LDGSTS", "-DIPM_SYM_NOCOMPUTE"],
             "ncldg2": ["-DIPM_SYM_NOCOMPUTE", "-DIPM_SYM_LDGW=2"], "ncldg3": ["-DIPM_SYM_NOCOMPUTE", "-DIPM_SYM_LDGW=3"],
             "ldg2": ["-DIPM_SYM_LDGW=2"],
             "hyb10": ["-DIPM_SYM_LDGW=2", "-DIPM_SYM_LDG_EVERY=10"], "hyb7": ["-DIPM_SYM_LDGW=2", "-DIPM_SYM_LDG_EVERY=7"],
             "hyb14": ["-DIPM_SYM_LDGW=2", "-DIPM_SYM_LDG_EVERY=14"], "hyb10w3": ["-DIPM_SYM_LDGW=3", "-DIPM_SYM_LDG_EVERY=10"],
             "l2p0": ["-DIPM_SYM_L2P=0"], "l2p2": ["-DIPM_SYM_L2P=2"], "nohint": ["-DIPM_SYM_NOHINT"],
             "nohintnc": ["-DIPM_SYM_NOHINT", "-DIPM_SYM_NOCOMPUTE"],
             "ldg8d3": ["-DIPM_SYMV_LDG_DEFAULT=1"], "ldgnoring": ["-DIPM_SYMV_LDG_DEFAULT=1", "-DIPM_LDG_NORING"],
             "ldg8d2": ["-DIPM_SYMV_LDG_DEFAULT=1", "-DIPM_LDG_DEPTH=2"],
             "ldg16d2": ["-DIPM_SYMV_LDG_DEFAULT=1", "-DIPM_LDG_NW=16", "-DIPM_LDG_DEPTH=2"], "l2p0nc": ["-DIPM_SYM_L2P=0", "-DIPM_SYM_NOCOMPUTE"]}.get(variant, [])
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers += [os.path.join(ROOT, "include", h) for h in ("ipm.h", "sqp.h")]
    objdir = os.path.join(PKG, "build" + (f"_{variant}" if variant else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC, *ARCH, *FLAGS, *extra, "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stderr

    with ThreadPoolExecutor(max_workers=4) as ex:
        logs = list(ex.map(run, jobs))
    if verbose:
        for lg in logs:
            sys.stderr.write(lg)
    if force or jobs or _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-Xcompiler", "-fvisibility=hidden", "-ldl"]
        run(cmd)
    return lib


if __name__ == "__main__":
    var = "tl" if "--timeline" in sys.argv else next((a[10:] for a in sys.argv if a.startswith("--variant=")), "")
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, variant=var))
