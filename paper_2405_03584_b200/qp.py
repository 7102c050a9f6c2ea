"""Python façade over the C ABI (include/ipm.h).

``QP`` owns a context created by ``ipm_create`` on torch-allocated device memory
(PyTorch is used only for device memory, streams and process groups — north_star (a)).
All compute runs in libipm.so's sm_100a kernels.  Inputs may be CUDA tensors (zero
copy, borrowed) or CPU tensors / numpy arrays, which are copied to the device first
(this is the end-to-end path ``bench.py`` times for ``e2e``).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Optional

import numpy as np
import torch

from . import _lib as L

_FAMILIES = ("lA", "uA", "lx", "ux")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def make_options(**kw) -> L.ipm_options:
    o = L.ipm_options()
    L.ipm_options_default(C.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise KeyError(f"unknown ipm option {k!r}")
        setattr(o, k, int(v) if isinstance(getattr(o, k), int) else float(v))
    return o


def _dev(x, dtype, device, pin=False):
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if x.dtype != dtype:
        x = x.to(dtype)
    if x.device.type != "cuda":
        if pin and not x.is_pinned():
            x = x.pin_memory()
        x = x.to(device, non_blocking=True)
    return x.contiguous()


class QP:
    """min 1/2 x^T H x + g^T x  s.t.  l <= A x <= u,  xl <= x <= xu   (eq:qp)."""

    def __init__(self, H, g, A_rowptr, A_col, A_val, l, u, xl, xu, *, ldh: Optional[int] = None,
                 device=None, stream: Optional[torch.cuda.Stream] = None, shard: Optional[dict] = None,
                 compact: Optional[dict] = None, **options):
        """shard (row-sharded path): dict(rank, nranks, comm_kind, handle) where
        H holds only this rank's row block (see paper_2405_03584_b200.dist.partition) and
        handle is a ctypes pointer to an ncclUniqueId (comm_kind 1) or an ipm_group (2).
        compact (matrix-free quasi-Newton H = diag(h0) + U diag(w) U^T, eq:bfgs_hessian, SURVEY
        NEXT-1): dict(h0=(n,), U=(n, ldu) row-major with the first k columns in use, w=(k,), k);
        H is then ignored (may be None) and rank-2 updates append columns of U."""
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2405_03584_b200 needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream or torch.cuda.current_stream(self.device)
        f64 = torch.float64
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            n = int(g.shape[0])
            if H is None:
                if compact is None:
                    raise ValueError("H is required unless compact= is given")
                H = torch.zeros(2, dtype=f64, device=self.device)   # placeholder, not read
                ldh = n
            if isinstance(H, np.ndarray):
                H = torch.from_numpy(H)
            if H.device.type != "cuda":
                H = H.to(f64)
                if not H.is_pinned():
                    H = H.pin_memory()
                H = H.to(self.device, non_blocking=True)
            if ldh is None:
                ldh = H.stride(0) if H.dim() == 2 else n
            self.H = H
            self.g = _dev(g, f64, self.device)
            self.A_rowptr = _dev(A_rowptr, torch.int64, self.device)
            self.A_col = _dev(A_col, torch.int32, self.device)
            self.A_val = _dev(A_val, f64, self.device)
            self.l = _dev(l, f64, self.device)
            self.u = _dev(u, f64, self.device)
            self.xl = _dev(xl, f64, self.device)
            self.xu = _dev(xu, f64, self.device)
            self.n, self.m, self.nnz = n, int(self.l.shape[0]), int(self.A_val.shape[0])
            prob = L.ipm_problem()
            prob.n, prob.m, prob.nnz = self.n, self.m, self.nnz
            prob.H, prob.ldh = self.H.data_ptr(), int(ldh)
            prob.g = self.g.data_ptr()
            prob.A_rowptr, prob.A_col, prob.A_val = self.A_rowptr.data_ptr(), self.A_col.data_ptr(), self.A_val.data_ptr()
            prob.l, prob.u, prob.xl, prob.xu = self.l.data_ptr(), self.u.data_ptr(), self.xl.data_ptr(), self.xu.data_ptr()
            prob.row_begin, prob.row_end, prob.rank, prob.nranks = 0, n, 0, 1
            self.row0, self.nloc = 0, n
            if compact is not None:
                self.c_h0 = _dev(compact["h0"], f64, self.device)
                Uc = compact["U"]
                if isinstance(Uc, np.ndarray):
                    Uc = torch.from_numpy(np.ascontiguousarray(Uc))
                self.c_U = Uc.to(self.device, f64).contiguous()
                self.c_w = _dev(compact["w"], f64, self.device) if int(compact["k"]) > 0 else torch.zeros(1, dtype=f64,
                                                                                                     device=self.device)
                prob.hess_kind, prob.k, prob.ldu = 1, int(compact["k"]), int(self.c_U.shape[1])
                prob.h0, prob.U, prob.w = self.c_h0.data_ptr(), self.c_U.data_ptr(), self.c_w.data_ptr()
            if shard is not None:
                from .dist import partition
                P = int(shard["nranks"])
                r = int(shard["rank"])
                b, e = partition(n, P)[r]
                prob.row_begin, prob.row_end, prob.rank, prob.nranks = b, e, r, P
                prob.comm_kind = int(shard["comm_kind"])
                prob.comm_handle_host = C.cast(shard["handle"], C.c_void_p)
                self._shard_keep = shard
                self.row0, self.nloc = b, e - b
            self._prob = prob
            self.options = make_options(**options)
            nbytes = C.c_size_t(0)
            L.check(L.ipm_workspace_size(C.byref(prob), C.byref(self.options), C.byref(nbytes)))
            self.workspace = torch.empty(max(int(nbytes.value), 256), dtype=torch.uint8, device=self.device)
            ctx = C.c_void_p()
            st = L.ipm_create(C.byref(ctx), C.byref(prob), C.byref(self.options), C.c_void_p(self.workspace.data_ptr()),
                              C.c_size_t(self.workspace.numel()), C.c_void_p(self.stream.cuda_stream))
            L.check(st, None)
            self.ctx = ctx

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "ctx", None):
            L.ipm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------------ solve
    def solve(self, raise_on_error: bool = True) -> str:
        st = L.ipm_solve(self.ctx)
        if raise_on_error:
            L.check(st, self.ctx, allow=(L.IPM_OK, L.IPM_NOT_CONVERGED))
        return L.STATUS_NAMES[st]

    def solution(self) -> Dict[str, torch.Tensor]:
        out = {"x": torch.empty(self.nloc, dtype=torch.float64, device=self.device)}
        for f in _FAMILIES:
            ln = self.m if f.endswith("A") else self.nloc
            out["lam_" + f] = torch.zeros(ln, dtype=torch.float64, device=self.device)
        obj = C.c_double()
        L.check(L.ipm_get_solution(self.ctx, _ptr(out["x"]), _ptr(out["lam_lA"]), _ptr(out["lam_uA"]),
                                   _ptr(out["lam_lx"]), _ptr(out["lam_ux"]), C.byref(obj)), self.ctx)
        out["obj"] = obj.value
        return out

    def stats(self) -> dict:
        s = L.ipm_stats()
        L.check(L.ipm_get_stats(self.ctx, C.byref(s)), self.ctx)
        d = {k: getattr(s, k) for k, _ in L.ipm_stats._fields_}
        d["status"] = L.STATUS_NAMES.get(d["status"], d["status"])
        return d

    def info(self) -> dict:
        i = L.ipm_info()
        L.check(L.ipm_get_info(self.ctx, C.byref(i)), self.ctx)
        return {k: getattr(i, k) for k, _ in L.ipm_info._fields_}

    def trace(self) -> list:
        cnt = C.c_int32()
        L.check(L.ipm_get_trace(self.ctx, None, 0, C.byref(cnt)), self.ctx)
        recs = (L.ipm_trace_rec * max(1, cnt.value))()
        L.check(L.ipm_get_trace(self.ctx, recs, cnt.value, C.byref(cnt)), self.ctx)
        return [{k: getattr(r, k) for k, _ in L.ipm_trace_rec._fields_} for r in recs[:cnt.value]]

    def profile(self, what: str = "gemv", reps: int = 20) -> float:
        """Average device ms per launch of one hot-path stage (CUDA events on our stream)."""
        code = {"gemv": 0, "spmv": 1, "pcg_iter": 2}[what]
        ms = C.c_double()
        L.check(L.ipm_profile(self.ctx, code, int(reps), C.byref(ms)), self.ctx)
        return ms.value

    def kernel_launches(self) -> int:
        return int(L.ipm_kernel_launches(self.ctx))

    def kernel_timer(self) -> tuple:
        """(cumulative ms, launches) of the PCG operator kernel, timed on the device."""
        ms, cnt = C.c_double(), C.c_int64()
        L.check(L.ipm_kernel_timer(self.ctx, C.byref(ms), C.byref(cnt)), self.ctx)
        return ms.value, cnt.value

    # ------------------------------------------------------------------ C4
    def set_linear_term(self, g):
        self._g_new = _dev(g, torch.float64, self.device)
        L.check(L.ipm_set_linear_term(self.ctx, _ptr(self._g_new)), self.ctx)

    def update_hessian_rank2(self, u, alpha: float, v, beta: float):
        uu = _dev(u, torch.float64, self.device)
        vv = _dev(v, torch.float64, self.device)
        L.check(L.ipm_update_hessian_rank2(self.ctx, _ptr(uu), float(alpha), _ptr(vv), float(beta)), self.ctx)
        self.stream.synchronize()

    def set_bounds(self, l, u, xl, xu):
        """New bounds for the next solve (same finite pattern; ipm_set_bounds)."""
        self._bounds_new = [_dev(a, torch.float64, self.device) for a in (l, u, xl, xu)]
        L.check(L.ipm_set_bounds(self.ctx, *[_ptr(a) for a in self._bounds_new]), self.ctx)

    def warm_start(self):
        L.check(L.ipm_warm_start(self.ctx), self.ctx)

    def set_iterate(self, x, s: Dict[str, torch.Tensor], lam: Dict[str, torch.Tensor], mu: float):
        keep = [_dev(x, torch.float64, self.device)]
        sp = (C.c_void_p * 4)()
        lp = (C.c_void_p * 4)()
        for i, f in enumerate(_FAMILIES):
            a = _dev(s[f], torch.float64, self.device)
            b = _dev(lam[f], torch.float64, self.device)
            keep += [a, b]
            sp[i] = a.data_ptr()
            lp[i] = b.data_ptr()
        L.check(L.ipm_set_iterate(self.ctx, _ptr(keep[0]), sp, lp, float(mu)), self.ctx)
        self.stream.synchronize()

    def get_iterate(self):
        x = torch.empty(self.nloc, dtype=torch.float64, device=self.device)
        s, lam = {}, {}
        sp = (C.c_void_p * 4)()
        lp = (C.c_void_p * 4)()
        for i, f in enumerate(_FAMILIES):
            ln = self.m if f.endswith("A") else self.nloc
            s[f] = torch.zeros(ln, dtype=torch.float64, device=self.device)
            lam[f] = torch.zeros(ln, dtype=torch.float64, device=self.device)
            sp[i] = s[f].data_ptr()
            lp[i] = lam[f].data_ptr()
        mu = C.c_double()
        L.check(L.ipm_get_iterate(self.ctx, _ptr(x), sp, lp, C.byref(mu)), self.ctx)
        return x, s, lam, mu.value

    # ------------------------------------------------------------------ test hooks
    def op_apply(self, sig_b, sig_c, v) -> torch.Tensor:
        sb, scv, vv = (_dev(a, torch.float64, self.device) for a in (sig_b, sig_c, v))
        y = torch.empty(self.nloc, dtype=torch.float64, device=self.device)
        L.check(L.ipm_op_apply(self.ctx, _ptr(sb), _ptr(scv), _ptr(vv), _ptr(y)), self.ctx)
        return y

    def op_diag(self, sig_b, sig_c) -> torch.Tensor:
        sb, scv = (_dev(a, torch.float64, self.device) for a in (sig_b, sig_c))
        d = torch.empty(self.nloc, dtype=torch.float64, device=self.device)
        L.check(L.ipm_op_diag(self.ctx, _ptr(sb), _ptr(scv), _ptr(d)), self.ctx)
        return d

    def pcg(self, sig_b, sig_c, rhs, rtol: float):
        sb, scv, r = (_dev(a, torch.float64, self.device) for a in (sig_b, sig_c, rhs))
        x = torch.empty(self.nloc, dtype=torch.float64, device=self.device)
        it = C.c_int32()
        st = L.ipm_pcg(self.ctx, _ptr(sb), _ptr(scv), _ptr(r), _ptr(x), float(rtol), C.byref(it))
        L.check(st, self.ctx, allow=(L.IPM_OK, L.IPM_NOT_CONVERGED))
        return x, it.value

    def pcg_iterate(self, sig_b, sig_c, rhs, k: int) -> dict:
        """Exactly k PCG iterations of the solve's own kernels (ipm_pcg_iterate test hook)."""
        sb, scv, r = (_dev(a, torch.float64, self.device) for a in (sig_b, sig_c, rhs))
        out = {key: torch.empty(self.nloc, dtype=torch.float64, device=self.device) for key in ("x", "r", "z", "p")}
        sc = (C.c_double * 4)()
        L.check(L.ipm_pcg_iterate(self.ctx, _ptr(sb), _ptr(scv), _ptr(r), int(k), _ptr(out["x"]), _ptr(out["r"]),
                                  _ptr(out["z"]), _ptr(out["p"]), sc), self.ctx)
        out.update(rho=sc[0], pKp=sc[1], alpha=sc[2], rr=sc[3])
        return out
