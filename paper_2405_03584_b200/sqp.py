"""Python façade over include/sqp.h — the closed-loop SQP driver.

``SQP`` marshals a dose-like NLP (gen.dose_nlp.DoseNLP fields, or tensors of the same
names) and its constant linear constraints into ``ipm_sqp_create``; every step (objective,
gradient, QP subproblems, line search, BFGS update) runs in libipm.so.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib as L
from .qp import _dev, make_options


def make_sqp_options(**kw) -> L.ipm_sqp_options:
    o = L.ipm_sqp_options()
    L.ipm_sqp_options_default(C.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise KeyError(f"unknown sqp option {k!r}")
        setattr(o, k, int(v) if isinstance(getattr(o, k), int) else float(v))
    return o


class SQP:
    """min f(x) (dose-like, R20)  s.t.  l <= A x <= u,  xl <= x <= xu, by SQP over GPU IPM QPs."""

    def __init__(self, D_rowptr, D_col, D_val, w, p, dmax, kappa, beta, A_rowptr, A_col, A_val, l, u, xl, xu, *,
                 device=None, stream: Optional[torch.cuda.Stream] = None, qp_options: Optional[dict] = None,
                 **sqp_options):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2405_03584_b200 needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream or torch.cuda.current_stream(self.device)
        f64, dev = torch.float64, self.device
        with torch.cuda.device(dev), torch.cuda.stream(self.stream):
            self.t = dict(D_rowptr=_dev(D_rowptr, torch.int64, dev), D_col=_dev(D_col, torch.int32, dev),
                          D_val=_dev(D_val, f64, dev), w=_dev(w, f64, dev), p=_dev(p, f64, dev),
                          dmax=_dev(dmax, f64, dev), kappa=_dev(kappa, f64, dev),
                          A_rowptr=_dev(A_rowptr, torch.int64, dev), A_col=_dev(A_col, torch.int32, dev),
                          A_val=_dev(A_val, f64, dev), l=_dev(l, f64, dev), u=_dev(u, f64, dev),
                          xl=_dev(xl, f64, dev), xu=_dev(xu, f64, dev))
            t = self.t
            self.n = int(t["xl"].shape[0])
            self.m = int(t["l"].shape[0])
            nlp = L.ipm_dose_nlp()
            nlp.nd, nlp.nnz = int(t["w"].shape[0]), int(t["D_val"].shape[0])
            for k in ("D_rowptr", "D_col", "D_val", "w", "p", "dmax", "kappa"):
                setattr(nlp, k, t[k].data_ptr())
            nlp.beta = float(beta)
            cons = L.ipm_problem()
            cons.n, cons.m, cons.nnz, cons.ldh = self.n, self.m, int(t["A_val"].shape[0]), self.n
            for k in ("A_rowptr", "A_col", "A_val", "l", "u", "xl", "xu"):
                setattr(cons, k, t[k].data_ptr())
            cons.row_begin, cons.row_end, cons.nranks = 0, self.n, 1
            self._nlp, self._cons = nlp, cons
            self.sqp_options = make_sqp_options(**sqp_options)
            self.qp_options = make_options(**(qp_options or {}))
            nb = C.c_size_t(0)
            st = L.ipm_sqp_workspace_size(C.byref(cons), C.byref(nlp), C.byref(self.sqp_options),
                                          C.byref(self.qp_options), C.byref(nb))
            if st != L.IPM_OK:
                raise L.IpmError(st, (L.ipm_sqp_last_error(None) or b"").decode(errors="replace"))
            self.workspace = torch.empty(max(int(nb.value), 256), dtype=torch.uint8, device=dev)
            h = C.c_void_p()
            st = L.ipm_sqp_create(C.byref(h), C.byref(cons), C.byref(nlp), C.byref(self.sqp_options),
                                  C.byref(self.qp_options), C.c_void_p(self.workspace.data_ptr()),
                                  C.c_size_t(self.workspace.numel()), C.c_void_p(self.stream.cuda_stream))
            if st != L.IPM_OK:
                raise L.IpmError(st, (L.ipm_sqp_last_error(None) or b"").decode(errors="replace"))
            self.h = h

    @staticmethod
    def from_nlp(q, **kw) -> "SQP":
        return SQP(q.D_rowptr, q.D_col, q.D_val, q.w, q.p, q.dmax, q.kappa, q.beta, q.A_rowptr, q.A_col, q.A_val,
                   q.l, q.u, q.xl, q.xu, **kw)

    def _check(self, st, allow=(L.IPM_OK,)):
        if st not in allow:
            raise L.IpmError(st, (L.ipm_sqp_last_error(self.h) or b"").decode(errors="replace"))
        return st

    def close(self):
        if getattr(self, "h", None):
            L.ipm_sqp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, x0, raise_on_error: bool = True) -> str:
        with torch.cuda.stream(self.stream):
            x0 = _dev(x0, torch.float64, self.device)
        st = L.ipm_sqp_solve(self.h, C.c_void_p(x0.data_ptr()))
        if raise_on_error:
            self._check(st, allow=(L.IPM_OK, L.IPM_NOT_CONVERGED))
        return L.STATUS_NAMES[st]

    def x(self) -> torch.Tensor:
        out = torch.empty(self.n, dtype=torch.float64, device=self.device)
        self._check(L.ipm_sqp_get_x(self.h, C.c_void_p(out.data_ptr())))
        self.stream.synchronize()
        return out

    def stats(self) -> dict:
        s = L.ipm_sqp_stats()
        self._check(L.ipm_sqp_get_stats(self.h, C.byref(s)))
        d = {k: getattr(s, k) for k, _ in L.ipm_sqp_stats._fields_}
        d["status"] = L.STATUS_NAMES.get(d["status"], d["status"])
        return d

    def trace(self) -> list:
        cnt = C.c_int32()
        self._check(L.ipm_sqp_get_trace(self.h, None, 0, C.byref(cnt)))
        recs = (L.ipm_sqp_trace_rec * max(1, cnt.value))()
        self._check(L.ipm_sqp_get_trace(self.h, recs, cnt.value, C.byref(cnt)))
        return [{k: getattr(r, k) for k, _ in L.ipm_sqp_trace_rec._fields_} for r in recs[:cnt.value]]

    def eval(self, x):
        with torch.cuda.stream(self.stream):
            x = _dev(x, torch.float64, self.device)
        g = torch.empty(self.n, dtype=torch.float64, device=self.device)
        f = C.c_double()
        self._check(L.ipm_sqp_eval(self.h, C.c_void_p(x.data_ptr()), C.byref(f), C.c_void_p(g.data_ptr())))
        self.stream.synchronize()
        return f.value, g

    def kernel_launches(self) -> int:
        return int(L.ipm_sqp_kernel_launches(self.h))
