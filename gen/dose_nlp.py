"""Seeded synthetic dose-like NLPs for the closed-loop SQP driver.

Holds NONE of the method's arithmetic: no objective or gradient evaluation, no SQP or BFGS
step.  It only draws the data of

    min f(x),  f(x) = sum_i [ 1/2 w_i (d_i - p_i)^2 + (kappa_i / beta) exp(beta (d_i - dmax_i)) ],
    d = D x,   s.t.  l <= A x <= u,  xl <= x <= xu

(eq:nlp_general P:131-137 with linear constraints g(x) = A x - u <= 0, l - A x <= 0 and the
variable bounds; the objective form is reading R20 in DESIGN.md — the paper only says the
objective is smooth, and the RayStation functions are not published).  D is a sparse
non-negative "dose deposition" matrix (voxels x spots/segments), so f is convex; targets
carry a prescription p_i = 1 with weight 1, organs at risk p_i = 0 with weight 0.1 and an
exponential over-dose penalty above dmax_i.

Recipe (restated in DESIGN.md §4):
* D: nd rows, each with kd distinct sorted uniform columns, values U(0.1, 1) * (2 / kd)
  (a uniform x = 1/2 gives d ~ 1/2 ... 1); every column is touched by at least one row
  (rows i < n get column i added), so diag(D^T W D) > 0.
* 30 % target voxels (w = 1, p = 1, kappa = 0), 70 % organ-at-risk voxels (w = 0.1, p = 0,
  kappa = 0.05, dmax ~ U(0.4, 0.8)); beta = 8.
* Bounds 0 <= x <= xu, xu ~ U(1, 2).  x0 = xu / 2 (strictly inside).
* Linear rows (optional): same sparsity recipe as gen/planted.py (density, VMAT lower/upper
  split P:381), bounds placed around A x0 with relative slack U(0.05, 0.3) so x0 is strictly
  feasible; the optimum typically makes some of them active.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

from gen.planted import VMAT_LOWER_FRACTION, _draw_sparse_rows


@dataclasses.dataclass
class DoseNLP:
    n: int
    nd: int
    m: int
    D_rowptr: np.ndarray     # (nd+1,) int64
    D_col: np.ndarray        # int32, strictly increasing within a row
    D_val: np.ndarray        # float64, > 0
    w: np.ndarray            # (nd,) > 0
    p: np.ndarray            # (nd,)
    dmax: np.ndarray         # (nd,)
    kappa: np.ndarray        # (nd,) >= 0
    beta: float
    A_rowptr: np.ndarray     # (m+1,)
    A_col: np.ndarray
    A_val: np.ndarray
    l: np.ndarray
    u: np.ndarray
    xl: np.ndarray
    xu: np.ndarray
    x0: np.ndarray
    name: str = ""
    seed: int = 0

    @property
    def D_nnz(self) -> int:
        return int(self.D_rowptr[-1])

    @property
    def nnz(self) -> int:
        return int(self.A_rowptr[-1])

    def D_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.D_val, self.D_col.astype(np.int64), self.D_rowptr), shape=(self.nd, self.n))

    def A_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.A_val, self.A_col.astype(np.int64), self.A_rowptr), shape=(self.m, self.n))


def _dose_rows(rng, nd, n, kd):
    rowptr, cols, vals = _draw_sparse_rows(rng, nd, n, kd)
    # guarantee every column is touched: row i (< n) also gets column i
    if nd < n:
        raise ValueError("nd >= n required (every spot must reach a voxel)")
    out_p = [0]
    out_c, out_v = [], []
    extra = rng.uniform(0.1, 1.0, size=n)
    for i in range(nd):
        c = cols[rowptr[i]:rowptr[i + 1]]
        v = vals[rowptr[i]:rowptr[i + 1]]
        if i < n and not np.any(c == i):
            j = np.searchsorted(c, i)
            c = np.insert(c, j, i)
            v = np.insert(v, j, extra[i])
        out_c.append(c)
        out_v.append(v)
        out_p.append(out_p[-1] + c.size)
    col = np.concatenate(out_c).astype(np.int32)
    val = np.concatenate(out_v) * (2.0 / kd)
    return np.asarray(out_p, dtype=np.int64), col, val


def dose_nlp(n: int, nd: int, kd: int, m: int = 0, *, density: float = 0.01, rows: str = "vmat",
             seed: int = 0, name: str = "") -> DoseNLP:
    rng = np.random.default_rng(seed)
    Dp, Dc, Dv = _dose_rows(rng, nd, n, kd)
    target = rng.uniform(size=nd) < 0.3
    w = np.where(target, 1.0, 0.1)
    p = np.where(target, 1.0, 0.0)
    kappa = np.where(target, 0.0, 0.05)
    dmax = np.where(target, np.inf, rng.uniform(0.4, 0.8, size=nd))
    dmax = np.where(np.isfinite(dmax), dmax, 0.0)      # kappa = 0 there: value irrelevant
    xl = np.zeros(n)
    xu = rng.uniform(1.0, 2.0, size=n)
    x0 = 0.5 * xu
    if m > 0:
        k = max(1, int(round(density * n)))
        Ap, Ac, Av = _draw_sparse_rows(rng, m, n, k)
        Ax0 = np.array([float(np.dot(Av[Ap[i]:Ap[i + 1]], x0[Ac[Ap[i]:Ap[i + 1]]])) for i in range(m)])
        slack = rng.uniform(0.05, 0.3, size=m) * np.maximum(np.abs(Ax0), 1e-3)
        lower = np.zeros(m, bool)
        if rows == "vmat":
            lower[rng.permutation(m)[:int(round(VMAT_LOWER_FRACTION * m))]] = True
        elif rows == "upper":
            pass
        else:
            raise ValueError(rows)
        l = np.where(lower, Ax0 - slack, -np.inf)
        u = np.where(lower, np.inf, Ax0 + slack)
    else:
        Ap, Ac, Av = np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0)
        l = np.zeros(0)
        u = np.zeros(0)
    return DoseNLP(n=n, nd=nd, m=m, D_rowptr=Dp, D_col=Dc, D_val=Dv, w=w, p=p, dmax=dmax, kappa=kappa,
                   beta=8.0, A_rowptr=Ap, A_col=Ac, A_val=Av, l=l, u=u, xl=xl, xu=xu, x0=x0,
                   name=name, seed=seed)


# Paper-shaped SQP workloads (Table 1; QP counts P:300)
NLP_CONFIGS = {
    "S1": dict(n=40, nd=80, kd=6, m=12, density=0.25),                 # oracle-sized
    "S-vmat": dict(n=13425, nd=40000, kd=48, m=68618, density=0.004),   # VMAT H&N shape, 33 SQP its
    "S-proton": dict(n=77373, nd=150000, kd=40, m=0),                   # proton H&N shape, 100 SQP its
    "S-c4": dict(n=20000, nd=40000, kd=64, m=5000, density=0.01),       # C4 closed loop, dense H
}


def nlp_config(name: str, seed: int = 0, **overrides) -> DoseNLP:
    kw = dict(NLP_CONFIGS[name])
    kw.update(overrides)
    return dose_nlp(seed=seed, name=name, **kw)
