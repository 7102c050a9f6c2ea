"""Seeded synthetic QP generator shared by the oracle tests and the GPU path.

This module holds NONE of the IPM's arithmetic (no residuals, no Newton
systems, no step rules). It only draws problem data

    min 1/2 x^T H x + g^T x   s.t.  l <= A x <= u,  xl <= x <= xu      (P:58-66 eq:qp,
                                                                       bounds split out P:176)

with a *planted* KKT point, so that every size has a closed-form optimum
(SURVEY.md §8(d) "Generator", decision D5).  Recipe (restated in DESIGN.md §4):

* H = diag(d) + U diag(w) U^T, the compact quasi-Newton shape H0 + U W U^T of P:240-245
  (eq:bfgs_hessian).  d_j = 1 + k_j/1024 (k_j uniform in 0..1023), U_ir in {-1,0,+1}/8
  with P(0)=1/3, w_r in {1/2, 1, 2}.  Every entry of H is a sum of r products of
  dyadic numbers with few bits, hence exactly representable in fp64 and
  *independent of summation order*: numpy, cuBLAS or any blocked kernel build the
  bit-identical matrix.
* A: each row has round(density*n) distinct sorted uniform columns, values
  U(0.1, 1) (non-negative, dose-deposition-like).  CSR with int64 row offsets and
  int32 column indices.
* Row bound families: "vmat" split 15751/68618 lower-only, rest upper-only;
  "mixed" 25% two-sided / 25% lower / 40% upper / 10% free.
* Variable bounds: box 0 <= x <= b, b ~ U(1,2) ("box"); "mixed" adds 10% one-sided
  and 5% free variables.
* Planted optimum: 30% of lower-bounded variables at their lower bound, 7% of
  upper-bounded variables at their upper bound, the rest interior; 10% of rows
  active.  Active multipliers ~ U(0.5, 2) (strict complementarity), inactive slacks
  ~ U(0.5, 1.5).  g = -H x* + A^T lam_lA - A^T lam_uA + lam_lx - lam_ux makes the
  stationarity row of eq:perturbed_KKT hold at mu = 0.

Random numbers come from numpy's PCG64 ``default_rng(seed)``; the draw order is
fixed by this file, so a (config, seed) pair names one problem.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

# VMAT H&N split of linear-constraint rows into lower/upper families.
VMAT_LOWER_FRACTION = 15751.0 / 68618.0


@dataclasses.dataclass
class QPData:
    n: int
    m: int
    d: np.ndarray            # (n,) diagonal of H0
    U: np.ndarray            # (n, r) update vectors
    w: np.ndarray            # (r,) update weights
    g: np.ndarray            # (n,)
    A_rowptr: np.ndarray     # (m+1,) int64
    A_col: np.ndarray        # (nnz,) int32, strictly increasing within a row
    A_val: np.ndarray        # (nnz,) float64
    l: np.ndarray            # (m,) -inf = absent
    u: np.ndarray            # (m,) +inf = absent
    xl: np.ndarray           # (n,) -inf = absent
    xu: np.ndarray           # (n,) +inf = absent
    x_star: np.ndarray       # planted optimum
    lam_lA: np.ndarray       # (m,) planted multipliers (0 when inactive / absent)
    lam_uA: np.ndarray
    lam_lx: np.ndarray       # (n,)
    lam_ux: np.ndarray
    f_star: float
    name: str = ""
    seed: int = 0
    _H: Optional[np.ndarray] = None

    @property
    def nnz(self) -> int:
        return int(self.A_rowptr[-1])

    @property
    def H(self) -> np.ndarray:
        """Dense row-major H (n x n fp64), built once on demand."""
        if self._H is None:
            self._H = dense_hessian(self.d, self.U, self.w)
        return self._H

    def A_dense(self) -> np.ndarray:
        Ad = np.zeros((self.m, self.n))
        for i in range(self.m):
            s, e = self.A_rowptr[i], self.A_rowptr[i + 1]
            Ad[i, self.A_col[s:e]] = self.A_val[s:e]
        return Ad

    def A_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.A_val, self.A_col.astype(np.int64), self.A_rowptr),
                             shape=(self.m, self.n))


def dense_hessian(d: np.ndarray, U: np.ndarray, w: np.ndarray) -> np.ndarray:
    """H = diag(d) + U diag(w) U^T, exact in fp64 for generator factors (see module doc)."""
    H = (U * w) @ U.T
    H[np.diag_indices_from(H)] += d
    return H


def hessian_rows(d, U, w, r0: int, r1: int) -> np.ndarray:
    """Rows [r0, r1) of H (same exact values as dense_hessian)."""
    Hb = (U[r0:r1] * w) @ U.T
    Hb[np.arange(r1 - r0), np.arange(r0, r1)] += d[r0:r1]
    return Hb


def hessian_matvec(d, U, w, x) -> np.ndarray:
    return d * x + U @ (w * (U.T @ x))


def _draw_factors(rng, n, r):
    d = 1.0 + rng.integers(0, 1024, size=n).astype(np.float64) / 1024.0
    Ui = rng.choice(np.array([-1.0, 0.0, 1.0]), size=(n, r), p=[1.0 / 3, 1.0 / 3, 1.0 / 3])
    U = Ui / 8.0
    w = rng.choice(np.array([0.5, 1.0, 2.0]), size=r)
    return d, U, w


def _draw_sparse_rows(rng, m, n, k):
    """m rows with k distinct sorted uniform columns each; values U(0.1, 1)."""
    k = max(1, min(n, k))
    rowptr = np.arange(m + 1, dtype=np.int64) * k
    cols = np.empty(m * k, dtype=np.int32)
    for i in range(m):
        if k * 4 >= n:
            c = rng.choice(n, size=k, replace=False)
        else:
            c = np.unique(rng.integers(0, n, size=k + k // 4 + 8))
            while c.size < k:
                c = np.unique(np.concatenate([c, rng.integers(0, n, size=k)]))
            c = rng.permutation(c)[:k]
        cols[i * k:(i + 1) * k] = np.sort(c)
    vals = rng.uniform(0.1, 1.0, size=m * k)
    return rowptr, cols, vals


def planted_qp(n: int, m: int, *, density: float = 0.01, rank: int = 64, seed: int = 0,
               rows: str = "vmat", var: str = "box", frac_lower_active: float = 0.30,
               frac_upper_active: float = 0.07, frac_rows_active: float = 0.10,
               name: str = "") -> QPData:
    """Planted-KKT convex QP.  See module docstring for the recipe."""
    rng = np.random.default_rng(seed)
    d, U, w = _draw_factors(rng, n, rank)

    # --- variable bounds -------------------------------------------------------
    xl = np.zeros(n)
    xu = rng.uniform(1.0, 2.0, size=n)
    if var == "mixed":
        kind = rng.choice(4, size=n, p=[0.85, 0.05, 0.05, 0.05])  # box, lower-only, upper-only, free
        xu[kind == 1] = np.inf
        xl[kind == 2] = -np.inf
        xl[kind == 3] = -np.inf
        xu[kind == 3] = np.inf
    elif var == "none":
        xl[:] = -np.inf
        xu[:] = np.inf
    elif var != "box":
        raise ValueError(var)
    has_l = np.isfinite(xl)
    has_u = np.isfinite(xu)
    # planted x*: at-lower / at-upper / interior
    state = rng.uniform(size=n)
    at_l = has_l & (state < frac_lower_active)
    at_u = has_u & ~at_l & (state >= 1.0 - frac_upper_active)
    frac = rng.uniform(0.2, 0.8, size=n)
    x = np.where(has_l & has_u, xl + frac * (np.where(has_u, xu, 0) - np.where(has_l, xl, 0)), 0.0)
    x = np.where(has_l & ~has_u, np.where(has_l, xl, 0) + 0.2 + frac, x)
    x = np.where(~has_l & has_u, np.where(has_u, xu, 0) - 0.2 - frac, x)
    x = np.where(~has_l & ~has_u, 2.0 * frac - 1.0, x)
    x = np.where(at_l, xl, x)
    x = np.where(at_u, xu, x)
    lam_lx = np.where(at_l, rng.uniform(0.5, 2.0, size=n), 0.0)
    lam_ux = np.where(at_u, rng.uniform(0.5, 2.0, size=n), 0.0)

    # --- linear constraints ---------------------------------------------------
    k = int(round(density * n)) if m > 0 else 0
    if m > 0:
        rowptr, cols, vals = _draw_sparse_rows(rng, m, n, k)
    else:
        rowptr, cols, vals = np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0)
    Ax = np.zeros(m)
    for i in range(m):
        s, e = rowptr[i], rowptr[i + 1]
        Ax[i] = math.fsum(vals[s:e] * x[cols[s:e]])
    fam = np.zeros(m, dtype=np.int64)  # 0 two-sided, 1 lower-only, 2 upper-only, 3 free
    if m > 0:
        if rows == "vmat":
            nl = int(round(VMAT_LOWER_FRACTION * m))
            perm = rng.permutation(m)
            fam[:] = 2
            fam[perm[:nl]] = 1
        elif rows == "mixed":
            fam = rng.choice(4, size=m, p=[0.25, 0.25, 0.40, 0.10])
        elif rows == "lower":
            fam[:] = 1
        elif rows == "upper":
            fam[:] = 2
        else:
            raise ValueError(rows)
    n_act = int(round(frac_rows_active * m))
    act_perm = rng.permutation(m)
    active = np.zeros(m, dtype=bool)
    active[act_perm[:n_act]] = True
    active &= fam != 3
    side = rng.uniform(size=m) < 0.5            # for two-sided rows: True = lower side active
    slack_l = rng.uniform(0.5, 1.5, size=m)
    slack_u = rng.uniform(0.5, 1.5, size=m)
    lam_r = rng.uniform(0.5, 2.0, size=m)
    l = np.full(m, -np.inf)
    u = np.full(m, np.inf)
    lam_lA = np.zeros(m)
    lam_uA = np.zeros(m)
    has_rl = (fam == 0) | (fam == 1)
    has_ru = (fam == 0) | (fam == 2)
    act_l = active & has_rl & ((fam == 1) | side)
    act_u = active & has_ru & ~act_l
    l = np.where(has_rl, np.where(act_l, Ax, Ax - slack_l), l)
    u = np.where(has_ru, np.where(act_u, Ax, Ax + slack_u), u)
    lam_lA = np.where(act_l, lam_r, 0.0)
    lam_uA = np.where(act_u, lam_r, 0.0)

    # --- linear term from stationarity (eq:perturbed_KKT first row at mu=0) -----
    Hx = hessian_matvec(d, U, w, x)
    ATy = np.zeros(n)
    yl = lam_lA - lam_uA
    if m > 0:
        rid = np.repeat(np.arange(m), np.diff(rowptr))
        np.add.at(ATy, cols, vals * yl[rid])
    g = -Hx + ATy + lam_lx - lam_ux
    f_star = 0.5 * math.fsum(x * Hx) + math.fsum(g * x)
    return QPData(n=n, m=m, d=d, U=U, w=w, g=g, A_rowptr=rowptr, A_col=cols, A_val=vals,
                  l=l, u=u, xl=xl, xu=xu, x_star=x, lam_lA=lam_lA, lam_uA=lam_uA,
                  lam_lx=lam_lx, lam_ux=lam_ux, f_star=f_star, name=name, seed=seed)


# --- BASELINE.json configs (SURVEY.md §8 "Config shorthand", §8(d) table) ---------------
CONFIGS = {
    # C1: tiny, dense full-rank SPD H, mixed families
    "C1": dict(n=50, m=20, density=0.3, rank=50, rows="mixed", var="mixed"),
    # C2: box-constrained only, low-rank+diag H, proton-like
    "C2": dict(n=5000, m=0, density=0.0, rank=100, rows="vmat", var="box"),
    # C3: patient-case-shaped, VMAT split
    "C3": dict(n=20000, m=5000, density=0.01, rank=64, rows="vmat", var="box"),
    # C5: large, row-sharded
    "C5": dict(n=100000, m=20000, density=0.01, rank=64, rows="vmat", var="box"),
}


def config(name: str, seed: int = 0, **overrides) -> QPData:
    kw = dict(CONFIGS[name])
    kw.update(overrides)
    return planted_qp(seed=seed, name=name, **kw)


def random_small_qp(n: int, m: int, seed: int, *, density: float = 0.6) -> QPData:
    """Non-planted small QP with a *random* optimum location (for the brute-force
    active-set pin).  H dense SPD, random A, random mixed finite/infinite bounds.
    The planted fields are NaN (unknown)."""
    rng = np.random.default_rng(10_000 + seed)
    r = n
    d = 0.5 + rng.uniform(size=n)
    U = rng.normal(size=(n, r)) / math.sqrt(n)
    w = np.ones(r)
    g = rng.normal(size=n) * 2.0
    k = max(1, int(round(density * n)))
    if m > 0:
        rowptr, cols, vals = _draw_sparse_rows(rng, m, n, k)
        vals = rng.normal(size=vals.size)
    else:
        rowptr, cols, vals = np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0)
    fam = rng.choice(4, size=m, p=[0.4, 0.25, 0.25, 0.10])   # two-sided, lower, upper, free
    vk = rng.choice(4, size=n, p=[0.6, 0.15, 0.15, 0.10])
    xlo = rng.uniform(-1.5, -0.2, size=n)
    xhi = rng.uniform(0.2, 1.5, size=n)
    xl = np.where((vk == 0) | (vk == 1), xlo, -np.inf)
    xu = np.where((vk == 0) | (vk == 2), xhi, np.inf)
    # x = 0 is strictly inside every variable bound; centre the row bounds on a point
    # xc inside the box so that a strictly feasible interior exists.
    xc = rng.uniform(-0.1, 0.1, size=n)
    Axc = np.zeros(m)
    for i in range(m):
        s, e = rowptr[i], rowptr[i + 1]
        Axc[i] = math.fsum(vals[s:e] * xc[cols[s:e]])
    l = np.where((fam == 0) | (fam == 1), Axc - rng.uniform(0.05, 1.5, size=m), -np.inf)
    u = np.where((fam == 0) | (fam == 2), Axc + rng.uniform(0.05, 1.5, size=m), np.inf)
    nan_n = np.full(n, np.nan)
    nan_m = np.full(m, np.nan)
    return QPData(n=n, m=m, d=d, U=U, w=w, g=g, A_rowptr=rowptr, A_col=cols, A_val=vals,
                  l=l, u=u, xl=xl, xu=xu, x_star=nan_n, lam_lA=nan_m, lam_uA=nan_m.copy(),
                  lam_lx=nan_n.copy(), lam_ux=nan_n.copy(), f_star=float("nan"),
                  name=f"random{n}x{m}", seed=seed)
