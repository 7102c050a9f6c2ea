"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/ipm.py header).

Reference values for the operator-level test hooks of the C ABI, written from the
definitions, plus a KKT optimality certificate.

* ``condensed_matrix``  K = H + diag(sig_b) + A^T diag(sig_c) A   — the north_star
  operator; it is Q + B^T D^-1 B of eq:2x2_reduced with
  sig_b = S_lx^-1 Lam_lx + S_ux^-1 Lam_ux and sig_c = Lam_lA S_lA^-1 + Lam_uA S_uA^-1
  (B = [A_l; -A_u] so B^T D^-1 B = A^T diag(sig_c) A).
* ``condensed_apply`` K v evaluated in the order the definition reads (dense H,
  dense A), in fp64 or, when asked, in numpy longdouble.
* ``jacobi_diag``  diag(K): diag(H) + sig_b + sum_i sig_c,i A_ij^2.
* ``kkt_certificate``  stationarity / feasibility / sign / complementarity of a
  returned point (SURVEY.md §8(c) "KKT certificates").
"""
from __future__ import annotations

import numpy as np


def condensed_matrix(H, A, sig_b, sig_c):
    return H + np.diag(sig_b) + A.T @ (A * sig_c[:, None])


def condensed_apply(H, A, sig_b, sig_c, v, dtype=np.float64):
    H = np.asarray(H, dtype=dtype)
    A = np.asarray(A, dtype=dtype)
    v = np.asarray(v, dtype=dtype)
    t = np.asarray(sig_c, dtype=dtype) * (A @ v)
    return H @ v + np.asarray(sig_b, dtype=dtype) * v + A.T @ t


def condensed_apply_rows(H_rows, rows, A, sig_b, sig_c, v):
    """K v restricted to the given rows (for sampled parity at full size).
    H_rows: H[rows, :]; A: scipy CSR."""
    t = sig_c * (A @ v)
    ATt = A.T @ t
    return H_rows @ v + sig_b[rows] * v[rows] + ATt[rows]


def jacobi_diag(H, A, sig_b, sig_c):
    return np.diag(H) + sig_b + (A * A).T @ sig_c


def kkt_certificate(H, g, A, l, u, xl, xu, x, lam_lA, lam_uA, lam_lx, lam_ux):
    """Return the inf-norms of: stationarity H x + g - A^T(lam_lA - lam_uA) - lam_lx + lam_ux,
    primal infeasibility, the most negative multiplier, and complementarity
    max |lam * gap| over finite bounds."""
    stat = H @ x + g - A.T @ (lam_lA - lam_uA) - lam_lx + lam_ux
    Ax = A @ x
    inf = 0.0
    comp = 0.0
    for v, lo, hi, ll, lu in ((Ax, l, u, lam_lA, lam_uA), (x, xl, xu, lam_lx, lam_ux)):
        fl = np.isfinite(lo)
        fu = np.isfinite(hi)
        if fl.any():
            inf = max(inf, float(np.max(np.maximum(lo[fl] - v[fl], 0.0))))
            comp = max(comp, float(np.max(np.abs(ll[fl] * (v[fl] - lo[fl])))))
        if fu.any():
            inf = max(inf, float(np.max(np.maximum(v[fu] - hi[fu], 0.0))))
            comp = max(comp, float(np.max(np.abs(lu[fu] * (hi[fu] - v[fu])))))
    neg = min(0.0, float(min(lam_lA.min(initial=0.0), lam_uA.min(initial=0.0),
                             lam_lx.min(initial=0.0), lam_ux.min(initial=0.0))))
    return dict(stationarity=float(np.max(np.abs(stat))) if stat.size else 0.0,
                infeasibility=inf, min_multiplier=neg, complementarity=comp)
