"""C4 input sequence: successive QP sub-problems with quasi-Newton (BFGS) Hessian updates.

Input plumbing only (no IPM arithmetic).  Follows SURVEY.md §8(d) "C4": start from a
planted QP (H0 = diag(d) + U W U^T); for k = 1..K-1 draw a step s_k ~ N(0, 1/n)
and a gradient difference y_k = G s_k from a hidden SPD G = diag + rank-32, so y^T s > 0 and
the BFGS update ("BFGS updates ... preserve definiteness")

    H_k = H_{k-1} + alpha u u^T + beta v v^T,   u = H_{k-1} s,  alpha = -1/(s^T H_{k-1} s),
                                                v = y,          beta  = 1/(y^T s)

keeps H_k SPD.  u is evaluated through the compact representation H0 + sum of rank-2 terms
(the matrix-free product of P:245), so no dense matrix is needed on the host.

The linear term keeps every QP of the sequence planted ("g_k from the planted
formula"): A and all bounds stay fixed (QP posed in x-space), so the planted point x* and its
active set are kept — moving x* would break the active rows l_i = A_i x* of the fixed bounds —
while the multipliers of the active constraints drift, lam_k = lam_{k-1} * U(0.8, 1.25) (still
strictly positive: strict complementarity), and
    g_k = -H_k x* + A^T (lam_lA - lam_uA) + lam_lx - lam_ux,
so x* stays the exact optimum of QP k and f*_k = 1/2 x*^T H_k x* + g_k^T x* is known.  (An
earlier version let g drift by 0.05 N(0, 1) per QP; that left the optimum unplanted and nearly
degenerate, and QP 1 at C3 size took 37 IPM / 4.1 M PCG iterations instead of 18 / 0.2 M.)
Every update (u, alpha, v, beta, g_k) is handed identically to the GPU path
(ipm_update_hessian_rank2 / ipm_set_linear_term) and to the oracle (oracle.bfgs.rank2_update);
this module only draws them.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List

import numpy as np


@dataclasses.dataclass
class Update:
    u: np.ndarray
    alpha: float
    v: np.ndarray
    beta: float
    g: np.ndarray
    f_star: float = float("nan")   # planted optimum value of this QP


def sqp_sequence(q, K: int, seed: int = 0, rank_G: int = 32) -> List[Update]:
    rng = np.random.default_rng(50_000 + seed)
    n = q.n
    dG = 1.0 + rng.uniform(size=n)
    VG = rng.normal(size=(n, rank_G)) / np.sqrt(n)
    terms = []                                  # (alpha, u, beta, v) of previous updates

    def Hmul(x):
        y = q.d * x + q.U @ (q.w * (q.U.T @ x))
        for a, u, b, v in terms:
            y = y + a * u * (u @ x) + b * v * (v @ x)
        return y

    out = []
    x = q.x_star
    lam = [q.lam_lA.copy(), q.lam_uA.copy(), q.lam_lx.copy(), q.lam_ux.copy()]
    rid = np.repeat(np.arange(q.m), np.diff(q.A_rowptr))
    for _ in range(1, K):
        s = rng.normal(size=n) / np.sqrt(n)
        y = dG * s + VG @ (VG.T @ s)
        u = Hmul(s)
        alpha = -1.0 / float(s @ u)
        beta = 1.0 / float(y @ s)
        terms.append((alpha, u, beta, y))
        for a in lam:
            a *= np.where(a > 0.0, rng.uniform(0.8, 1.25, size=a.shape), 1.0)
        ATy = np.zeros(n)
        if q.m > 0:
            np.add.at(ATy, q.A_col, q.A_val * (lam[0] - lam[1])[rid])
        Hx = Hmul(x)
        g = -Hx + ATy + lam[2] - lam[3]
        f_star = 0.5 * math.fsum(x * Hx) + math.fsum(g * x)
        out.append(Update(u=u, alpha=alpha, v=y, beta=beta, g=g, f_star=f_star))
    return out

