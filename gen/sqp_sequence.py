"""C4 input sequence: successive QP sub-problems with quasi-Newton (BFGS) Hessian updates.

Input plumbing only (no IPM arithmetic).  Follows SURVEY.md §8(d) "C4": start from a
planted QP (H0 = diag(d) + U W U^T); for k = 1..K-1 draw a step s_k ~ N(0, 1/n)
and a gradient difference y_k = G s_k from a hidden SPD G = diag + rank-32, so y^T s > 0 and
the BFGS update ("BFGS updates ... preserve definiteness")

    H_k = H_{k-1} + alpha u u^T + beta v v^T,   u = H_{k-1} s,  alpha = -1/(s^T H_{k-1} s),
                                                v = y,          beta  = 1/(y^T s)

keeps H_k SPD.  u is evaluated through the compact representation H0 + sum of rank-2 terms
(the matrix-free product of P:245), so no dense matrix is needed on the host.  The linear
term drifts, g_k = g_{k-1} + 0.05 * N(0, 1), as the objective gradient does along an SQP run;
A and all bounds stay fixed (QP posed in x-space).  Every update (u, alpha, v, beta, g_k) is
handed identically to the GPU path (ipm_update_hessian_rank2 / ipm_set_linear_term) and to
the oracle (dense numpy update).
"""
from __future__ import annotations

import dataclasses
from typing import List

import numpy as np


@dataclasses.dataclass
class Update:
    u: np.ndarray
    alpha: float
    v: np.ndarray
    beta: float
    g: np.ndarray


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
    g = q.g.copy()
    for _ in range(1, K):
        s = rng.normal(size=n) / np.sqrt(n)
        y = dG * s + VG @ (VG.T @ s)
        u = Hmul(s)
        alpha = -1.0 / float(s @ u)
        beta = 1.0 / float(y @ s)
        terms.append((alpha, u, beta, y))
        g = g + 0.05 * rng.normal(size=n)
        out.append(Update(u=u, alpha=alpha, v=y, beta=beta, g=g.copy()))
    return out


def apply_dense(H: np.ndarray, up: Update) -> None:
    """In-place dense update used by the oracle side (numpy)."""
    H += up.alpha * np.outer(up.u, up.u)
    H += up.beta * np.outer(up.v, up.v)
