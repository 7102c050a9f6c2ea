"""C4 input sequence: successive QP sub-problems with quasi-Newton (BFGS) Hessian updates.

Input plumbing only (no IPM arithmetic).  Follows SURVEY.md §8(d) "C4": start from a
planted QP (H0 = diag(d) + U W U^T); for k = 1..K-1 draw a step s_k ~ N(0, 1/n)
and a gradient difference y_k = G s_k from a hidden SPD G = diag + rank-32, so y^T s > 0 and
the BFGS update ("BFGS updates ... preserve definiteness")

    H_k = H_{k-1} + alpha u u^T + beta v v^T,   u = H_{k-1} s,  alpha = -1/(s^T H_{k-1} s),
                                                v = y,          beta  = 1/(y^T s)

keeps H_k SPD.  u is evaluated through the compact representation H0 + sum of rank-2 terms
(the matrix-free product of P:245), so no dense matrix is needed on the host.

Planted optimum of every QP ("x*_k is a planted random walk of x*_{k-1}
(5 % active-set flips), g_k from the planted formula"; `walk` = the flip fraction):
  * variables: `walk` of the active variable bounds are released (x*_j moves into the box,
    multiplier 0) and as many interior variables of two-sided boxes become active (at a bound,
    multiplier U(0.5, 2)); the other interior variables take a clipped random-walk step
    N(0, 0.02)·(xu - xl); the box itself is fixed;
  * rows: `walk` of the active rows are released (slack U(0.5, 1.5)) and as many inactive rows
    become active at one of their finite bounds; because x*_k moved, every row's bound is
    re-planted around A x*_k (active: l_i = A_i x*_k; inactive: A_i x*_k - slack_i) — the
    paper's sub-problems linearise the constraints at the current iterate, g(x_k) + grad g^T d
    <= 0, so their bounds shift with every QP.  Which bounds are finite never
    changes (ipm_set_bounds);
  * active multipliers drift by U(0.8, 1.25) per QP (strict complementarity kept), and
    g_k = -H_k x*_k + A^T (lam_lA - lam_uA) + lam_lx - lam_ux,
so x*_k is the exact optimum of QP k and f*_k = 1/2 x*^T H_k x* + g_k^T x* is known.
walk = 0 keeps x* and the bounds fixed (round-1 reading R22).  Every update (u, alpha, v, beta,
g_k, l_k, u_k) is handed identically to the GPU path (ipm_update_hessian_rank2 /
ipm_set_linear_term / ipm_set_bounds) and to the oracle (oracle.bfgs.rank2_update); this module
only draws them.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np


@dataclasses.dataclass
class Update:
    u: np.ndarray
    alpha: float
    v: np.ndarray
    beta: float
    g: np.ndarray
    f_star: float = float("nan")   # planted optimum value of this QP
    l: Optional[np.ndarray] = None  # row bounds of this QP (None: unchanged)
    ub: Optional[np.ndarray] = None
    x_star: Optional[np.ndarray] = None


def sqp_sequence(q, K: int, seed: int = 0, rank_G: int = 32, walk: float = 0.05) -> List[Update]:
    rng = np.random.default_rng(50_000 + seed)
    n, m = q.n, q.m
    dG = 1.0 + rng.uniform(size=n)
    VG = rng.normal(size=(n, rank_G)) / np.sqrt(n)
    terms = []                                  # (alpha, u, beta, v) of previous updates

    def Hmul(x):
        y = q.d * x + q.U @ (q.w * (q.U.T @ x))
        for a, u, b, v in terms:
            y = y + a * u * (u @ x) + b * v * (v @ x)
        return y

    out = []
    x = q.x_star.copy()
    lam = [q.lam_lA.copy(), q.lam_uA.copy(), q.lam_lx.copy(), q.lam_ux.copy()]
    rid = np.repeat(np.arange(m), np.diff(q.A_rowptr))
    has_rl, has_ru = np.isfinite(q.l), np.isfinite(q.u)
    has_xl, has_xu = np.isfinite(q.xl), np.isfinite(q.xu)
    box = has_xl & has_xu
    width = np.where(box, np.where(has_xu, q.xu, 0.0) - np.where(has_xl, q.xl, 0.0), 1.0)
    slack = np.where(has_rl | has_ru, rng.uniform(0.5, 1.5, size=m), 0.0)
    for _ in range(1, K):
        s = rng.normal(size=n) / np.sqrt(n)
        y = dG * s + VG @ (VG.T @ s)
        u = Hmul(s)
        alpha = -1.0 / float(s @ u)
        beta = 1.0 / float(y @ s)
        terms.append((alpha, u, beta, y))
        for a in lam:
            a *= np.where(a > 0.0, rng.uniform(0.8, 1.25, size=a.shape), 1.0)
        l_k = ub_k = None
        if walk > 0.0:
            # --- variables: release / activate `walk` of the active bounds, walk the interior
            at_l, at_u = lam[2] > 0.0, lam[3] > 0.0
            act = np.flatnonzero(at_l | at_u)
            nf = int(round(walk * act.size))
            rel = rng.choice(act, size=nf, replace=False) if nf else np.zeros(0, np.int64)
            inter = np.flatnonzero(~at_l & ~at_u & box)
            new = rng.choice(inter, size=min(nf, inter.size), replace=False) if nf else np.zeros(0, np.int64)
            step = rng.normal(size=n) * 0.02 * width
            moving = ~at_l & ~at_u
            lo = np.where(has_xl, q.xl, -np.inf) + 0.1 * width
            hi = np.where(has_xu, q.xu, np.inf) - 0.1 * width
            x = np.where(moving, np.clip(x + step, np.where(box, lo, -np.inf), np.where(box, hi, np.inf)), x)
            if rel.size:
                x[rel] = np.where(box[rel], np.where(has_xl[rel], q.xl[rel], 0.0)
                                  + rng.uniform(0.2, 0.8, size=rel.size) * width[rel], x[rel])
                lam[2][rel] = 0.0
                lam[3][rel] = 0.0
            if new.size:
                up_side = rng.uniform(size=new.size) < 0.07 / 0.37
                x[new] = np.where(up_side, q.xu[new], q.xl[new])
                lam[2][new] = np.where(up_side, 0.0, rng.uniform(0.5, 2.0, size=new.size))
                lam[3][new] = np.where(up_side, rng.uniform(0.5, 2.0, size=new.size), 0.0)
            # --- rows: release / activate `walk` of the active rows, re-plant every bound at A x*
            act_r = np.flatnonzero((lam[0] > 0.0) | (lam[1] > 0.0))
            nr = int(round(walk * act_r.size))
            if nr:
                rel_r = rng.choice(act_r, size=nr, replace=False)
                lam[0][rel_r] = 0.0
                lam[1][rel_r] = 0.0
                slack[rel_r] = rng.uniform(0.5, 1.5, size=nr)
                cand = np.flatnonzero((lam[0] == 0.0) & (lam[1] == 0.0) & (has_rl | has_ru))
                cand = np.setdiff1d(cand, rel_r)
                new_r = rng.choice(cand, size=min(nr, cand.size), replace=False)
                lower = np.where(has_rl[new_r] & has_ru[new_r], rng.uniform(size=new_r.size) < 0.5, has_rl[new_r])
                lam[0][new_r] = np.where(lower, rng.uniform(0.5, 2.0, size=new_r.size), 0.0)
                lam[1][new_r] = np.where(lower, 0.0, rng.uniform(0.5, 2.0, size=new_r.size))
            Ax = np.array([math.fsum(q.A_val[q.A_rowptr[i]:q.A_rowptr[i + 1]] * x[q.A_col[q.A_rowptr[i]:q.A_rowptr[i + 1]]])
                           for i in range(m)])
            act_l, act_u = lam[0] > 0.0, lam[1] > 0.0
            l_k = np.where(has_rl, np.where(act_l, Ax, Ax - slack), -np.inf)
            ub_k = np.where(has_ru, np.where(act_u, Ax, Ax + slack), np.inf)
        ATy = np.zeros(n)
        if m > 0:
            np.add.at(ATy, q.A_col, q.A_val * (lam[0] - lam[1])[rid])
        Hx = Hmul(x)
        g = -Hx + ATy + lam[2] - lam[3]
        f_star = 0.5 * math.fsum(x * Hx) + math.fsum(g * x)
        out.append(Update(u=u, alpha=alpha, v=y, beta=beta, g=g, f_star=f_star, l=l_k, ub=ub_k, x_star=x.copy()))
    return out
