"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/ipm.py header).

Dense cross-checks of the Newton step at tiny sizes:

* ``full_newton_step``: assembles the Newton system eq:newton_system,
  extended by the variable-bound families exactly like the linear-constraint
  families (bounds separated out as in P:176), in ALL unknowns
  (dx, dlam_lA, dlam_uA, dlam_lx, dlam_ux, ds_lA, ds_uA, ds_lx, ds_ux) and solves it
  by dense LU (numpy.linalg.solve).  No elimination is performed, so it pins the
  block-row elimination + recovery of oracle/ipm.py.
* ``doubly_augmented_solve``: the paper's own symmetric system eq:2x2_augmented
  
        [ Q + 2 B^T D^-1 B   B^T ] [dx    ]   [ r1 + 2 B^T D^-1 r2 ]
        [ B                  D   ] [dlam_A] = [ r2                 ]
  solved densely; the condensed (Schur) solve must give the same (dx, dlam_A).
"""
from __future__ import annotations

import numpy as np

from .ipm import FAMILIES, Iterate, Problem


def full_newton_step(p: Problem, it: Iterate, r):
    n = p.n
    Cd = {f: p.C[f].toarray() for f in FAMILIES}     # tiny sizes: dense blocks
    sizes = [Cd[f].shape[0] for f in FAMILIES]
    nl = sum(sizes)
    N = n + 2 * nl
    Kf = np.zeros((N, N))
    rhs = np.zeros(N)
    # offsets: [dx | dlam_f ... | ds_f ...]
    off_l, off_s = {}, {}
    o = n
    for f, sz in zip(FAMILIES, sizes):
        off_l[f] = o
        o += sz
    for f, sz in zip(FAMILIES, sizes):
        off_s[f] = o
        o += sz
    # stationarity row: H dx - C_lA^T dlam_lA + C_uA^T dlam_uA - C_lx^T dlam_lx + C_ux^T dlam_ux = -r_H
    Kf[:n, :n] = p.H
    sign = {"lA": -1.0, "uA": 1.0, "lx": -1.0, "ux": 1.0}
    for f, sz in zip(FAMILIES, sizes):
        Kf[:n, off_l[f]:off_l[f] + sz] = sign[f] * Cd[f].T
    rhs[:n] = -r["H"]
    # primal rows: lower families  C dx - ds = -r ;  upper families  -C dx - ds = -r
    row = n
    for f, sz in zip(FAMILIES, sizes):
        sg = 1.0 if f in ("lA", "lx") else -1.0
        Kf[row:row + sz, :n] = sg * Cd[f]
        Kf[row:row + sz, off_s[f]:off_s[f] + sz] = -np.eye(sz)
        rhs[row:row + sz] = -r[f]
        row += sz
    # complementarity rows:  S dlam + Lam ds = -r_c
    for f, sz in zip(FAMILIES, sizes):
        Kf[row:row + sz, off_l[f]:off_l[f] + sz] = np.diag(it.s[f])
        Kf[row:row + sz, off_s[f]:off_s[f] + sz] = np.diag(it.lam[f])
        rhs[row:row + sz] = -r["c" + f]
        row += sz
    sol = np.linalg.solve(Kf, rhs)
    dx = sol[:n]
    dl = {f: sol[off_l[f]:off_l[f] + sz] for f, sz in zip(FAMILIES, sizes)}
    ds = {f: sol[off_s[f]:off_s[f] + sz] for f, sz in zip(FAMILIES, sizes)}
    return dx, ds, dl, (Kf, rhs, sol)


def doubly_augmented_solve(Q, B, D, r1, r2):
    B = B.toarray() if hasattr(B, "toarray") else B
    n = Q.shape[0]
    mA = B.shape[0]
    Dinv = 1.0 / D
    M = np.zeros((n + mA, n + mA))
    M[:n, :n] = Q + 2.0 * B.T @ (B * Dinv[:, None])
    M[:n, n:] = B.T
    M[n:, :n] = B
    M[n:, n:] = np.diag(D)
    rhs = np.concatenate([r1 + 2.0 * B.T @ (Dinv * r2), r2])
    sol = np.linalg.solve(M, rhs)
    return sol[:n], sol[n:], M
