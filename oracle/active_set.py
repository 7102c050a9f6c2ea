"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/ipm.py header).

Brute-force active-set enumeration for tiny convex QPs (used to pin
oracle/ipm.py independently of any interior-point arithmetic).

Every row i of A and every variable j is in one of three states: inactive, at its
lower bound, at its upper bound (a state is only allowed when that bound is
finite).  For each candidate the equality-constrained QP

    min 1/2 x^T H x + g^T x   s.t.  c_k^T x = b_k  (k active)

is solved through its dense KKT system  [H  -C^T; C 0] [x; nu] = [-g; b].
The candidate is accepted when x is feasible (tolerance 1e-9) and the multipliers
have the right sign (nu_k >= 0 for lower-active, nu_k <= 0 for upper-active,
tolerance 1e-9).  For strictly convex H the accepted point is the unique minimiser;
the lowest objective over accepted candidates is returned.
"""
from __future__ import annotations

import itertools
import math

import numpy as np


def solve_active_set(H, g, A, l, u, xl, xu, tol=1e-9):
    n = H.shape[0]
    m = A.shape[0]
    rows = [np.asarray(A[i]) for i in range(m)] + [np.eye(n)[j] for j in range(n)]
    lo = list(l) + list(xl)
    hi = list(u) + list(xu)
    choices = []
    for k in range(m + n):
        c = [0]
        if math.isfinite(lo[k]):
            c.append(1)
        if math.isfinite(hi[k]):
            c.append(2)
        choices.append(c)
    best = None
    for state in itertools.product(*choices):
        act = [k for k in range(m + n) if state[k] != 0]
        C = np.array([rows[k] for k in act]).reshape(len(act), n)
        b = np.array([lo[k] if state[k] == 1 else hi[k] for k in act])
        na = len(act)
        KKT = np.zeros((n + na, n + na))
        KKT[:n, :n] = H
        KKT[:n, n:] = -C.T
        KKT[n:, :n] = C
        rhs = np.concatenate([-g, b])
        try:
            sol = np.linalg.solve(KKT, rhs)
        except np.linalg.LinAlgError:
            continue
        if not np.all(np.isfinite(sol)):
            continue
        x = sol[:n]
        nu = sol[n:]
        ok = True
        for k in range(m + n):
            v = float(rows[k] @ x)
            if math.isfinite(lo[k]) and v < lo[k] - tol:
                ok = False
                break
            if math.isfinite(hi[k]) and v > hi[k] + tol:
                ok = False
                break
        if not ok:
            continue
        for idx, k in enumerate(act):
            if state[k] == 1 and nu[idx] < -tol:
                ok = False
            if state[k] == 2 and nu[idx] > tol:
                ok = False
        if not ok:
            continue
        f = 0.5 * float(x @ H @ x) + float(g @ x)
        if best is None or f < best[1] - 1e-12:
            best = (x, f, state)
    return best
