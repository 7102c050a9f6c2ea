"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/ipm.py header).

The dense quasi-Newton Hessian update of the SQP sequence:

    H_k = H_{k-1} + alpha u u^T + beta v v^T,
    u = H_{k-1} s,  alpha = -1 / (s^T H_{k-1} s),  v = y,  beta = 1 / (y^T s)

— the BFGS update the paper's SQP applies between QP sub-problems ("BFGS updates ... preserve
definiteness"; its compact form H0 + U W U^T appends the two columns u, v).
Written out as the definition reads: two outer products added to a dense copy.  Pinned in
tests/test_oracle_pins.py by the secant equation H_k s = y, SPEC's hand case (H = I,
s = e1, y = 2 e1 gives diag(2, 1, ...)) and preserved positive definiteness.
"""
from __future__ import annotations

import numpy as np


def rank2_update(H: np.ndarray, u: np.ndarray, alpha: float, v: np.ndarray, beta: float) -> np.ndarray:
    """H + alpha u u^T + beta v v^T (a new array)."""
    return H + alpha * np.outer(u, u) + beta * np.outer(v, v)


def bfgs_terms(H: np.ndarray, s: np.ndarray, y: np.ndarray):
    """(u, alpha, v, beta) of the BFGS update of H for the pair (s, y)."""
    u = H @ s
    return u, -1.0 / float(s @ u), y, 1.0 / float(y @ s)
