"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/ipm.py header).

Textbook Jacobi-preconditioned conjugate gradients — the iterative solver the paper's GPU
path uses for every Newton system ("solve ... with the PCG method", Jacobi
preconditioner from the diagonal of the system) — written as the recurrence reads
(Saad, Iterative Methods for Sparse Linear Systems, Alg. 9.1):

    r0 = b - K x0,  z0 = M^-1 r0,  p0 = z0
    for j = 0, 1, ...:
        alpha_j = (r_j, z_j) / (K p_j, p_j)
        x_{j+1} = x_j + alpha_j p_j
        r_{j+1} = r_j - alpha_j K p_j
        z_{j+1} = M^-1 r_{j+1}
        beta_j  = (r_{j+1}, z_{j+1}) / (r_j, z_j)
        p_{j+1} = z_{j+1} + beta_j p_j

stopping when ||r_{j+1}||_2 <= max(rtol ||b||_2, atol) or after maxit iterations (reading R11:
x0 = 0).  ``K_apply`` is any callable v -> K v (tests pass oracle.kkt.condensed_apply, i.e.
K = H + Sigma_b + A^T Sigma_c A from its definition).  The oracle's IPM itself never calls this
(its directions come from Cholesky, oracle/ipm.py); this function is the reference for the GPU
PCG iterates (ipm_pcg_iterate) and is pinned in tests/test_oracle_pins.py against Cholesky
solves, exact-Jacobi and identity cases and CG's conjugacy / finite termination.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, List, Optional

import numpy as np


@dataclasses.dataclass
class PcgResult:
    x: np.ndarray
    r: np.ndarray
    z: np.ndarray
    p: np.ndarray           # the search direction used by the last iteration
    rho: float              # (r, z) after the last iteration
    pKp: float              # (K p, p) of the last iteration
    alpha: float            # alpha of the last iteration
    iters: int
    breakdown: bool
    directions: List[np.ndarray]


def pcg(K_apply: Callable[[np.ndarray], np.ndarray], Minv: np.ndarray, b: np.ndarray, rtol: float = 0.0,
        atol: float = 0.0, maxit: Optional[int] = None, keep_directions: bool = False) -> PcgResult:
    n = b.shape[0]
    maxit = 10 * n if maxit is None else maxit
    x = np.zeros(n)
    r = b.copy()
    z = Minv * r
    p = z.copy()
    rho = float(r @ z)
    tol = max(rtol * float(np.sqrt(b @ b)), atol)
    dirs = []
    pKp = alpha = 0.0
    j = 0
    breakdown = False
    while j < maxit:
        if keep_directions:
            dirs.append(p.copy())
        Kp = K_apply(p)
        pKp = float(p @ Kp)
        if not (pKp > 0.0) or not np.isfinite(pKp):
            breakdown = True
            break
        alpha = rho / pKp
        x = x + alpha * p
        r = r - alpha * Kp
        z = Minv * r
        rho_new = float(r @ z)
        j += 1
        if float(np.sqrt(r @ r)) <= tol or j >= maxit:
            rho = rho_new
            break
        beta = rho_new / rho
        rho = rho_new
        p = z + beta * p
    return PcgResult(x=x, r=r, z=z, p=p, rho=rho, pKp=pKp, alpha=alpha, iters=j, breakdown=breakdown,
                     directions=dirs)
