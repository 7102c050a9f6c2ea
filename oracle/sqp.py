"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (same rules as oracle/ipm.py: only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may use it).

Closed-loop SQP driver for  min f(x)  s.t.  l <= A x <= u,  xl <= x <= xu,
following PAPER.md §2.3 and SPEC.md's sqp module step by step:

  for k = 0, 1, ...:
    g_k = grad f(x_k)
    QP subproblem eq:qp_subproblem (reading R17: the standard 1/2 d^T B d + g^T d),
    written in x-space with y = x_k + d so that A and the bounds stay constant:
        min 1/2 y^T B_k y + (g_k - B_k x_k)^T y   s.t.  l <= A y <= u,  xl <= y <= xu
    solved EXACTLY by the oracle IPM (oracle.ipm.solve; optionally warm-started, R15);
    d = y - x_k;  stop when ||d||_inf <= tol_d * max(1, ||x_k||_inf)
    Armijo backtracking on f (reading R21: the constraints are linear and x_k, y are
    feasible, so every point of the segment is feasible and f itself is the merit
    function of SPEC's l1 merit with zero constraint violation):
        t = 1; while f(x_k + t d) > f(x_k) + c1 t g_k^T d: t <- t / 2
    x_{k+1} = x_k + t d;  s = t d;  y = grad f(x_{k+1}) - g_k
      (the Lagrangian's constraint term is linear, so grad_x L differences equal grad f
       differences)
    BFGS with Powell damping: theta = 1 if s^T y >= 0.2 s^T B s, else
        0.8 s^T B s / (s^T B s - s^T y);  y~ = theta y + (1 - theta) B s
    compact update (eq:bfgs_hessian P:240-245, "each iteration adds two terms"):
        B_{k+1} = B_k - (B s)(B s)^T / (s^T B s) + y~ y~^T / (y~^T s)
      i.e. append columns (B s, -1/(s^T B s)) and (y~, 1/(y~^T s)) to (U, w).

B_0 = diag(h0) ("initial guess for the Hessian (usually diagonal in our case)"; reading
R20 for the dose NLP: h0 = diag(D^T W D) + 1e-3, the Gauss-Newton diagonal of the quadratic
term).  Arithmetic fp64.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, List, Optional, Tuple

import numpy as np
import scipy.sparse as sp

from oracle.ipm import Options, Problem, solve, warm_start_point

H0_FLOOR = 1e-3


# ------------------------------------------------------------ the dose objective (R20)
def dose_objective(q, x: np.ndarray) -> float:
    """f(x) = sum_i 1/2 w_i (d_i - p_i)^2 + kappa_i / beta exp(beta (d_i - dmax_i)),  d = D x."""
    d = q.D_scipy() @ x
    return float(np.sum(0.5 * q.w * (d - q.p) ** 2 + q.kappa / q.beta * np.exp(q.beta * (d - q.dmax))))


def dose_gradient(q, x: np.ndarray) -> np.ndarray:
    """grad f = D^T e,  e_i = w_i (d_i - p_i) + kappa_i exp(beta (d_i - dmax_i))."""
    D = q.D_scipy()
    d = D @ x
    e = q.w * (d - q.p) + q.kappa * np.exp(q.beta * (d - q.dmax))
    return D.T @ e


def dose_h0(q) -> np.ndarray:
    """R20: h0_j = sum_i w_i D_ij^2 + 1e-3."""
    D = q.D_scipy()
    return np.asarray(D.multiply(D).T @ q.w).ravel() + H0_FLOOR


# ------------------------------------------------------------ compact BFGS operator
@dataclasses.dataclass
class Bfgs:
    h0: np.ndarray
    U: np.ndarray            # n x k
    w: np.ndarray            # k

    @staticmethod
    def diagonal(h0):
        return Bfgs(h0.copy(), np.zeros((h0.size, 0)), np.zeros(0))

    def apply(self, v):
        """B v = h0 o v + U (w o (U^T v))."""
        return self.h0 * v + self.U @ (self.w * (self.U.T @ v))

    def dense(self):
        B = (self.U * self.w) @ self.U.T
        B[np.diag_indices_from(B)] += self.h0
        return B

    def append(self, u, a, v, b):
        self.U = np.column_stack([self.U, u, v])
        self.w = np.concatenate([self.w, [a, b]])


def bfgs_update(B: Bfgs, s: np.ndarray, y: np.ndarray, powell: float = 0.2):
    """Powell-damped BFGS update in compact form.  Returns
    (updated, theta, Bs, a, ytilde, b); updated = False when s^T B s <= 0 or y~^T s <= 0."""
    Bs = B.apply(s)
    sBs = float(s @ Bs)
    sy = float(s @ y)
    if not sBs > 0.0:
        return False, 1.0, Bs, 0.0, y, 0.0
    theta = 1.0 if sy >= powell * sBs else (1.0 - powell) * sBs / (sBs - sy)
    yt = theta * y + (1.0 - theta) * Bs
    ys = float(yt @ s)
    if not ys > 0.0:
        return False, theta, Bs, 0.0, yt, 0.0
    a, b = -1.0 / sBs, 1.0 / ys
    B.append(Bs, a, yt, b)
    return True, theta, Bs, a, yt, b


# ------------------------------------------------------------ the driver
@dataclasses.dataclass
class SqpOptions:
    max_iter: int = 50
    tol_d: float = 1e-6
    armijo_c1: float = 1e-4
    max_backtrack: int = 30
    powell: float = 0.2
    warm_start: bool = False
    qp: Options = dataclasses.field(default_factory=Options)


@dataclasses.dataclass
class SqpResult:
    status: str
    x: np.ndarray
    f: float
    iters: int
    B: Bfgs
    trace: List[dict]


def sqp_solve(f: Callable, grad: Callable, h0: np.ndarray, A, l, u, xl, xu, x0,
              opt: Optional[SqpOptions] = None) -> SqpResult:
    opt = opt or SqpOptions()
    A = sp.csr_matrix(A)
    x = np.asarray(x0, dtype=np.float64).copy()
    B = Bfgs.diagonal(np.asarray(h0, dtype=np.float64))
    fx = f(x)
    g = grad(x)
    trace: List[dict] = []
    prev = None
    status = "not_converged"
    k = 0
    for k in range(opt.max_iter):
        H = B.dense()
        qp = Problem(H=H, g=g - B.apply(x), A=A, l=l, u=u, xl=xl, xu=xu)
        start = None
        if opt.warm_start and prev is not None:
            start = warm_start_point(qp, prev.it.x, prev.it.lam, opt.qp)
        res = solve(qp, opt.qp, start=start)
        if res.status != "converged":
            status = "qp_failed"
            break
        prev = res
        d = res.x - x
        dinf = float(np.max(np.abs(d))) if d.size else 0.0
        rec = dict(it=k, f=fx, d_inf=dinf, ipm_iters=res.iters)
        if dinf <= opt.tol_d * max(1.0, float(np.max(np.abs(x)))):
            trace.append(dict(rec, step=0.0, theta=1.0, updated=False))
            status = "converged"
            break
        gd = float(g @ d)
        t = 1.0
        ft = f(x + d)
        nb = 0
        while not (ft <= fx + opt.armijo_c1 * t * gd) and nb < opt.max_backtrack:
            t *= 0.5
            ft = f(x + t * d)
            nb += 1
        if not (ft <= fx + opt.armijo_c1 * t * gd):
            # no sufficient decrease (or a non-finite trial value): the step is not taken, since
            # the merit function must be nonincreasing across accepted steps
            trace.append(dict(rec, step=0.0, theta=1.0, updated=False))
            status = "line_search_failed"
            break
        s = t * d
        x = x + s
        g_new = grad(x)
        updated, theta, _, _, _, _ = bfgs_update(B, s, g_new - g, opt.powell)
        trace.append(dict(rec, step=t, theta=theta, updated=updated))
        fx, g = ft, g_new
    return SqpResult(status=status, x=x, f=fx, iters=k + 1, B=B, trace=trace)


def sqp_dose(q, opt: Optional[SqpOptions] = None) -> SqpResult:
    """The driver on a gen.dose_nlp.DoseNLP."""
    return sqp_solve(lambda x: dose_objective(q, x), lambda x: dose_gradient(q, x), dose_h0(q),
                     q.A_scipy(), q.l, q.u, q.xl, q.xu, q.x0, opt)
