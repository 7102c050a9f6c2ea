"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product path
(``paper_2405_03584_b200``) never imports, links or executes anything under
``oracle/``, and this module imports nothing from it.

A plain, slow, obviously correct primal-dual interior point method for

    min 1/2 x^T H x + g^T x   s.t.  l <= A x <= u,  xl <= x <= xu

(eq:qp; variable bounds split out as in P:176), following Algorithm 1
 step by step, with EXACT Newton directions: every search direction
comes from a dense Cholesky factorisation of the condensed matrix
Q + B^T D^-1 B (Schur complement of the reduced system eq:2x2_reduced, P:176-212;
SURVEY.md decision D1), never from an iteration.  Arithmetic is IEEE fp64
(the paper states no precision).

Layout: every bound family is stored *compacted* over its finite entries (the
index sets I_l, I_u, J_l, J_u below), as in the paper's block matrices — the GPU
path uses masked full-length vectors instead, so the two share no layout.

Readings of the paper (DESIGN.md §3 lists them all):
  R1  r_u = u - A x - s_u (P:71/83/94 disagree; the Newton row (-A, -I) of
      eq:newton_system, fixes this sign).
  R3  r_c = lambda o s - mu e  ("e" of P:128).
  R4  ||r|| in Alg. 1 line 10 is the absolute inf-norm over all nine families.
  R5  initial point: SPEC S:290 rule.
  R6  tau = 0.995, mu_tol = 1e-8, N = 100.
  R7  one alpha_x for x and all slacks, one alpha_lambda for all multipliers
      (Alg. 1 lines 5-7).
  R8  mu changes at most once per iteration; each iteration starts with a solve.
  R9  r_c is recomputed with the new mu after mu <- mu/10.
  R10 infinite bounds carry no slack / multiplier / residual.
  R13 with no finite bound at all, mu = mu_tol and one exact Newton step solves
      the problem (x = -H^-1 g).
  R15 warm start (C4): see ``warm_start_point``.
  R18 Mehrotra predictor-corrector (option): standard formulas, see ``_mehrotra``.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

FAMILIES = ("lA", "uA", "lx", "ux")


@dataclasses.dataclass
class Options:
    mu_tol: float = 1e-8
    mu0_scale: float = 0.1
    mu_divisor: float = 10.0
    tau: float = 0.995
    max_iter: int = 100
    predictor_corrector: bool = False
    warm_shift: float = 0.1          # R15 theta (R15: sweep 1e-3 .. 1 on the C4 sequence)


@dataclasses.dataclass
class Problem:
    """The QP as the oracle sees it: dense H, sparse A (scipy CSR; a library container,
    no arithmetic of the method), and the four bound families in compact form."""
    H: np.ndarray
    g: np.ndarray
    A: "sp.csr_matrix"       # m x n
    l: np.ndarray
    u: np.ndarray
    xl: np.ndarray
    xu: np.ndarray

    def __post_init__(self):
        self.A = sp.csr_matrix(self.A)
        self.n = self.H.shape[0]
        self.m = self.A.shape[0]
        # index sets of finite bounds (R10)
        self.I_l = np.flatnonzero(np.isfinite(self.l))
        self.I_u = np.flatnonzero(np.isfinite(self.u))
        self.J_l = np.flatnonzero(np.isfinite(self.xl))
        self.J_u = np.flatnonzero(np.isfinite(self.xu))
        # constraint matrix of each family: rows of A, or rows of the identity
        I = sp.identity(self.n, format="csr")
        self.C = {"lA": self.A[self.I_l], "uA": self.A[self.I_u],
                  "lx": I[self.J_l], "ux": I[self.J_u]}
        self.bound = {"lA": self.l[self.I_l], "uA": self.u[self.I_u],
                      "lx": self.xl[self.J_l], "ux": self.xu[self.J_u]}
        self.n_bounds = sum(self.C[f].shape[0] for f in FAMILIES)

    @staticmethod
    def from_data(q, H: Optional[np.ndarray] = None) -> "Problem":
        return Problem(H=q.H if H is None else H, g=q.g.copy(), A=q.A_scipy(), l=q.l.copy(),
                       u=q.u.copy(), xl=q.xl.copy(), xu=q.xu.copy())

    def A_dense(self) -> np.ndarray:
        return self.A.toarray()

    def objective(self, x):
        return 0.5 * float(x @ (self.H @ x)) + float(self.g @ x)


@dataclasses.dataclass
class Iterate:
    x: np.ndarray
    s: Dict[str, np.ndarray]      # compact per family
    lam: Dict[str, np.ndarray]
    mu: float

    def copy(self):
        return Iterate(self.x.copy(), {k: v.copy() for k, v in self.s.items()},
                       {k: v.copy() for k, v in self.lam.items()}, self.mu)


# ------------------------------------------------------------------ Eq. 2 / eq:perturbed_KKT
def primal_value(p: Problem, f: str, x: np.ndarray) -> np.ndarray:
    """The quantity whose distance to the bound is the slack: s_lA = A x - l,
    s_uA = u - A x, s_lx = x - xl, s_ux = xu - x (slack reformulation P:66-75, R1)."""
    Cx = p.C[f] @ x
    return Cx - p.bound[f] if f in ("lA", "lx") else p.bound[f] - Cx


def residuals(p: Problem, it: Iterate, mu: Optional[float] = None) -> Dict[str, np.ndarray]:
    """eq:perturbed_KKT extended by the variable-bound families:

      r_H  = H x + g - A^T lam_lA + A^T lam_uA - lam_lx + lam_ux
      r_lA = A x - s_lA - l          r_uA = u - A x - s_uA      (R1)
      r_lx = x - s_lx - xl           r_ux = xu - x - s_ux
      r_c,f = lam_f o s_f - mu                                   (R3)
    """
    mu = it.mu if mu is None else mu
    r = {}
    rH = p.H @ it.x + p.g
    rH -= p.C["lA"].T @ it.lam["lA"]
    rH += p.C["uA"].T @ it.lam["uA"]
    rH -= p.C["lx"].T @ it.lam["lx"]
    rH += p.C["ux"].T @ it.lam["ux"]
    r["H"] = rH
    for f in FAMILIES:
        r[f] = primal_value(p, f, it.x) - it.s[f]
        r["c" + f] = it.lam[f] * it.s[f] - mu
    return r


def kkt_norm(r: Dict[str, np.ndarray]) -> float:
    """R4: absolute inf-norm over all nine residual families."""
    return max((float(np.max(np.abs(v))) for v in r.values() if v.size), default=0.0)


# ------------------------------------------------------------------ initial point (R5)
def initial_point(p: Problem, opt: Options) -> Iterate:
    """x0 = projection of 0 onto [xl+delta, xu-delta], delta=min(1,(xu-xl)/4)
    for two-sided bounds, xl+1 / xu-1 one-sided, 0 free; slacks max(gap, 1);
    multipliers 1; mu0 = mu0_scale * sum(lam s) / (#bounds)."""
    x = np.zeros(p.n)
    for j in range(p.n):
        lo, hi = p.xl[j], p.xu[j]
        if math.isfinite(lo) and math.isfinite(hi):
            delta = min(1.0, (hi - lo) / 4.0)
            x[j] = min(max(0.0, lo + delta), hi - delta)
        elif math.isfinite(lo):
            x[j] = max(0.0, lo + 1.0)
        elif math.isfinite(hi):
            x[j] = min(0.0, hi - 1.0)
    s = {f: np.maximum(primal_value(p, f, x), 1.0) for f in FAMILIES}
    lam = {f: np.ones_like(s[f]) for f in FAMILIES}
    if p.n_bounds == 0:
        mu = opt.mu_tol                                     # R13
    else:
        mu = opt.mu0_scale * sum(float(lam[f] @ s[f]) for f in FAMILIES) / p.n_bounds
    return Iterate(x, s, lam, mu)


def warm_start_point(p: Problem, x_prev: np.ndarray, lam_prev: Dict[str, np.ndarray],
                     opt: Options) -> Iterate:
    """R15 (SURVEY.md §8(c) point 15; the paper only names warm starting):
    x0 = x_prev projected into the box with margin min(theta, (xu-xl)/4);
    s = max(gap(x0), theta); lam = max(lam_prev, theta); mu0 = mu0_scale*mean(lam s)."""
    th = opt.warm_shift
    x = x_prev.copy()
    for j in range(p.n):
        lo, hi = p.xl[j], p.xu[j]
        mlo = min(th, (hi - lo) / 4.0) if (math.isfinite(lo) and math.isfinite(hi)) else th
        if math.isfinite(lo):
            x[j] = max(x[j], lo + mlo)
        if math.isfinite(hi):
            x[j] = min(x[j], hi - mlo)
    s = {f: np.maximum(primal_value(p, f, x), th) for f in FAMILIES}
    lam = {f: np.maximum(lam_prev[f], th) for f in FAMILIES}
    if p.n_bounds == 0:
        mu = opt.mu_tol
    else:
        mu = opt.mu0_scale * sum(float(lam[f] @ s[f]) for f in FAMILIES) / p.n_bounds
    return Iterate(x, s, lam, mu)


# ------------------------------------------------------------------ eq:2x2_reduced blocks
def reduced_system(p: Problem, it: Iterate, r: Dict[str, np.ndarray]):
    """Blocks of eq:2x2_reduced:

        [ Q  -B^T ] [dx     ]   [r1]      Q = H + S_lx^-1 Lam_lx + S_ux^-1 Lam_ux
        [ B   D   ] [dlam_A ] = [r2],     B = [A_l; -A_u],  D = diag(Lam_A^-1 S_A)

    r1 and r2 are what block-row elimination of the Newton system (eq:newton_system,
    P:102-128, extended by the variable-bound rows) leaves:
        r1 = -r_H - S_lx^-1 (r_c,lx + Lam_lx r_lx) + S_ux^-1 (r_c,ux + Lam_ux r_ux)
        r2 = ( -r_lA - Lam_lA^-1 r_c,lA ;  -r_uA - Lam_uA^-1 r_c,uA ).
    """
    s, lam = it.s, it.lam
    # S_lx^-1 Lam_lx + S_ux^-1 Lam_ux is diagonal: C_f^T diag(v) C_f = diag(C_f^T v) for the
    # identity-row families, so Q = H + diag(sigma_b).
    sigma_b = p.C["lx"].T @ (lam["lx"] / s["lx"]) + p.C["ux"].T @ (lam["ux"] / s["ux"])
    Q = p.H.copy()
    Q[np.diag_indices(p.n)] += sigma_b
    B = sp.vstack([p.C["lA"], -p.C["uA"]], format="csr")
    D = np.concatenate([s["lA"] / lam["lA"], s["uA"] / lam["uA"]])
    r1 = -r["H"].copy()
    r1 -= p.C["lx"].T @ ((r["clx"] + lam["lx"] * r["lx"]) / s["lx"])
    r1 += p.C["ux"].T @ ((r["cux"] + lam["ux"] * r["ux"]) / s["ux"])
    r2 = np.concatenate([-r["lA"] - r["clA"] / lam["lA"], -r["uA"] - r["cuA"] / lam["uA"]])
    return Q, B, D, r1, r2


def condensed_solve(Q, B, D, r1, r2):
    """Exact solve of eq:2x2_reduced through its Schur complement (D1):
       (Q + B^T D^-1 B) dx = r1 + B^T D^-1 r2 ;  dlam_A = D^-1 (r2 - B dx).
    The matrix is SPD (Q SPD, D > 0); a Cholesky failure is an error."""
    K = Q + (B.T @ sp.diags(1.0 / D) @ B).toarray()
    rhs = r1 + B.T @ (r2 / D)
    c = sla.cho_factor(K, lower=True, check_finite=True)
    dx = sla.cho_solve(c, rhs)
    dlamA = (r2 - B @ dx) / D
    return dx, dlamA, (K, rhs, c)


def recover_step(p: Problem, it: Iterate, r, dx, dlamA):
    """Alg. 1 line 3 "Assemble full search direction" — back-substitution of the
    eliminated rows of eq:newton_system:
      ds_lA = A dx + r_lA      ds_uA = -A dx + r_uA     (rows 2-3)
      ds_lx = dx + r_lx        ds_ux = -dx + r_ux
      dlam_f = -S_f^-1 (r_c,f + Lam_f ds_f)  for the bound families (rows 4-5)."""
    nl = p.I_l.size
    ds, dl = {}, {}
    ds["lA"] = p.C["lA"] @ dx + r["lA"]
    ds["uA"] = -(p.C["uA"] @ dx) + r["uA"]
    ds["lx"] = p.C["lx"] @ dx + r["lx"]
    ds["ux"] = -(p.C["ux"] @ dx) + r["ux"]
    dl["lA"] = dlamA[:nl]
    dl["uA"] = dlamA[nl:]
    for f in ("lx", "ux"):
        dl[f] = -(r["c" + f] + it.lam[f] * ds[f]) / it.s[f]
    return ds, dl


def max_step(v: Dict[str, np.ndarray], dv: Dict[str, np.ndarray], tau: float) -> float:
    """Fraction to the boundary (Alg. 1 line 4):
       alpha = min(1, tau * min{ -v_i / dv_i : dv_i < 0 })   (empty set -> 1)."""
    a = 1.0
    for f in FAMILIES:
        neg = dv[f] < 0
        if np.any(neg):
            a = min(a, tau * float(np.min(-v[f][neg] / dv[f][neg])))
    return a


def newton_direction(p: Problem, it: Iterate, r):
    Q, B, D, r1, r2 = reduced_system(p, it, r)
    dx, dlamA, _ = condensed_solve(Q, B, D, r1, r2)
    ds, dl = recover_step(p, it, r, dx, dlamA)
    return dx, ds, dl


# ------------------------------------------------------------------ Mehrotra option (R18)
def _mehrotra(p: Problem, it: Iterate, opt: Options):
    """Predictor-corrector (north_star; not in the paper, SPEC S:343 non-goal) —
    R18: affine direction with r_c = lam o s (mu = 0); alpha_aff at tau = 1;
    mu_aff = sum (lam + a_l dlam)(s + a_x ds) / N_b; sigma = (mu_aff / mu_cur)^3
    with mu_cur = sum(lam s)/N_b; corrector r_c = lam o s + dlam_aff o ds_aff - sigma mu_cur.
    Both solves use the same Q, B, D (same factor)."""
    r_aff = residuals(p, it, mu=0.0)
    Q, B, D, r1, r2 = reduced_system(p, it, r_aff)
    dx, dlamA, (K, rhs, c) = condensed_solve(Q, B, D, r1, r2)
    ds_a, dl_a = recover_step(p, it, r_aff, dx, dlamA)
    ax = max_step(it.s, ds_a, 1.0)
    al = max_step(it.lam, dl_a, 1.0)
    nb = p.n_bounds
    mu_cur = sum(float(it.lam[f] @ it.s[f]) for f in FAMILIES) / nb
    mu_aff = sum(float((it.lam[f] + al * dl_a[f]) @ (it.s[f] + ax * ds_a[f])) for f in FAMILIES) / nb
    sigma = (mu_aff / mu_cur) ** 3
    r_cor = dict(r_aff)
    for f in FAMILIES:
        r_cor["c" + f] = it.lam[f] * it.s[f] + dl_a[f] * ds_a[f] - sigma * mu_cur
    Q, B, D, r1, r2 = reduced_system(p, it, r_cor)
    rhs2 = r1 + B.T @ (r2 / D)
    dx2 = sla.cho_solve(c, rhs2)
    dlamA2 = (r2 - B @ dx2) / D
    ds, dl = recover_step(p, it, r_cor, dx2, dlamA2)
    return dx2, ds, dl, sigma * mu_cur


# ------------------------------------------------------------------ Algorithm 1
@dataclasses.dataclass
class Result:
    status: str              # "converged" | "not_converged"
    x: np.ndarray
    it: Iterate
    iters: int
    obj: float
    kkt_inf: float
    trace: List[dict]


def solve(p: Problem, opt: Optional[Options] = None, start: Optional[Iterate] = None) -> Result:
    """Algorithm 1 with exact (Cholesky) Newton directions.

    for i = 1..N:
        direction (line 2-3), alpha_x, alpha_lambda (line 4), update x, lambda, s
        (lines 5-7), residuals (line 9);
        if ||r|| < mu: if mu <= mu_tol: return; mu <- mu/10      (lines 10-15)
    Mehrotra mode (R18): direction from ``_mehrotra``; converged when
    max(||r_H||, ||primal||, max lam o s) < mu_tol.
    """
    opt = opt or Options()
    it = (start or initial_point(p, opt)).copy()
    trace = []
    r = residuals(p, it)
    status = "not_converged"
    k = 0
    for k in range(1, opt.max_iter + 1):
        if opt.predictor_corrector and p.n_bounds > 0:
            dx, ds, dl, _ = _mehrotra(p, it, opt)
        else:
            dx, ds, dl = newton_direction(p, it, r)
        ax = max_step(it.s, ds, opt.tau)
        al = max_step(it.lam, dl, opt.tau)
        it.x = it.x + ax * dx
        for f in FAMILIES:
            it.s[f] = it.s[f] + ax * ds[f]
            it.lam[f] = it.lam[f] + al * dl[f]
        if opt.predictor_corrector and p.n_bounds > 0:
            nb = p.n_bounds
            it.mu = sum(float(it.lam[f] @ it.s[f]) for f in FAMILIES) / nb
            r = residuals(p, it, mu=0.0)
            prim = max([float(np.max(np.abs(r[f]))) for f in FAMILIES if r[f].size] + [0.0])
            comp = max([float(np.max(it.lam[f] * it.s[f])) for f in FAMILIES if r[f].size] + [0.0])
            nrm = max(float(np.max(np.abs(r["H"]))), prim, comp)
            trace.append(dict(it=k, mu=it.mu, kkt=nrm, ax=ax, al=al))
            if nrm < opt.mu_tol:
                status = "converged"
                break
            continue
        r = residuals(p, it)
        nrm = kkt_norm(r)
        trace.append(dict(it=k, mu=it.mu, kkt=nrm, ax=ax, al=al))
        if nrm < it.mu:
            if it.mu <= opt.mu_tol:
                status = "converged"
                break
            it.mu = it.mu / opt.mu_divisor
            r = residuals(p, it)                                  # R9
    r_final = residuals(p, it)
    return Result(status=status, x=it.x.copy(), it=it, iters=k, obj=p.objective(it.x),
                  kkt_inf=kkt_norm(r_final), trace=trace)


def full_multipliers(p: Problem, it: Iterate):
    """Expand compact multipliers to full-length (zero where the bound is absent)."""
    out = {"lA": np.zeros(p.m), "uA": np.zeros(p.m), "lx": np.zeros(p.n), "ux": np.zeros(p.n)}
    out["lA"][p.I_l] = it.lam["lA"]
    out["uA"][p.I_u] = it.lam["uA"]
    out["lx"][p.J_l] = it.lam["lx"]
    out["ux"][p.J_u] = it.lam["ux"]
    return out
