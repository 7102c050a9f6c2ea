"""Move generator output (gen/planted.py) onto a CUDA device as the tensors the
C ABI borrows.  Input plumbing only: no arithmetic of the method lives here.

H is built ON THE DEVICE from its exact dyadic factors, H = diag(d) + U diag(w) U^T
(see gen/planted.py: every entry is exactly representable, so the fp64 GEMM gives the
bit-identical matrix numpy builds; tests/test_gpu_parity.py checks this).  The leading
dimension is padded to an even number so rows are 16-byte aligned.
"""
from __future__ import annotations

import numpy as np
import torch


def device_hessian(q, device, ldh=None, rows=None):
    n = q.n
    ldh = ldh or (n + (n & 1))
    r0, r1 = (0, n) if rows is None else rows
    U = torch.from_numpy(q.U).to(device)
    Uw = U * torch.from_numpy(q.w).to(device)
    H = torch.zeros((r1 - r0, ldh), dtype=torch.float64, device=device)
    step = 4096
    for a in range(r0, r1, step):
        b = min(r1, a + step)
        H[a - r0:b - r0, :n] = Uw[a:b] @ U.T
    idx = torch.arange(r0, r1, device=device)
    H[idx - r0, idx] += torch.from_numpy(q.d).to(device)[r0:r1]
    return H, ldh


def host_hessian_padded(q):
    n = q.n
    ldh = n + (n & 1)
    H = np.zeros((n, ldh))
    H[:, :n] = q.H
    return H, ldh


def problem_tensors(q, device, H=None, ldh=None, host=False):
    """Dict of the ipm_problem arrays.  host=True returns pinned CPU tensors (e2e path)."""
    if H is None:
        if host:
            Hn, ldh = host_hessian_padded(q)
            H = torch.from_numpy(Hn).pin_memory()
        else:
            H, ldh = device_hessian(q, device)
    def t(a, dt):
        x = torch.from_numpy(np.ascontiguousarray(a)).to(dt)
        return x.pin_memory() if host else x.to(device)
    return dict(H=H, ldh=ldh, g=t(q.g, torch.float64), A_rowptr=t(q.A_rowptr, torch.int64),
                A_col=t(q.A_col, torch.int32), A_val=t(q.A_val, torch.float64), l=t(q.l, torch.float64),
                u=t(q.u, torch.float64), xl=t(q.xl, torch.float64), xu=t(q.xu, torch.float64))
