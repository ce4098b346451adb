"""Harness Krylov solver (not the method): Jacobi-preconditioned CG on the harness operator.

Stopping criteria of PAPER.md:1373-1390 (§6.4):
  INITRESID (Eq. STOPCRITINITRESID, the libParanumal default): ||r|| < eps * max(||r0||, 1)
  RHS       (Eq. STOPCRITRHS):                                   ||r|| < eps * max(||b||, 1)
with eps = 1e-8 by default.  Device-agnostic torch fp64: the same harness drives the CUDA
library's guesses (cuda tensors) and the oracle's guesses (cpu tensors) in closed-loop runs.
"""

from __future__ import annotations

import torch

from .gen import Grid, helmholtz_apply, helmholtz_diag


def pcg(g: Grid, b: torch.Tensor, x0: torch.Tensor, eps: float = 1e-8, criterion: str = "initresid",
        maxit: int = 5000):
    """Solve A x = b from x0; returns (x, iterations, ||r0||, ||r||)."""
    dinv = 1.0 / helmholtz_diag(g)  # Jacobi (constant diagonal for this operator)
    x = x0.clone()
    r = b - helmholtz_apply(g, x)
    r0 = float(torch.linalg.vector_norm(r))
    ref = r0 if criterion == "initresid" else float(torch.linalg.vector_norm(b))
    thr = eps * max(ref, 1.0)
    rn = r0
    it = 0
    if rn < thr:
        return x, 0, r0, rn
    z = dinv * r
    p = z.clone()
    rz = float(torch.dot(r, z))
    while it < maxit:
        Ap = helmholtz_apply(g, p)
        alpha = rz / float(torch.dot(p, Ap))
        x += alpha * p
        r -= alpha * Ap
        it += 1
        rn = float(torch.linalg.vector_norm(r))
        if rn < thr:
            break
        z = dinv * r
        rz_new = float(torch.dot(r, z))
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, it, r0, rn
