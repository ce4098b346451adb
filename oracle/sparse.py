"""Oracle: sparse polynomial extrapolation, Eq. CPQRCOEFFS (§3.3).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

  V^T P = Q R (column-pivoted QR of the (m+1) x M matrix V^T, Legendre basis on the §3.2 grid),
  beta = P [ Rhat^{-1} Q^T v ; 0 ].
Only the m+1 pivot columns carry weight, and on them beta solves V_S^T beta_S = v exactly
("computing a degree-m polynomial interpolant through the data points corresponding
to the nonzero coefficients").  This oracle performs the pivoting in EXACT rational arithmetic:
the pivot at step k is the column with the largest squared residual norm after (unnormalised,
exact) Gram-Schmidt against the previous pivots -- the same quantity Householder CPQR compares
-- with exact ties broken toward the lowest (oldest) index (AMB-16 reading); beta_S is then the
exact solution of the square system, rounded once to fp64.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

from .extrap_ls import _legendre_values, _solve_exact


def cpqr_pivots_exact(m: int, M: int) -> list:
    """0-based indices (oldest = 0) of the m+1 CPQR pivot columns of V^T, in pivot order."""
    if M == 1:
        return [0]
    h = Fraction(2, M - 1)
    cols = [_legendre_values(m, Fraction(-1) + i * h) for i in range(M)]  # column i of V^T
    resid = [list(c) for c in cols]
    piv = []
    for _ in range(m + 1):
        norms = [(sum(x * x for x in resid[j]) if j not in piv else Fraction(-1)) for j in range(M)]
        best = max(norms)
        j = min(i for i in range(M) if norms[i] == best)  # exact tie -> lowest index
        piv.append(j)
        u = resid[j]
        uu = sum(x * x for x in u)
        for i in range(M):  # remove the u component from every remaining residual column
            if i in piv:
                continue
            c = sum(a * b for a, b in zip(u, resid[i])) / uu
            resid[i] = [a - c * b for a, b in zip(resid[i], u)]
    return piv


def sparse_weights_exact(m: int, M: int) -> list:
    """beta (oldest first, exact Fractions) of SPEXTRAP(m, M)."""
    if m < 0 or M < m + 1:
        raise ValueError(f"SPEXTRAP({m},{M}) needs M >= m+1 (PAPER.md:416)")
    beta = [Fraction(0)] * M
    if M == 1:
        beta[0] = Fraction(1)
        return beta
    piv = cpqr_pivots_exact(m, M)
    h = Fraction(2, M - 1)
    VS_T = [[_legendre_values(m, Fraction(-1) + j * h)[r] for j in piv] for r in range(m + 1)]  # V_S^T
    v = _legendre_values(m, Fraction(1) + h)
    bS = _solve_exact(VS_T, v)  # V_S^T beta_S = v  (Rhat beta_S = Q^T v)
    for j, bj in zip(piv, bS):
        beta[j] = bj
    return beta


def sparse_weights(m: int, M: int) -> np.ndarray:
    return np.array([float(b) for b in sparse_weights_exact(m, M)], dtype=np.float64)


class ExtrapSparse:
    """SPEXTRAP(m, M) with the same warm-up rule as ExtrapLS (AMB-13): (min(m, f-1), f)."""

    def __init__(self, N: int, M: int, m: int):
        if m < 0 or M < m + 1:
            raise ValueError(f"SPEXTRAP({m},{M}) needs M >= m+1 (PAPER.md:416)")
        self.N, self.M, self.m = int(N), int(M), int(m)
        self.table = [sparse_weights(min(self.m, f - 1), f) for f in range(1, self.M + 1)]
        self.ring: list = []

    @property
    def fill(self) -> int:
        return len(self.ring)

    def weights(self) -> np.ndarray:
        return self.table[self.fill - 1]

    def form_guess(self, b, x0):
        f = self.fill
        if f == 0:
            return np.array(x0, dtype=np.float64, copy=True)
        beta = self.table[f - 1]
        acc = None
        for i in range(f):  # Eq. EXTRAPEXPN over the nonzero weights, oldest first
            if beta[i] != 0.0:
                acc = beta[i] * self.ring[i] if acc is None else acc + beta[i] * self.ring[i]
        return acc

    def update(self, x, Ax=None) -> bool:
        self.ring.append(np.array(x, dtype=np.float64, copy=True))
        if len(self.ring) > self.M:
            self.ring.pop(0)
        return True
