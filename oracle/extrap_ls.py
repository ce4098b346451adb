"""Oracle: stabilized least-squares polynomial extrapolation of arXiv 2009.10863.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

* Guess (Eq. EXTRAPEXPN):
      x^_{n+1} = sum_{i=1}^{M} beta_i x_{n-M+i},   beta_1 multiplies the OLDEST.
* Weights (Eq. LSQRCOEFFS, §3.2):
      t_i = -1 + (i-1) h,  h = 2/(M-1),  1 <= i <= M;  t_{n+1} = 1 + h;
      V_ij = psi_j(t_i),  v_j = psi_j(t_{n+1}),  0 <= j <= m (Legendre psi_j);
      beta^T = v^T (V^T V)^{-1} V^T.
  Evaluated literally in EXACT rational arithmetic (``fractions.Fraction``):
  form V^T V, solve (V^T V) y = v by Gauss-Jordan elimination, beta = V y; then
  each beta_i is rounded once to the nearest double.
* Naive weights (Theorem 3.1, Eq. NAIVEEXTRAPCOEFFS):
      beta_i = (-1)^{M-i} C(M, i-1).
* Lebesgue constant (§6.5): Lambda = ||beta||_1.

Readings: AMB-11 M = 1 -> beta = [1] (h undefined); AMB-13 warm-up with
fill f < M uses the (min(m, f-1), f) scheme; f = 0 leaves x0 untouched;
AMB-14 M >= m+1 required.
"""

from __future__ import annotations

from fractions import Fraction
from math import comb

import numpy as np


def _legendre_values(m: int, t: Fraction) -> list:
    """psi_0..psi_m at t: Legendre three-term recurrence (j+1) P_{j+1} = (2j+1) t P_j - j P_{j-1}."""
    vals = [Fraction(1)]
    if m >= 1:
        vals.append(Fraction(t))
    for j in range(1, m):
        vals.append(((2 * j + 1) * t * vals[j] - j * vals[j - 1]) / (j + 1))
    return vals


def _solve_exact(A: list, rhs: list) -> list:
    """Gauss-Jordan elimination over the rationals (exact; A square, nonsingular)."""
    n = len(A)
    Aug = [list(A[r]) + [rhs[r]] for r in range(n)]
    for col in range(n):
        piv = next(r for r in range(col, n) if Aug[r][col] != 0)
        Aug[col], Aug[piv] = Aug[piv], Aug[col]
        pv = Aug[col][col]
        Aug[col] = [a / pv for a in Aug[col]]
        for r in range(n):
            if r != col and Aug[r][col] != 0:
                f = Aug[r][col]
                Aug[r] = [a - f * b for a, b in zip(Aug[r], Aug[col])]
    return [Aug[r][n] for r in range(n)]


def ls_weights_exact(m: int, M: int) -> list:
    """beta (oldest first) of EXTRAP(m, M) as exact Fractions, Eq. LSQRCOEFFS."""
    if m < 0 or M < 1 or M < m + 1:
        raise ValueError(f"EXTRAP({m},{M}) needs M >= m+1 >= 1 (PAPER.md:416)")
    if M == 1:
        return [Fraction(1)]  # AMB-11
    h = Fraction(2, M - 1)
    t = [Fraction(-1) + (i - 1) * h for i in range(1, M + 1)]
    V = [_legendre_values(m, ti) for ti in t]  # V_ij = psi_j(t_i)
    v = _legendre_values(m, Fraction(1) + h)  # v_j = psi_j(t_{n+1})
    VtV = [[sum(V[i][a] * V[i][b] for i in range(M)) for b in range(m + 1)] for a in range(m + 1)]
    y = _solve_exact(VtV, v)  # (V^T V)^{-1} v
    return [sum(V[i][j] * y[j] for j in range(m + 1)) for i in range(M)]  # beta = V (V^T V)^{-1} v


def ls_weights(m: int, M: int) -> np.ndarray:
    """EXTRAP(m, M) weights rounded once from the exact rationals (Fraction -> float is correctly rounded)."""
    return np.array([float(b) for b in ls_weights_exact(m, M)], dtype=np.float64)


def naive_weights(M: int) -> list:
    """Theorem 3.1: beta_i = (-1)^{M-i} C(M, i-1), i = 1..M, exact integers."""
    return [(-1) ** (M - i) * comb(M, i - 1) for i in range(1, M + 1)]


def warmup_weights(m: int, M: int, f: int) -> np.ndarray:
    """Weights used with f stored solutions (AMB-13): EXTRAP(min(m, f-1), f); f = M is the steady scheme."""
    if not (1 <= f <= M):
        raise ValueError("1 <= f <= M")
    return ls_weights(min(m, f - 1), f)


def lebesgue(beta) -> float:
    """Lambda = ||beta||_1."""
    return float(sum(abs(float(b)) for b in beta))


class ExtrapLS:
    """EXTRAP(m, M): least-squares extrapolation over a window of M solutions (§3.2)."""

    def __init__(self, N: int, M: int, m: int):
        if m < 0 or M < m + 1:
            raise ValueError(f"EXTRAP({m},{M}) needs M >= m+1 (PAPER.md:416)")
        self.N, self.M, self.m = int(N), int(M), int(m)
        self.table = [warmup_weights(self.m, self.M, f) for f in range(1, self.M + 1)]
        self.ring: list = []  # oldest first

    @property
    def fill(self) -> int:
        return len(self.ring)

    def weights(self) -> np.ndarray:
        return self.table[self.fill - 1]

    # Eq. EXTRAPEXPN: x^ = sum_i beta_i x_{n-M+i}, summed oldest first.
    def form_guess(self, b, x0: np.ndarray) -> np.ndarray:
        f = self.fill
        if f == 0:
            return np.array(x0, dtype=np.float64, copy=True)
        beta = self.table[f - 1]
        acc = beta[0] * self.ring[0]
        for i in range(1, f):
            acc = acc + beta[i] * self.ring[i]
        return acc

    def update(self, x: np.ndarray, Ax=None) -> bool:
        self.ring.append(np.array(x, dtype=np.float64, copy=True))
        if len(self.ring) > self.M:
            self.ring.pop(0)
        return True
