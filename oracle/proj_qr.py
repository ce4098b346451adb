"""Oracle: Fischer right-hand-side projection, Algorithms 1 and 2 of arXiv 2009.10863.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Plain numpy fp64,
written line by line from the listings:

* Algorithm 2 "Rolling QR" -- PAPER.md:253-308 (§2), notation PAPER.md:310-325.
* Algorithm 1 "Classic"    -- PAPER.md:217-251 (§2).

Readings of the paper taken here:

* AMB-2 (garbled Givens formula): after ``R <- R_{:,2:d}`` the
  matrix is upper Hessenberg; rotation i uses a = H_{i,i}, b = H_{i+1,i}
  (the sub-diagonal), r = hypot(a, b), c = a/r, s = b/r, G = [[c, s], [-s, c]].
  This zeroes H_{i+1,i} and keeps diag(R) > 0.
* AMB-3 (PAPER.md:209-215 vs 246/302): the admission test is RELATIVE,
  admit iff ||b~|| > eps * ||A x||, default eps = 1e-10.
* AMB-6: when d = 0 the guess is the caller's
  x0 unchanged; an update with ||A x|| = 0 at d = 0 is skipped.
* AMB-7/8: this oracle keeps the listing's per-pass x~ update and the explicit
  norm ||b~|| after pass 2 (the CUDA path uses an algebraically equal schedule).
"""

from __future__ import annotations

import math

import numpy as np


class ProjQR:
    """QR(M): rolling-QR projection, Algorithm 2.

    State: ``Bt`` (B~, N x M, orthonormal columns),
    ``Xt`` (X~, N x M, A X~ = B~), ``R`` (M x M upper triangular factor of the
    retained right-hand-side history, B~ playing the role of Q), ``d``.
    """

    def __init__(self, N: int, M: int, eps: float = 1e-10):
        if M < 1:
            raise ValueError("M >= 1 required")
        self.N, self.M, self.eps = int(N), int(M), float(eps)
        self.Bt = np.zeros((self.N, self.M))
        self.Xt = np.zeros((self.N, self.M))
        self.R = np.zeros((self.M, self.M))
        self.d = 0
        self.admitted = False  # outcome of the last update
        self.rho = float("nan")  # ||b~|| / ||A x|| of the last update

    # Alg. 2 line 1: "if d > 0: x0 = X~ B~_{:,1:d}^T b"
    def form_guess(self, b: np.ndarray, x0: np.ndarray) -> np.ndarray:
        d = self.d
        if d == 0:
            return np.array(x0, dtype=np.float64, copy=True)  # x0: "arbitrary input"
        alpha = self.Bt[:, :d].T @ b
        return self.Xt[:, :d] @ alpha

    # Alg. 2, QR update block with the AMB-2 Givens reading.
    def downdate(self) -> None:
        d = self.d
        H = self.R[:d, 1:d].copy()  # "R <- R_{:,2:d}"  (d x (d-1), upper Hessenberg)
        for i in range(d - 1):
            a = H[i, i]
            b = H[i + 1, i]
            r = math.hypot(a, b)
            if r == 0.0:
                c, s = 1.0, 0.0
            else:
                c, s = a / r, b / r
            G = np.array([[c, s], [-s, c]])
            H[i:i + 2, :] = G @ H[i:i + 2, :]  # "R_{i:i+1,:} <- G R_{i:i+1,:}"
            self.Bt[:, i:i + 2] = self.Bt[:, i:i + 2] @ G.T  # "B~_{:,i:i+1} <- B~_{:,i:i+1} G^T"
            self.Xt[:, i:i + 2] = self.Xt[:, i:i + 2] @ G.T  # "X~_{:,i:i+1} <- X~_{:,i:i+1} G^T"
        self.R[:, :] = 0.0
        self.R[:d - 1, :d - 1] = H[:d - 1, :]
        self.Bt[:, d - 1] = 0.0  # the last rotated column leaves the space
        self.Xt[:, d - 1] = 0.0
        self.d = d - 1  # "d <- d - 1"

    # Alg. 2 lines after the solve.
    def update(self, x: np.ndarray, Ax: np.ndarray) -> bool:
        xt = np.array(x, dtype=np.float64, copy=True)  # "x~ <- x"
        bt = np.array(Ax, dtype=np.float64, copy=True)  # "b~ <- A x~"
        n0 = float(np.linalg.norm(bt))
        if self.d == self.M:
            self.downdate()
        d = self.d
        if d == 0:  # P:291-294, no eps test
            self.rho = 1.0 if n0 > 0 else 0.0
            if n0 == 0.0:  # S:144 reading: skip a zero vector
                self.admitted = False
                return False
            self.R[0, 0] = n0
            self.Xt[:, 0] = xt / n0
            self.Bt[:, 0] = bt / n0
            self.d = 1
            self.admitted = True
            return True
        self.R[:d, d] = 0.0  # "R_{1:d,d+1} <- 0"
        for _ in range(2):  # twice-iterated Gram--Schmidt
            c = self.Bt[:, :d].T @ bt  # "c <- B~_{:,1:d}^T b~"
            bt = bt - self.Bt[:, :d] @ c  # "b~ <- b~ - B~ c"
            xt = xt - self.Xt[:, :d] @ c  # "x~ <- x~ - X~ c"
            self.R[:d, d] += c  # "R_{1:d,d+1} <- R_{1:d,d+1} + c"
        nb = float(np.linalg.norm(bt))
        self.rho = nb / n0 if n0 > 0 else 0.0
        if nb > self.eps * n0:  # AMB-3 relative reading of "||b~|| > eps"
            self.R[d, d] = nb
            self.Xt[:, d] = xt / nb
            self.Bt[:, d] = bt / nb
            self.d = d + 1
            self.admitted = True
            return True
        self.admitted = False
        return False


class ProjClassic:
    """CLASSIC(M): Algorithm 1, restart when d = 0 or d >= M."""

    def __init__(self, N: int, M: int, eps: float = 1e-10):
        if M < 1:
            raise ValueError("M >= 1 required")
        self.N, self.M, self.eps = int(N), int(M), float(eps)
        self.Bt = np.zeros((self.N, self.M))
        self.Xt = np.zeros((self.N, self.M))
        self.d = 0
        self.admitted = False
        self.rho = float("nan")

    def form_guess(self, b: np.ndarray, x0: np.ndarray) -> np.ndarray:
        d = self.d
        if d == 0:
            return np.array(x0, dtype=np.float64, copy=True)
        alpha = self.Bt[:, :d].T @ b
        return self.Xt[:, :d] @ alpha

    def update(self, x: np.ndarray, Ax: np.ndarray) -> bool:
        xt = np.array(x, dtype=np.float64, copy=True)
        bt = np.array(Ax, dtype=np.float64, copy=True)
        n0 = float(np.linalg.norm(bt))
        d = self.d
        if d == 0 or d >= self.M:  # restart branch
            self.rho = 1.0 if n0 > 0 else 0.0
            if n0 == 0.0:
                self.admitted = False
                return False
            self.Bt[:, :] = 0.0
            self.Xt[:, :] = 0.0
            self.Xt[:, 0] = xt / n0
            self.Bt[:, 0] = bt / n0
            self.d = 1
            self.admitted = True
            return True
        for _ in range(2):
            c = self.Bt[:, :d].T @ bt
            bt = bt - self.Bt[:, :d] @ c
            xt = xt - self.Xt[:, :d] @ c
        nb = float(np.linalg.norm(bt))
        self.rho = nb / n0 if n0 > 0 else 0.0
        if nb > self.eps * n0:  # P:246-249 with the AMB-3 relative reading
            self.Xt[:, d] = xt / nb
            self.Bt[:, d] = bt / nb
            self.d = d + 1
            self.admitted = True
            return True
        self.admitted = False
        return False
