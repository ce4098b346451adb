"""Pins for the sparse-extrapolation oracle (oracle/sparse.py), Eq. CPQRCOEFFS."""

from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg as sl
from numpy.polynomial import legendre as L

from oracle import ExtrapSparse, cpqr_pivots_exact, lebesgue, ls_weights, naive_weights, sparse_weights, \
    sparse_weights_exact

CASES = [(1, 3), (2, 6), (2, 8), (3, 8), (2, 12), (3, 12), (4, 12), (3, 16), (5, 30)]


def _grid(M):
    h = 2.0 / (M - 1)
    return np.array([-1.0 + i * h for i in range(M)]), 1.0 + h


# The pivot set equals LAPACK's column-pivoted QR (dgeqp3 via scipy) of V^T.
@pytest.mark.parametrize("m,M", CASES)
def test_pivots_match_lapack_cpqr(m, M):
    t, _ = _grid(M)
    _, _, P = sl.qr(L.legvander(t, m).T, pivoting=True)
    assert sorted(P[:m + 1].tolist()) == sorted(cpqr_pivots_exact(m, M))


# Exactness beta^T V = v^T (Eq. POLYEXACTNESS) with at most m+1 nonzeros.
@pytest.mark.parametrize("m,M", CASES)
def test_exactness_and_sparsity(m, M):
    beta = sparse_weights(m, M)
    t, tn = _grid(M)
    assert np.count_nonzero(beta) <= m + 1
    for k in range(m + 1):
        assert abs(beta @ t ** k - tn ** k) <= 1e-12 * max(1.0, tn ** k) * lebesgue(beta)


# "computing a degree-m polynomial interpolant through the data points corresponding to the nonzero
# coefficients": beta_j = Lagrange basis polynomial of the selected nodes at t_new.
@pytest.mark.parametrize("m,M", CASES)
def test_is_interpolant_through_selected_points(m, M):
    t, tn = _grid(M)
    S = sorted(cpqr_pivots_exact(m, M))
    beta = sparse_weights(m, M)
    for j in S:
        e = np.array([1.0 if i == j else 0.0 for i in S])
        c = np.polynomial.polynomial.polyfit(t[S], e, m)
        assert abs(np.polynomial.polynomial.polyval(tn, c) - beta[j]) <= 1e-10 * max(1.0, lebesgue(beta))


# Square case m = M-1 is the naive interpolation (Theorem 3.1); m = 0 is one weight 1.
@pytest.mark.parametrize("M", [2, 3, 5, 7])
def test_special_cases(M):
    assert sparse_weights_exact(M - 1, M) == [Fraction(b) for b in naive_weights(M)]
    w = sparse_weights(0, M)
    assert np.count_nonzero(w) == 1 and w.sum() == 1.0


# The LS weights are the minimum-norm solution of the exactness equation: the sparse
# solution cannot be shorter.
@pytest.mark.parametrize("m,M", CASES)
def test_not_shorter_than_least_squares(m, M):
    assert np.linalg.norm(sparse_weights(m, M)) >= np.linalg.norm(ls_weights(m, M)) - 1e-14


# Fig. 4: the Lebesgue constant of SPEXTRAP(floor(sqrt M), M) grows far slower than
# the naive 2^M - 1.
def test_lebesgue_growth_is_tame():
    for M in (4, 9, 16, 25, 30):
        m = int(np.sqrt(M))
        assert lebesgue(sparse_weights(m, M)) < 10.0 < 2 ** M - 1


def test_guess_uses_only_selected_history():
    N, M, m = 6, 8, 3
    ex = ExtrapSparse(N, M, m)
    rng = np.random.default_rng(0)
    xs = [rng.standard_normal(N) for _ in range(M)]
    for x in xs:
        ex.update(x)
    beta = sparse_weights(m, M)
    ref = sum(b * x for b, x in zip(beta, xs) if b != 0.0)
    assert np.allclose(ex.form_guess(None, np.zeros(N)), ref, rtol=1e-15, atol=1e-15)
