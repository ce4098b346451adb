"""Pins for the extrapolation oracle (oracle/extrap_ls.py) against what the paper and mathematics fix.

Each test names the passage it follows.  None of these re-types the oracle's
formula: they compare it with paper-printed values, Theorem 3.1's closed form,
textbook closed forms (mean, simple linear regression), numpy least squares
on unit data, the exactness/min-norm properties and Theorem 4.1(iii)'s order.
"""

from fractions import Fraction

import numpy as np
import pytest

from oracle import ExtrapLS, lebesgue, ls_weights, ls_weights_exact, naive_weights, warmup_weights


def _grid(M):
    h = 2.0 / (M - 1)
    return np.array([-1.0 + i * h for i in range(M)]), 1.0 + h


# PIN-E3: the paper's only printed worked example.
def test_paper_naive_m2(golden):
    val, _ = golden["naive_M2_beta"]
    expect = [int(v) for v in val.split()]
    assert naive_weights(2) == expect
    assert ls_weights_exact(1, 2) == [Fraction(v) for v in expect]  # degree M-1 LS = interpolation


# ignoring sign, the naive weights are row M+1 of Pascal's triangle.
def test_naive_pascal_row_built_by_additions():
    row = [1]
    for M in range(1, 16):
        row = [1] + [row[k] + row[k + 1] for k in range(len(row) - 1)] + [1]  # row M of Pascal's triangle
        assert [abs(b) for b in naive_weights(M)] == row[:M]
        signs = [1 if b > 0 else -1 for b in naive_weights(M)]
        assert signs[-1] == 1 and all(signs[i] == -signs[i + 1] for i in range(M - 1))


# Theorem 3.1: degree M-1 least squares is interpolation -> the binomial closed form.
@pytest.mark.parametrize("M", range(1, 9))
def test_ls_full_degree_equals_theorem_3_1(M):
    assert ls_weights_exact(M - 1, M) == [Fraction(b) for b in naive_weights(M)]


# §6.5 Theorem: Lambda(naive) = 2^M - 1.
@pytest.mark.parametrize("M", [1, 2, 3, 5, 8, 13, 20])
def test_naive_lebesgue(M):
    assert sum(abs(b) for b in naive_weights(M)) == 2 ** M - 1
    assert lebesgue(naive_weights(M)) == 2 ** M - 1


# Constant least-squares fit is the mean (textbook).
@pytest.mark.parametrize("M", [1, 2, 4, 7, 16, 30])
def test_degree0_is_mean(M):
    assert ls_weights_exact(0, M) == [Fraction(1, M)] * M


# Degree-1 least squares = textbook simple linear regression evaluated at t_new.
@pytest.mark.parametrize("M", [2, 3, 4, 8, 12, 31])
def test_degree1_is_linear_regression(M):
    # regression on the integer grid s_i = i (affine-equivalent to the paper's t_i), evaluated at s = M
    s = [Fraction(i) for i in range(M)]
    sbar = sum(s) / M
    sxx = sum((si - sbar) ** 2 for si in s)
    expect = [Fraction(1, M) + (Fraction(M) - sbar) * (si - sbar) / sxx for si in s]
    assert ls_weights_exact(1, M) == expect


def test_spec_extrap_1_3(golden):
    val, _ = golden["extrap_1_3_beta"]
    assert ls_weights_exact(1, 3) == [Fraction(v) for v in val.split()]


# Brute force: beta_i is the value at 1+h of the degree-m LS fit to unit data e_i.
@pytest.mark.parametrize("m,M", [(0, 3), (1, 4), (2, 4), (2, 8), (3, 8), (3, 12), (4, 12), (3, 16), (5, 30)])
def test_bruteforce_lstsq_unit_data(m, M):
    t, tn = _grid(M)
    V = np.vander(t, m + 1, increasing=True)  # monomial basis: LS weights are basis independent
    beta_bf = np.empty(M)
    for i in range(M):
        e = np.zeros(M)
        e[i] = 1.0
        c, *_ = np.linalg.lstsq(V, e, rcond=None)
        beta_bf[i] = np.polynomial.polynomial.polyval(tn, c)
    beta = ls_weights(m, M)
    assert np.max(np.abs(beta - beta_bf)) <= 1e-12 * max(1.0, lebesgue(beta))


# Exactness (Eq. POLYEXACTNESS): beta^T V = v^T, so sum(beta) = 1 and polynomials of
# degree <= m are reproduced; degree m+1 generally is not.
@pytest.mark.parametrize("m,M", [(1, 3), (2, 4), (2, 8), (3, 8), (4, 8), (2, 12), (3, 12), (4, 12), (3, 16), (5, 30)])
def test_exactness_and_sum(m, M):
    beta = ls_weights(m, M)
    assert abs(beta.sum() - 1.0) <= 1e-14 * lebesgue(beta)
    t, tn = _grid(M)
    for k in range(m + 1):
        assert abs(beta @ t ** k - tn ** k) <= 1e-12 * max(1.0, tn ** k) * lebesgue(beta)
    if M > m + 1:
        assert abs(beta @ t ** (m + 1) - tn ** (m + 1)) > 1e-6


# Minimum norm: ||beta||_2 <= ||beta + z||_2 for every z in null(V^T).
@pytest.mark.parametrize("m,M", [(1, 4), (2, 8), (3, 8), (3, 16)])
def test_minimum_norm(m, M):
    t, _ = _grid(M)
    V = np.vander(t, m + 1, increasing=True)
    _, _, Wt = np.linalg.svd(V.T)
    Z = Wt[m + 1:].T  # basis of null(V^T)
    beta = ls_weights(m, M)
    assert np.max(np.abs(Z.T @ beta)) < 1e-12  # beta is orthogonal to the null space -> min-norm
    rng = np.random.default_rng(10863)
    for _ in range(50):
        z = Z @ rng.standard_normal(Z.shape[1]) * 0.1
        assert np.linalg.norm(beta + z) > np.linalg.norm(beta)


# Theorem 4.1(iii): extrapolation error O(h^{m+1}).
@pytest.mark.parametrize("m,M", [(1, 4), (2, 6), (3, 8)])
def test_order_h_pow_m_plus_1(m, M):
    f = lambda s: np.sin(1.3 * s + 0.4) + 0.5 * np.cos(2.1 * s)  # noqa: E731
    beta = ls_weights(m, M)
    errs = []
    hs = [0.2 * 2.0 ** -k for k in range(5)]
    for h in hs:
        s = np.array([i * h for i in range(M)])
        errs.append(abs(beta @ f(s) - f(M * h)))
    slopes = [np.log2(errs[k] / errs[k + 1]) for k in range(len(errs) - 1)]
    assert abs(slopes[-1] - (m + 1)) < 0.5, slopes


def test_warmup_rule_and_guess():
    M, m, N = 4, 2, 7
    ex = ExtrapLS(N, M, m)
    x0 = np.full(N, 3.25)
    assert np.array_equal(ex.form_guess(None, x0), x0)  # fill 0: x0 untouched (AMB-13)
    rng = np.random.default_rng(1)
    a, b, c = rng.standard_normal((3, N))
    xs = [a + b * n + c * n * n for n in range(6)]  # quadratic in time: reproduced by EXTRAP(2, M>=3)
    for n in range(6):
        ex.update(xs[n])
        f = min(n + 1, M)
        np.testing.assert_array_equal(ex.weights(), warmup_weights(m, M, f))
        if f >= 3:  # degree min(2, f-1) = 2 -> exact for quadratics
            x_next = a + b * (n + 1) + c * (n + 1) ** 2
            assert np.max(np.abs(ex.form_guess(None, x0) - x_next)) <= 1e-11 * np.max(np.abs(x_next))
    assert warmup_weights(m, M, 1).tolist() == [1.0]  # fill 1 -> LAST
    assert np.allclose(warmup_weights(m, M, 2), [-1.0, 2.0])  # fill 2 -> linear interpolation


def test_constant_history_reproduced():
    ex = ExtrapLS(5, 8, 3)
    w = np.linspace(-2, 3, 5)
    for _ in range(10):
        ex.update(w)
    assert np.max(np.abs(ex.form_guess(None, np.zeros(5)) - w)) <= 1e-15 * 8 * lebesgue(ex.weights())


def test_argument_errors():
    with pytest.raises(ValueError):
        ls_weights_exact(4, 4)  # M >= m+1
    with pytest.raises(ValueError):
        ExtrapLS(3, 2, 2)
