"""Pins for the projection oracle (oracle/proj_qr.py): Algorithms 1 and 2 of arXiv 2009.10863.

Pinned against: the optimality definition (brute-force least squares over the
retained raw pairs), span exactness,
orthonormality/A X~ = B~, numpy's QR of the retained
columns (the downdate), the QR(1) closed form, Theorem 4.1
(i)/(ii), and the d-transition rules of the listings.
"""

import math

import numpy as np
import pytest

from oracle import ExtrapLS, ProjClassic, ProjQR, ls_weights


def _spd(N, seed=10863, lo=1.0, hi=50.0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((N, N)))
    return (Q * np.linspace(lo, hi, N)) @ Q.T


def _smooth_seq(N, steps, seed=7, modes=12, dt=0.05):
    rng = np.random.default_rng(seed)
    V = rng.standard_normal((N, modes))
    w = rng.uniform(0.5, 3.0, modes)
    ph = rng.uniform(0, 2 * np.pi, modes)
    return [V @ np.sin(w * n * dt + ph) for n in range(steps)]


def _run_qr_with_raw(A, xs, M, eps=1e-10, cls=ProjQR):
    """Run the oracle and record the raw admitted (x, Ax) pairs it should be projecting onto."""
    N = A.shape[0]
    p = cls(N, M, eps)
    raw = []
    for x in xs:
        Ax = A @ x
        adm = p.update(x, Ax)
        if cls is ProjQR:
            if adm:
                raw.append((x, Ax))
            raw = raw[-p.d:] if p.d else []
        else:
            raw = [(x, Ax)] if p.d == 1 else (raw + [(x, Ax)] if adm else raw)
        yield p, raw


# PIN-P2: brute force.  x0 = X_raw argmin_y ||b - B_raw y||_2 over the retained raw pairs.
@pytest.mark.parametrize("M", [1, 2, 4, 8])
@pytest.mark.parametrize("cls", [ProjQR, ProjClassic])
def test_guess_equals_bruteforce_lstsq(M, cls):
    N = 80
    A = _spd(N)
    xs = _smooth_seq(N, 3 * M + 5, modes=40, dt=0.4)  # well-conditioned raw history for lstsq
    rng = np.random.default_rng(3)
    for p, raw in _run_qr_with_raw(A, xs, M, cls=cls):
        b = A @ xs[-1] + rng.standard_normal(N)
        x0 = p.form_guess(b, np.zeros(N))
        Xr = np.stack([r[0] for r in raw], 1)
        Br = np.stack([r[1] for r in raw], 1)
        y, *_ = np.linalg.lstsq(Br, b, rcond=None)
        x_bf = Xr @ y
        assert p.d == len(raw)
        assert np.linalg.norm(x0 - x_bf) <= 1e-10 * np.linalg.norm(x_bf)
        # the residual is the least-squares residual
        assert abs(np.linalg.norm(b - A @ x0) - np.linalg.norm(b - Br @ y)) <= 1e-12 * np.linalg.norm(b)


# PIN-P1: b in span{A x_k retained} -> zero residual.
def test_b_in_span_gives_zero_residual():
    N, M = 60, 5
    A = _spd(N)
    rng = np.random.default_rng(5)
    xs = [rng.standard_normal(N) for _ in range(M)]
    p = ProjQR(N, M)
    for x in xs:
        p.update(x, A @ x)
    assert p.d == M
    coef = rng.standard_normal(M)
    b = sum(c * (A @ x) for c, x in zip(coef, xs))
    x0 = p.form_guess(b, np.zeros(N))
    assert np.linalg.norm(b - A @ x0) <= 1e-12 * np.linalg.norm(b)
    assert np.linalg.norm(x0 - sum(c * x for c, x in zip(coef, xs))) <= 1e-10 * np.linalg.norm(x0)


# PIN-P3: for a fixed b the residual is non-increasing while d grows (nested spans).
def test_residual_monotone_while_filling():
    N, M = 70, 10
    A = _spd(N)
    xs = _smooth_seq(N, M + 1, modes=30)
    b = A @ xs[-1]
    p = ProjQR(N, M, eps=1e-14)
    last = np.linalg.norm(b)
    for x in xs[:-1]:
        p.update(x, A @ x)
        r = np.linalg.norm(b - A @ p.form_guess(b, np.zeros(N)))
        assert r <= last * (1 + 1e-12) + 1e-14 * np.linalg.norm(b)
        last = r


# PIN-P4 and A X~ = B~ after every update, through many downdates.
@pytest.mark.parametrize("M", [2, 3, 8])
def test_orthonormal_and_AX_equals_B(M):
    N = 50
    A = _spd(N, hi=5.0)
    rng = np.random.default_rng(11)
    p = ProjQR(N, M)
    for _ in range(4 * M + 3):
        x = rng.standard_normal(N)
        p.update(x, A @ x)
        d = p.d
        B = p.Bt[:, :d]
        assert np.max(np.abs(B.T @ B - np.eye(d))) <= 1e-12
        assert np.max(np.abs(A @ p.Xt[:, :d] - B)) <= 1e-10
        assert np.all(np.diag(p.R[:d, :d]) > 0)
        assert np.allclose(np.tril(p.R[:d, :d], -1), 0.0)


# PIN-P5: the Givens downdate (AMB-2 reading) equals numpy's positive-diagonal QR of the
# retained raw right-hand sides, and B~ R reproduces them.
@pytest.mark.parametrize("M", [2, 4, 7])
def test_downdate_matches_fresh_qr(M):
    N = 40
    A = _spd(N, hi=3.0)
    rng = np.random.default_rng(2)
    p = ProjQR(N, M, eps=0.0)
    raw = []
    for _ in range(M):
        x = rng.standard_normal(N)
        p.update(x, A @ x)
        raw.append(A @ x)
    p.downdate()
    Braw = np.stack(raw[1:], 1)
    Q, Rq = np.linalg.qr(Braw)
    sg = np.sign(np.diag(Rq))
    Q, Rq = Q * sg, (Rq.T * sg).T
    d = p.d
    assert d == M - 1
    assert np.max(np.abs(p.Bt[:, :d] @ p.R[:d, :d] - Braw)) <= 1e-12 * np.max(np.abs(Braw))
    assert np.max(np.abs(p.Bt[:, :d] - Q)) <= 1e-12
    assert np.max(np.abs(p.R[:d, :d] - Rq)) <= 1e-12 * np.max(np.abs(Rq))


# The printed Givens formula (s = sign(a)/r with no factor b) does NOT zero the
# sub-diagonal; the AMB-2 reading does (documents why the reading was needed).
def test_literal_givens_is_garbled_and_reading_is_standard(golden):
    a, b = 3.0, 4.0
    r = math.hypot(a, b)
    c_lit, s_lit = abs(a) / r, math.copysign(1.0, a) / r
    assert abs(-s_lit * a + c_lit * b) > 0.1
    c, s = a / r, b / r
    assert (c, s) == tuple(float(v) for v in golden["givens_3_4"][0].split())
    assert abs(-s * a + c * b) <= 1e-15 and abs(c * a + s * b - 5.0) < 1e-15


# PIN-P8: QR(1) closed form (Alg. 2 with M = 1): x0 = (<A x_{n-1}, b> / ||A x_{n-1}||^2) x_{n-1}.
def test_qr1_closed_form():
    N = 30
    A = _spd(N)
    rng = np.random.default_rng(4)
    p = ProjQR(N, 1)
    for _ in range(6):
        x = rng.standard_normal(N)
        Ax = A @ x
        p.update(x, Ax)
        assert p.d == 1
        b = rng.standard_normal(N)
        x0 = p.form_guess(b, np.zeros(N))
        assert np.linalg.norm(x0 - (Ax @ b) / (Ax @ Ax) * x) <= 1e-14 * np.linalg.norm(x0)


# PIN-P9: b = B~_j -> x0 = X~_j; d = 0 -> x0 unchanged.
def test_basis_vector_and_empty_history():
    N, M = 25, 4
    A = _spd(N)
    rng = np.random.default_rng(6)
    p = ProjQR(N, M)
    x0 = rng.standard_normal(N)
    assert np.array_equal(p.form_guess(rng.standard_normal(N), x0), x0)
    for _ in range(M):
        x = rng.standard_normal(N)
        p.update(x, A @ x)
    for j in range(M):
        assert np.max(np.abs(p.form_guess(p.Bt[:, j], x0) - p.Xt[:, j])) <= 1e-13 * np.max(np.abs(p.Xt[:, j]))
    # zero A x at d = 0 is skipped (SPEC S:144 reading, AMB-6)
    q = ProjQR(N, M)
    assert q.update(np.zeros(N), np.zeros(N)) is False and q.d == 0


# PIN-P10: d transitions: fill 1..M, then stays M; a dependent pair after the downdate
# is rejected and leaves d = M-1.
def test_d_transitions_and_rejection():
    N, M = 30, 4
    A = _spd(N)
    rng = np.random.default_rng(8)
    p = ProjQR(N, M)
    ds = []
    xs = []
    for _ in range(M + 3):
        x = rng.standard_normal(N)
        xs.append(x)
        p.update(x, A @ x)
        ds.append(p.d)
    assert ds == list(range(1, M + 1)) + [M] * 3
    dup = xs[-2] * 0.5 + xs[-1] * 2.0  # lies in the span of the retained pairs after the downdate
    assert p.update(dup, A @ dup) is False
    assert p.d == M - 1 and p.rho < 1e-10


# CLASSIC (Alg. 1): d cycles 1..M then restarts.
def test_classic_restart_cycle():
    N, M = 30, 3
    A = _spd(N)
    rng = np.random.default_rng(9)
    p = ProjClassic(N, M)
    ds = []
    for _ in range(3 * M + 1):
        x = rng.standard_normal(N)
        p.update(x, A @ x)
        ds.append(p.d)
    assert ds == [1, 2, 3] * 3 + [1]


# Theorem 4.1(i) and (ii): ||r^P|| <= ||r^E|| and r^P = O(h^M).
@pytest.mark.parametrize("M,m", [(3, 1), (4, 2), (5, 2)])
def test_theorem_4_1(M, m):
    N = 120
    A = _spd(N)
    rng = np.random.default_rng(10863)
    K = 40
    V = rng.standard_normal((N, K)) / np.sqrt(N)
    w = rng.uniform(0.5, 2.0, K)
    ph = rng.uniform(0, 2 * np.pi, K)
    xfun = lambda s: V @ np.sin(w * s + ph)  # noqa: E731
    beta = ls_weights(m, M)
    rP, rE = [], []
    hs = [0.4 * 2.0 ** -k for k in range(5)]
    for h in hs:
        xs = [xfun(i * h) for i in range(M)]
        x_new = xfun(M * h)
        b = A @ x_new
        p = ProjQR(N, M, eps=0.0)
        for x in xs:
            p.update(x, A @ x)
        assert p.d == M
        xP = p.form_guess(b, np.zeros(N))
        xE = sum(bi * xi for bi, xi in zip(beta, xs))
        rP.append(np.linalg.norm(b - A @ xP))
        rE.append(np.linalg.norm(b - A @ xE))
        assert rP[-1] <= rE[-1] + 1e-12 * np.linalg.norm(b)
    slopes = [math.log2(rP[k] / rP[k + 1]) for k in range(len(hs) - 1) if rP[k + 1] > 1e-11]
    assert abs(slopes[-1] - M) < 0.5, slopes


# Projection beats extrapolation on the same history in the open-loop harness sequence (qualitative check
# of the §6.3 claim): more reduction of the initial residual.
def test_projection_vs_extrapolation_harness_sequence():
    import torch

    from workloads import Grid, manufactured_step

    g = Grid(12, 2)
    p, e = ProjQR(g.N, 8), ExtrapLS(g.N, 4, 2)
    resP, resE = [], []
    for n in range(14):
        b, x, Ax = (t.numpy() for t in manufactured_step(g, n, dt=1e-2))
        if n >= 9:
            # residual of the guess measured through the operator the sequence was built with
            from workloads import helmholtz_apply

            for o, store in ((p, resP), (e, resE)):
                x0 = o.form_guess(b, np.zeros(g.N))
                store.append(np.linalg.norm(b - helmholtz_apply(g, torch.from_numpy(x0)).numpy()) / np.linalg.norm(b))
        p.update(x, Ax)
        e.update(x, Ax)
    assert max(resP) < min(resE)


def test_closed_loop_envelope_fixture_matches_the_oracle():
    """tests/golden/closed_loop_envelope.json (scripts/closed_loop_envelope.py, oracle only; DESIGN.md
    AMB-21) was written by the current oracle: its unperturbed closed-loop CG counts reproduce
    exactly, and it records the oracle's own rounding-level spread (> 1 for QR(8): the fully
    closed loop's +-1 is not implied by correctness alone)."""
    import json
    import os

    import torch

    from oracle import ExtrapLS, ExtrapSparse, ProjClassic, ProjQR
    from workloads import Grid, helmholtz_apply, prescribed_rhs
    from workloads.cg import pcg

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "closed_loop_envelope.json")
    fx = json.load(open(path))
    g = Grid(32, 2)
    for key, mk in (("proj_qr(8,0)", lambda: ProjQR(g.N, 8)), ("extrap_ls(8,3)", lambda: ExtrapLS(g.N, 8, 3)),
                    ("proj_classic(4,0)", lambda: ProjClassic(g.N, 4)),
                    ("extrap_sparse(8,3)", lambda: ExtrapSparse(g.N, 8, 3))):
        obj, x_prev, its = mk(), np.zeros(g.N), []
        for n in range(40):
            b = prescribed_rhs(g, n, 1e-3)
            x0 = np.asarray(obj.form_guess(b.numpy(), x_prev.copy()), dtype=np.float64)
            x, it, _, _ = pcg(g, b, torch.from_numpy(x0))
            its.append(int(it))
            obj.update(x.numpy(), helmholtz_apply(g, x).numpy())
            x_prev = x.numpy()
        assert its == fx["methods"][key]["unperturbed"], key
    assert fx["methods"]["proj_qr(8,0)"]["1e-15"]["max_abs_diff"] > 1
