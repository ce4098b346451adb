"""GPU parity: libig (CUDA, through the C ABI) against the CPU oracle on identical seeded inputs.

Protocol: OPEN LOOP -- one generated sequence (b_n, x_n, A x_n) is fed to
both sides; every guess must satisfy ||x0_gpu - x0_oracle||_2 <= 1e-11 ||x0_oracle||_2
(BASELINE.json north_star tolerance), every admission decision and history dimension must
be identical.  Sizes span several thread blocks and ragged tails; the full C2 size
(128^3 = 2,097,152 DOFs) is checked in the bench launch configuration.
"""

import numpy as np
import pytest
import torch

from oracle import ExtrapLS, ProjClassic, ProjQR, warmup_weights
from workloads import Grid, manufactured_step

pytestmark = pytest.mark.gpu

TOL = 1e-11


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2009_10863_b200.build import build

    build()


def _seq(g, steps, dt=1e-3):
    return [tuple(t.numpy() for t in manufactured_step(g, n, dt=dt)) for n in range(steps)]


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def run_proj_parity(g, M, steps, method="proj_qr", dt=1e-3, seq=None, misalign=False, fused=True):
    from paper_2009_10863_b200 import InitialGuess

    seq = seq or _seq(g, steps, dt)
    N = g.N
    ora = (ProjQR if method == "proj_qr" else ProjClassic)(N, M)
    ig = InitialGuess(N, method, M, fused=fused)
    off = 1 if misalign else 0
    buf = torch.zeros(4 * (N + 1) + 8, dtype=torch.float64, device="cuda")
    views = [buf[i * (N + 1) + off:i * (N + 1) + off + N] for i in range(4)]
    worst = 0.0
    x_prev = np.zeros(N)
    for n, (b, x, Ax) in enumerate(seq):
        x0_o = ora.form_guess(b, x_prev)  # fallback LAST
        vb, vx0, vx, vAx = views
        vb.copy_(torch.from_numpy(b))
        vx0.copy_(torch.from_numpy(x_prev))
        ig.form_guess(vb, vx0)
        x0_g = vx0.cpu().numpy()
        e = _rel(x0_g, x0_o)
        worst = max(worst, e)
        assert e <= TOL, f"step {n}: guess rel err {e:.3e}"
        ora.update(x, Ax)
        vx.copy_(torch.from_numpy(x))
        vAx.copy_(torch.from_numpy(Ax))
        ig.update(vx, vAx)
        st = ig.stats()
        assert st["d"] == ora.d, f"step {n}: d {st['d']} vs oracle {ora.d}"
        assert bool(st["admitted"]) == bool(ora.admitted), f"step {n}: admission differs"
        x_prev = x
    ig.close()
    return worst


# fused = persistent single-launch schedule (single-GPU default); split = one kernel per pass
# (the schedule used with a multi-rank communicator).
SCHEDULES = [pytest.param(True, id="fused"), pytest.param(False, id="split")]


@pytest.mark.parametrize("fused", SCHEDULES)
@pytest.mark.parametrize("M", [1, 2, 3, 5, 6, 8, 9, 10, 12, 13, 14, 16, 17, 20, 24, 25, 28, 30, 32])
def test_proj_qr_open_loop_c1(M, fused):
    # configs[0]: 2D 32x32 5-point Helmholtz, 40 steps
    run_proj_parity(Grid(32, 2), M, 40, fused=fused)


@pytest.mark.parametrize("fused", SCHEDULES)
@pytest.mark.parametrize("M", [4, 8])
def test_proj_classic_open_loop_c1(M, fused):
    run_proj_parity(Grid(32, 2), M, 30, method="proj_classic", fused=fused)


@pytest.mark.parametrize("fused", SCHEDULES)
@pytest.mark.parametrize("n,dim", [(31, 2), (23, 3), (1001, 1), (3, 1), (1, 1)])
def test_proj_qr_ragged_sizes(n, dim, fused):
    run_proj_parity(Grid(n, dim), 8, 14, dt=1e-2, fused=fused)


@pytest.mark.parametrize("M", [5, 6, 10, 12, 14, 16, 20, 28, 32])
def test_proj_qr_buckets_multi_trip_odd_n(M):
    """Every history bucket of the fused kernels (rolling passes, one-copy pass 3, split pass 3,
    rolling form) on an odd, multi-trip vector: 61^3 = 226,981 DOFs (three grid-stride trips per
    thread with a ragged last one, plus the odd scalar tail), through fill, downdates and the
    dynamic pass-3 claims."""
    run_proj_parity(Grid(61, 3), M, M + 4, dt=1e-2)


@pytest.mark.parametrize("fused", SCHEDULES)
@pytest.mark.parametrize("M", [4, 5, 6, 10, 14, 20, 28])
def test_proj_qr_misaligned_vectors_take_scalar_path(M, fused):
    run_proj_parity(Grid(33, 2), M, M + 6, misalign=True, fused=fused)


@pytest.mark.parametrize("fused", SCHEDULES)
def test_proj_qr_many_blocks_3d(fused):
    # 64^3 = 262,144 DOFs: hundreds of blocks, exercises the block-ordered reductions
    run_proj_parity(Grid(64, 3), 8, 12, fused=fused)


def test_proj_orthonormality_and_R_vs_oracle():
    from paper_2009_10863_b200 import InitialGuess, ig_copy_history

    g = Grid(40, 2)
    M = 6
    seq = _seq(g, 15, dt=1e-2)
    ora = ProjQR(g.N, M)
    ig = InitialGuess(g.N, "proj_qr", M)
    for b, x, Ax in seq:
        ora.update(x, Ax)
        ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
        Bt, Xt, R = ig_copy_history(ig.h, M, g.N)
        d = ig.d
        B = Bt[:d].cpu().numpy().T
        assert np.max(np.abs(B.T @ B - np.eye(d))) <= 1e-12  # PIN-P4 on the GPU state
        # guesses, not bases, are unique (AMB-20); R and B~ agree with the oracle at the
        # well-conditioned level of this sequence
        assert np.max(np.abs(R.numpy()[:d, :d] - ora.R[:d, :d])) <= 1e-8 * np.max(np.abs(ora.R))
    ig.close()


def test_proj_rejection_and_zero_paths():
    from paper_2009_10863_b200 import InitialGuess

    N, M = 500, 3
    rng = np.random.default_rng(1)
    ig = InitialGuess(N, "proj_qr", M)
    ora = ProjQR(N, M)
    z = torch.zeros(N, dtype=torch.float64, device="cuda")
    ig.update(z, z)  # ||Ax|| = 0 at d = 0: skipped
    ora.update(np.zeros(N), np.zeros(N))
    assert ig.d == 0 == ora.d
    x0 = torch.full((N,), 7.0, dtype=torch.float64, device="cuda")
    ig.form_guess(torch.ones(N, dtype=torch.float64, device="cuda"), x0)
    assert torch.all(x0 == 7.0)  # d = 0: x0 untouched
    xs = [rng.standard_normal(N) for _ in range(M + 1)]
    A = lambda v: 3.0 * v + np.roll(v, 1)  # noqa: E731  any nonsingular operator
    for x in xs:
        ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(A(x)).cuda())
        ora.update(x, A(x))
    dup = 0.3 * xs[-1] - 2.0 * xs[-2]  # in the span after the downdate -> rejected
    ig.update(torch.from_numpy(dup).cuda(), torch.from_numpy(A(dup)).cuda())
    ora.update(dup, A(dup))
    st = ig.stats()
    assert st["admitted"] == 0 and ora.admitted is False
    assert ig.d == ora.d == M - 1
    b = rng.standard_normal(N)
    x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    ig.form_guess(torch.from_numpy(b).cuda(), x0)
    assert _rel(x0.cpu().numpy(), ora.form_guess(b, np.zeros(N))) <= TOL
    ig.close()


def test_proj_x0_may_alias_b():
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(20, 2)
    seq = _seq(g, 6, dt=1e-2)
    ora, ig = ProjQR(g.N, 4), InitialGuess(g.N, "proj_qr", 4)
    for b, x, Ax in seq:
        ora.update(x, Ax)
        ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
    b = seq[-1][0] * 1.01
    t = torch.from_numpy(b).cuda()
    ig.form_guess(t, t)
    assert _rel(t.cpu().numpy(), ora.form_guess(b, np.zeros(g.N))) <= TOL
    ig.close()


def test_independent_handles():
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(16, 2)
    s1, s2 = _seq(g, 8, dt=1e-2), _seq(g, 8, dt=3e-2)
    o1, o2 = ProjQR(g.N, 3), ProjQR(g.N, 5)
    h1, h2 = InitialGuess(g.N, "proj_qr", 3), InitialGuess(g.N, "proj_qr", 5)
    for (b1, x1, a1), (b2, x2, a2) in zip(s1, s2):
        for o, h, b, x, a in ((o1, h1, b1, x1, a1), (o2, h2, b2, x2, a2)):
            x0 = torch.zeros(g.N, dtype=torch.float64, device="cuda")
            h.form_guess(torch.from_numpy(b).cuda(), x0)
            assert _rel(x0.cpu().numpy(), o.form_guess(b, np.zeros(g.N))) <= TOL
            o.update(x, a)
            h.update(torch.from_numpy(x).cuda(), torch.from_numpy(a).cuda())
    h1.close()
    h2.close()


# ------------------------------------------------------------------ extrapolation
@pytest.mark.parametrize("m,M", [(2, 4), (3, 8), (2, 12), (3, 16), (5, 30), (0, 1), (1, 2), (7, 8)])
def test_extrap_weights_match_exact_rational(m, M):
    from paper_2009_10863_b200 import InitialGuess

    ig = InitialGuess(10, "extrap_ls", M, m)
    for f in range(1, M + 1):
        w_o = warmup_weights(m, M, f)
        w_g = np.array(ig.weights(f))
        assert np.max(np.abs(w_g - w_o)) <= 4e-16 * max(1.0, np.abs(w_o).sum()) * M, f
    ig.close()


@pytest.mark.parametrize("m,M", [(2, 4), (3, 8), (3, 16), (5, 30), (4, 8)])
@pytest.mark.parametrize("zero_copy", [True, False])
def test_extrap_open_loop(m, M, zero_copy):
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(32, 2) if M <= 8 else Grid(45, 2)
    seq = _seq(g, M + 10)
    ora = ExtrapLS(g.N, M, m)
    ig = InitialGuess(g.N, "extrap_ls", M, m)
    for n, (b, x, Ax) in enumerate(seq):
        fallback = torch.full((g.N,), -3.0, dtype=torch.float64, device="cuda")
        if zero_copy:
            x0 = ig.next_slot()  # the solver would solve in place from the guess
            if n == 0:
                x0.copy_(fallback)  # the slot may be written only while it holds no history
        else:
            x0 = fallback
        ig.form_guess(None, x0)
        x0_o = ora.form_guess(b, np.full(g.N, -3.0))
        assert _rel(x0.cpu().numpy(), x0_o) <= TOL, f"step {n}"
        ora.update(x)
        if zero_copy:
            x0.copy_(torch.from_numpy(x))  # "solve" into the slot
            ig.update(x0)
            assert ig.bytes()[1] == 0  # zero-copy push
        else:
            ig.update(torch.from_numpy(x).cuda())
    ig.close()


@pytest.mark.parametrize("N", [1, 2, 3, 999, 4097])
def test_extrap_ragged(N):
    from paper_2009_10863_b200 import InitialGuess

    rng = np.random.default_rng(N)
    M, m = 6, 2
    ora, ig = ExtrapLS(N, M, m), InitialGuess(N, "extrap_ls", M, m)
    for n in range(9):
        x = rng.standard_normal(N)
        x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
        ig.form_guess(None, x0)
        assert _rel(x0.cpu().numpy(), ora.form_guess(None, np.zeros(N))) <= TOL
        ora.update(x)
        ig.update(torch.from_numpy(x).cuda())
    ig.close()


# ------------------------------------------------------------------ host-buffer (end-to-end) entry points
def test_host_entry_points_match_oracle():
    from paper_2009_10863_b200 import InitialGuess, ig_form_guess_host, ig_update_host

    g = Grid(24, 2)
    seq = _seq(g, 12, dt=1e-2)
    op, oe = ProjQR(g.N, 4), ExtrapLS(g.N, 4, 2)
    hp, he = InitialGuess(g.N, "proj_qr", 4), InitialGuess(g.N, "extrap_ls", 4, 2)
    for b, x, Ax in seq:
        for o, h in ((op, hp), (oe, he)):
            x0 = torch.zeros(g.N, dtype=torch.float64).pin_memory()
            ig_form_guess_host(h.h, torch.from_numpy(b), x0)
            assert _rel(x0.numpy(), o.form_guess(b, np.zeros(g.N))) <= TOL
            o.update(x, Ax)
            ig_update_host(h.h, torch.from_numpy(x), torch.from_numpy(Ax))
    hp.close()
    he.close()


def test_host_entry_points_accept_pageable_memory():
    """The host-buffer calls also take ordinary (pageable) host arrays -- slower transfers, same
    results as pinned buffers."""
    from paper_2009_10863_b200 import InitialGuess, ig_form_guess_batch_host, ig_update_batch_host

    g = Grid(20, 2)
    seq = _seq(g, 8, dt=1e-2)
    A = [InitialGuess(g.N, "proj_qr", 4), InitialGuess(g.N, "extrap_ls", 4, 2)]
    B = [InitialGuess(g.N, "proj_qr", 4), InitialGuess(g.N, "extrap_ls", 4, 2)]
    for b, x, Ax in seq:
        xa = [torch.zeros(g.N, dtype=torch.float64) for _ in A]  # pageable
        xb = [torch.zeros(g.N, dtype=torch.float64).pin_memory() for _ in B]
        ig_form_guess_batch_host(A, [torch.from_numpy(b.copy()), None], xa)
        ig_form_guess_batch_host(B, [torch.from_numpy(b).pin_memory(), None], xb)
        for u, v in zip(xa, xb):
            assert torch.equal(u, v)
        ig_update_batch_host(A, [torch.from_numpy(x.copy())] * 2, [torch.from_numpy(Ax.copy()), None])
        ig_update_batch_host(B, [torch.from_numpy(x).pin_memory()] * 2, [torch.from_numpy(Ax).pin_memory(), None])
    for h in A + B:
        h.close()


def test_batch_host_entry_points_match_single_calls_and_oracle():
    """ig_form_guess_batch_host / ig_update_batch_host (transfers of the fields overlapped on two
    streams per handle) against the device-buffer single calls on twin handles, bitwise, and the
    oracle within 1e-11 -- including the fill phase (d = 0: the fallback x0 must come back
    unchanged), a restart of a CLASSIC field and a zero right-hand side."""
    from paper_2009_10863_b200 import InitialGuess, ig_form_guess_batch_host, ig_update_batch_host

    g = Grid(26, 2)
    N = g.N
    seq = _seq(g, 14, dt=1e-2)
    specs = [("extrap_ls", 4, 2), ("proj_qr", 5, 0), ("extrap_sparse", 6, 1), ("proj_classic", 3, 0)]
    A = [InitialGuess(N, m, M, p) for m, M, p in specs]
    B = [InitialGuess(N, m, M, p) for m, M, p in specs]
    oras = [ExtrapLS(N, 4, 2), ProjQR(N, 5), None, ProjClassic(N, 3)]
    for n, (b, x, Ax) in enumerate(seq):
        if n == 5:
            b = np.zeros(N)  # zero right-hand side: projection guess 0
        fb = np.full(N, -2.5)
        x0h = [torch.from_numpy(fb.copy()).pin_memory() for _ in specs]
        bh = [torch.from_numpy(b).pin_memory() if m.startswith("proj") else None for m, _, _ in specs]
        ig_form_guess_batch_host(A, bh, x0h)
        for i, ((m, _, _), h) in enumerate(zip(specs, B)):
            x0d = torch.from_numpy(fb.copy()).cuda()
            h.form_guess(torch.from_numpy(b).cuda() if m.startswith("proj") else None, x0d)
            assert torch.equal(x0h[i], x0d.cpu()), (n, specs[i])
            if oras[i] is not None:
                assert _rel(x0h[i].numpy(), oras[i].form_guess(b, fb)) <= TOL, (n, specs[i])
        xh = [torch.from_numpy(x).pin_memory() for _ in specs]
        Axh = [torch.from_numpy(Ax).pin_memory() if m.startswith("proj") else None for m, _, _ in specs]
        ig_update_batch_host(A, xh, Axh)
        for (m, _, _), h, o in zip(specs, B, oras):
            h.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda() if m.startswith("proj") else None)
            if o is not None:
                o.update(x, Ax)
    for ha, hb in zip(A, B):
        assert ha.save_state() == hb.save_state()
        ha.close()
        hb.close()


# ------------------------------------------------------------------ full C2 size (bench launch config)
@pytest.mark.slow
def test_c2_full_size_parity():
    """configs[1]: 3D 128^3 (2,097,152 DOFs), QR(8) and EXTRAP(3,8) exactly as bench.py launches them."""
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(128, 3)
    steps = 12
    op, oe = ProjQR(g.N, 8), ExtrapLS(g.N, 8, 3)
    hp, he = InitialGuess(g.N, "proj_qr", 8), InitialGuess(g.N, "extrap_ls", 8, 3)
    x_prev = np.zeros(g.N)
    for n in range(steps):
        b, x, Ax = (t.numpy() for t in manufactured_step(g, n))
        tb, tx, tA = (torch.from_numpy(v).cuda() for v in (b, x, Ax))
        x0p = torch.from_numpy(x_prev).cuda()
        hp.form_guess(tb, x0p)
        assert _rel(x0p.cpu().numpy(), op.form_guess(b, x_prev)) <= TOL
        x0e = he.next_slot()
        if n == 0:
            x0e.copy_(torch.from_numpy(x_prev))
        he.form_guess(None, x0e)
        assert _rel(x0e.cpu().numpy(), oe.form_guess(b, x_prev)) <= TOL
        op.update(x, Ax)
        hp.update(tx, tA)
        oe.update(x)
        x0e.copy_(tx)
        he.update(x0e)
        assert hp.d == op.d
        x_prev = x
    hp.close()
    he.close()


@pytest.mark.slow
def test_2p24_open_loop_parity():
    """Open-loop oracle parity at 2^24 DOFs (3D 256^3, HBM-scale: 128 MB vectors, the B~/X~
    history 2 GB) with QR(8) and EXTRAP(3,8) in the bench launch configuration: every guess vs
    the oracle, d identical, through history fill and 3 downdates (multi-trip passes and the
    dynamic pass-3 tail at a size where no vector fits in L2)."""
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(256, 3)
    assert g.N == 1 << 24
    M, steps = 8, 12
    op, oe = ProjQR(g.N, M), ExtrapLS(g.N, M, 3)
    hp, he = InitialGuess(g.N, "proj_qr", M), InitialGuess(g.N, "extrap_ls", M, 3)
    x_prev = np.zeros(g.N)
    for n in range(steps):
        b, x, Ax = (t.numpy() for t in manufactured_step(g, n))
        tb, tx, tA = (torch.from_numpy(v).cuda() for v in (b, x, Ax))
        x0p = torch.from_numpy(x_prev).cuda()
        hp.form_guess(tb, x0p)
        e = _rel(x0p.cpu().numpy(), op.form_guess(b, x_prev))
        assert e <= TOL, f"step {n}: QR guess {e:.3e}"
        x0e = torch.from_numpy(x_prev).cuda()
        he.form_guess(None, x0e)
        e = _rel(x0e.cpu().numpy(), oe.form_guess(b, x_prev))
        assert e <= TOL, f"step {n}: EXTRAP guess {e:.3e}"
        op.update(x, Ax)
        hp.update(tx, tA)
        oe.update(x)
        he.update(tx)
        assert hp.d == op.d
        x_prev = x
        del tb, tx, tA, x0p, x0e
    hp.close()
    he.close()


@pytest.mark.parametrize("M", [12, 20])
def test_2p24_open_loop_parity_large_m(M):
    """As test_2p24_open_loop_parity for the large-vector kernels of the M = 9..12 and 17..24
    buckets (k_update_fused<12, 2>; k_form_fused<24, 2, RF>, k_update_fused<24, 2> with rolling
    passes 1-2 and the split pass 3): QR(M) at 2^24 DOFs through history fill and 3 downdates,
    every guess vs the oracle."""
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(256, 3)
    steps = M + 3
    op, hp = ProjQR(g.N, M), InitialGuess(g.N, "proj_qr", M)
    x_prev = np.zeros(g.N)
    for n in range(steps):
        b, x, Ax = (t.numpy() for t in manufactured_step(g, n))
        tb, tx, tA = (torch.from_numpy(v).cuda() for v in (b, x, Ax))
        x0p = torch.from_numpy(x_prev).cuda()
        hp.form_guess(tb, x0p)
        e = _rel(x0p.cpu().numpy(), op.form_guess(b, x_prev))
        assert e <= TOL, f"step {n}: QR guess {e:.3e}"
        op.update(x, Ax)
        hp.update(tx, tA)
        assert hp.d == op.d
        x_prev = x
        del tb, tx, tA, x0p
    hp.close()


# ------------------------------------------------------------------ sparse extrapolation (NEXT row f2)
@pytest.mark.parametrize("m,M", [(2, 8), (3, 8), (3, 16), (2, 12), (5, 30), (0, 4), (3, 4)])
def test_sparse_weights_match_exact_cpqr(m, M):
    from oracle import sparse_weights
    from paper_2009_10863_b200 import InitialGuess

    ig = InitialGuess(10, "extrap_sparse", M, m)
    for f in range(1, M + 1):
        w_o = sparse_weights(min(m, f - 1), f)
        w_g = np.array(ig.weights(f))
        assert np.array_equal(w_g != 0.0, w_o != 0.0), (f, w_g, w_o)  # same selected history
        assert np.max(np.abs(w_g - w_o)) <= 1e-14 * max(1.0, np.abs(w_o).sum()), f
    ig.close()


@pytest.mark.parametrize("m,M", [(2, 8), (3, 16)])
def test_sparse_open_loop_and_bytes(m, M):
    from oracle import ExtrapSparse
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(30, 2)
    seq = _seq(g, M + 6)
    ora = ExtrapSparse(g.N, M, m)
    ig = InitialGuess(g.N, "extrap_sparse", M, m)
    for n, (b, x, Ax) in enumerate(seq):
        x0 = ig.next_slot()
        if n == 0:
            x0.zero_()
        ig.form_guess(None, x0)
        assert _rel(x0.cpu().numpy(), ora.form_guess(b, np.zeros(g.N))) <= TOL, n
        if n >= M:  # steady: (m+2) values per element (Table 1) with the zero-copy push
            fb, ub = ig.bytes()
            assert fb == (m + 2) * 8 * g.N and ub == 0
        ora.update(x)
        x0.copy_(torch.from_numpy(x))
        ig.update(x0)
        if n >= M:
            assert ig.bytes()[1] == 0
    ig.close()


# ------------------------------------------------------------------ CUDA-graph capture (row f3)
@pytest.mark.parametrize("fused", SCHEDULES)
def test_projection_step_is_graph_capturable(fused):
    """All projection control state lives on the device (no host sync on the hot path), so one
    form+update step can be captured once and replayed every time step with new data copied into
    the captured buffers."""
    from paper_2009_10863_b200 import InitialGuess, ig_set_stream

    g = Grid(48, 2)
    M = 6
    seq = _seq(g, 3 * M, dt=1e-2)
    ora = ProjQR(g.N, M)
    ig = InitialGuess(g.N, "proj_qr", M, fused=fused)
    b_s, x0_s, x_s, A_s = (torch.zeros(g.N, dtype=torch.float64, device="cuda") for _ in range(4))
    n0 = M + 1
    for b, x, Ax in seq[:n0]:  # fill the history with ordinary calls
        ora.update(x, Ax)
        ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    ig_set_stream(ig.h, s)
    with torch.cuda.graph(graph, stream=s):
        ig.form_guess(b_s, x0_s)
        ig.update(x_s, A_s)
    for b, x, Ax in seq[n0:]:
        b_s.copy_(torch.from_numpy(b))
        x_s.copy_(torch.from_numpy(x))
        A_s.copy_(torch.from_numpy(Ax))
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        ref = ora.form_guess(b, np.zeros(g.N))
        assert _rel(x0_s.cpu().numpy(), ref) <= TOL
        ora.update(x, Ax)
        assert ig.d == ora.d
    ig.close()


def test_history_in_caller_storage():
    """ig_create_ext: the history slabs live in a torch-owned allocation (caching allocator)."""
    from paper_2009_10863_b200 import IG_EXTRAP_LS, IG_PROJ_QR, InitialGuess, ig_storage_bytes

    g = Grid(30, 2)
    seq = _seq(g, 12, dt=1e-2)
    M = 5
    sp = torch.empty(ig_storage_bytes(g.N, IG_PROJ_QR, M), dtype=torch.uint8, device="cuda")
    se = torch.empty(ig_storage_bytes(g.N, IG_EXTRAP_LS, M), dtype=torch.uint8, device="cuda")
    hp = InitialGuess(g.N, "proj_qr", M, storage=sp)
    he = InitialGuess(g.N, "extrap_ls", M, 2, storage=se)
    op, oe = ProjQR(g.N, M), ExtrapLS(g.N, M, 2)
    for b, x, Ax in seq:
        for o, h in ((op, hp), (oe, he)):
            x0 = torch.zeros(g.N, dtype=torch.float64, device="cuda")
            h.form_guess(torch.from_numpy(b).cuda(), x0)
            assert _rel(x0.cpu().numpy(), o.form_guess(b, np.zeros(g.N))) <= TOL
            o.update(x, Ax)
            h.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
    hp.close()
    he.close()
    with pytest.raises(Exception):
        InitialGuess(g.N, "proj_qr", M, storage=sp[:100])  # too small -> IG_E_ARG


# ------------------------------------------------------------------ multi-field batch (row f4)
def test_multi_field_batch_one_launch_for_the_velocity_fields():
    """u_x, u_y, u_z by EXTRAP (different schemes) and p by QR, as the paper's solver keeps one
    history space per field (Table 7): one batched call, the three
    extrapolation guesses share one kernel launch, every guess matches its oracle."""
    from oracle import ExtrapSparse
    from paper_2009_10863_b200 import InitialGuess, ig_form_guess_batch, ig_total_launches, ig_update_batch

    g = Grid(30, 2)
    N = g.N
    specs = [("extrap_ls", 8, 3), ("extrap_ls", 4, 2), ("extrap_sparse", 8, 2), ("proj_qr", 6, 0)]
    oras = [ExtrapLS(N, 8, 3), ExtrapLS(N, 4, 2), ExtrapSparse(N, 8, 2), ProjQR(N, 6)]
    igs = [InitialGuess(N, m, M, p) for m, M, p in specs]
    seqs = [_seq(g, 14, dt=dt) for dt in (1e-2, 2e-2, 3e-2, 1e-2)]
    for n in range(14):
        bs = [torch.from_numpy(s[n][0]).cuda() for s in seqs]
        x0s = [torch.zeros(N, dtype=torch.float64, device="cuda") for _ in specs]
        l0 = ig_total_launches()
        ig_form_guess_batch(igs, bs, x0s)
        torch.cuda.synchronize()
        if n >= 8:
            assert ig_total_launches() - l0 == 2  # one batched extrapolation launch + one QR launch
        for o, s, x0 in zip(oras, seqs, x0s):
            assert _rel(x0.cpu().numpy(), o.form_guess(s[n][0], np.zeros(N))) <= TOL, n
        xs = [torch.from_numpy(s[n][1]).cuda() for s in seqs]
        As = [torch.from_numpy(s[n][2]).cuda() for s in seqs]
        ig_update_batch(igs, xs, As)
        for o, s in zip(oras, seqs):
            o.update(s[n][1], s[n][2])
    for ig in igs:
        ig.close()


@pytest.mark.parametrize("eps", [1e-4, 1e-6, 0.0])
def test_admission_tolerance_parity(eps):
    """ig_set_admit_tol (AMB-3): with a tolerance above the sequence's rho ~ 1e-6..1e-5 most pairs
    are rejected; the CUDA path must take exactly the oracle's decisions."""
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(32, 2)
    seq = _seq(g, 20)
    ora = ProjQR(g.N, 6, eps)
    ig = InitialGuess(g.N, "proj_qr", 6, eps=eps)
    ds = []
    for b, x, Ax in seq:
        x0 = torch.zeros(g.N, dtype=torch.float64, device="cuda")
        ig.form_guess(torch.from_numpy(b).cuda(), x0)
        assert _rel(x0.cpu().numpy(), ora.form_guess(b, np.zeros(g.N))) <= TOL
        ora.update(x, Ax)
        ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
        st = ig.stats()
        # a decision with |rho/eps - 1| < 1e-9 is ill-posed (rounding may flip it);
        # the sequence must not contain one, or the exact comparison below would mean nothing
        assert eps == 0.0 or abs(ora.rho / eps - 1.0) > 1e-9
        assert abs(st["rho"] - ora.rho) <= 1e-7 * max(ora.rho, 1e-300)  # same rho (cancellation-limited)
        assert (st["d"], bool(st["admitted"])) == (ora.d, ora.admitted)
        ds.append(ora.d)
    if eps >= 1e-4:
        assert max(ds) < 6  # the tolerance really rejected pairs
    ig.close()


# ------------------------------------------------------------------ full-size properties (configs[2] scale)
@pytest.mark.slow
@pytest.mark.parametrize("N,M,p", [pytest.param(1 << 27, 4, 2, id="2^27-M4"),
                                   pytest.param(1 << 27, 8, 3, id="C3-2^27-M8"),
                                   pytest.param(1 << 28, 16, 3, id="C4-2^28-M16")])
def test_properties_at_full_size(N, M, p):
    """configs[2] / configs[3] sizes (2^27 / 2^28 DOFs per GPU, the C3 / C4 histories) in the bench
    launch configuration, where the oracle cannot run whole: properties that hold at any size --
    B~ orthonormal, b = B~_j gives x0 = X~_j, and extrapolation
    sampled element by element against Eq. EXTRAPEXPN with the oracle's exact-rational weights.
    The histories live in caller storage (ig_create_ext), read in place (C4: ~110 GB in HBM)."""
    from paper_2009_10863_b200 import IG_EXTRAP_LS, IG_PROJ_QR, InitialGuess, ig_storage_bytes

    need = ig_storage_bytes(N, IG_PROJ_QR, M) + ig_storage_bytes(N, IG_EXTRAP_LS, M) + 6 * 8 * N
    free, _ = torch.cuda.mem_get_info()
    if need > 0.95 * free:
        pytest.skip(f"needs {need / 1e9:.0f} GB of HBM, {free / 1e9:.0f} GB free")
    gen = torch.Generator(device="cuda").manual_seed(10863)
    sp = torch.empty(ig_storage_bytes(N, IG_PROJ_QR, M) // 8, dtype=torch.float64, device="cuda")
    se = torch.empty(ig_storage_bytes(N, IG_EXTRAP_LS, M) // 8, dtype=torch.float64, device="cuda")
    ig = InitialGuess(N, "proj_qr", M, storage=sp)
    ie = InitialGuess(N, "extrap_ls", M, p, storage=se)
    idx = torch.randint(0, N, (4096,), generator=gen, device="cuda")
    window = []  # sampled x values of the extrapolation window, oldest first
    for _ in range(M + 2):
        x = torch.randn(N, dtype=torch.float64, device="cuda", generator=gen)
        Ax = torch.randn(N, dtype=torch.float64, device="cuda", generator=gen)
        ig.update(x, Ax)
        ie.update(x)
        window = (window + [x[idx].cpu().numpy()])[-M:]
        del x, Ax
    assert ig.d == M
    ld = sp.numel() // (2 * M)
    Bt = sp[: M * ld].view(M, ld)[:, :N]
    Xt = sp[M * ld:].view(M, ld)[:, :N]
    G = Bt @ Bt.T
    assert torch.max(torch.abs(G - torch.eye(M, dtype=torch.float64, device="cuda"))).item() <= 1e-12
    x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    for j in range(M):
        bj = Bt[j].contiguous()
        ig.form_guess(bj, x0)
        err = torch.linalg.vector_norm(x0 - Xt[j]) / torch.linalg.vector_norm(Xt[j])
        assert err.item() <= 1e-11, j
        del bj
    ie.form_guess(None, x0)
    beta = warmup_weights(p, M, M)
    ref = np.zeros(idx.numel())
    for k in range(M):  # Eq. EXTRAPEXPN, oldest first, one element at a time
        ref = ref + beta[k] * window[k]
    got = x0[idx].cpu().numpy()
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref)) * np.abs(beta).sum()
    ig.close()
    ie.close()


# ------------------------------------------------------------------ planner CTA edge grids
@pytest.mark.parametrize("grid", [1, 2, 3, 37])
@pytest.mark.parametrize("M", [1, 2, 8, 12, 20, 30])
def test_planner_cta_and_single_cta_grids(grid, M):
    """The last CTA of a QR update grid is the planner (R update + Givens plan); with a
    one-CTA grid the plan runs serially in CTA 0.  Grids of 1, 2 (one streaming CTA + planner),
    3 and 37 CTAs through fill and downdates: every guess matches the oracle, d identical, and the
    history equals the full-grid run's to rounding."""
    from paper_2009_10863_b200 import InitialGuess, ig_set_grid_limit

    g = Grid(37, 2)  # N = 1369: ragged, several trips per thread on small grids
    seq = _seq(g, 2 * M + 4, dt=1e-2)
    ora = ProjQR(g.N, M)
    ig = InitialGuess(g.N, "proj_qr", M)
    ig_set_grid_limit(ig.h, grid)
    ref = InitialGuess(g.N, "proj_qr", M)
    x_prev = np.zeros(g.N)
    for n, (b, x, Ax) in enumerate(seq):
        x0 = torch.from_numpy(x_prev).cuda()
        x0r = x0.clone()
        ig.form_guess(torch.from_numpy(b).cuda(), x0)
        ref.form_guess(torch.from_numpy(b).cuda(), x0r)
        e = _rel(x0.cpu().numpy(), ora.form_guess(b, x_prev))
        assert e <= TOL, f"grid {grid} step {n}: {e:.3e}"
        assert _rel(x0.cpu().numpy(), x0r.cpu().numpy()) <= TOL
        ora.update(x, Ax)
        ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
        ref.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
        assert ig.d == ora.d
        x_prev = x
    ig.close()
    ref.close()
