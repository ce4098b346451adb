"""Closed loop (BASELINE north_star "downstream CG iteration counts must agree within +-1"; SURVEY
§8(c) closed-loop protocol) on the configs[0] sequence (2D 32x32 Helmholtz, prescribed smooth RHS,
40 steps, Jacobi-PCG INITRESID eps = 1e-8, fallback LAST), for all five
methods (QR, EXTRAP, CLASSIC, SPEXTRAP).  Both sides run the SAME harness CG arithmetic (torch
fp64 on the host): the CUDA library's guesses are copied out and its solutions copied back, so the
comparison isolates the initial-guess implementations.  Three protocols:

* identical systems, oracle-driven: the oracle's closed loop feeds both histories; per step the CG
  from each side's guess must take the same count +-1;
* identical systems, CUDA-driven ("shadowed"): the CUDA path's OWN closed loop (its guesses feed
  its CG, its solutions feed its history) with the oracle fed the same pairs: every step's guess
  within 1e-11 of the oracle's and the counts within +-1;
* fully independent closed loops: per-step counts within +-1 and the same steady-state mean.

The fully closed loop is chaotic at the CG stopping test (DESIGN.md AMB-21): the ORACLE against
itself, with its guesses perturbed at the 1e-15 rounding level, drifts by up to 3 (QR(8)) / 2
(EXTRAP(3,8)) iterations per step (tests/golden/closed_loop_envelope.json, written by
scripts/closed_loop_envelope.py from oracle/ only).  The +-1 of the independent loops therefore
holds for this implementation pair, not for every correct one; the shadowed protocol is the
per-step check that stays well posed.  Also checks the qualitative ordering the paper reports
(§6.3): projection needs fewer iterations than extrapolation, which needs
fewer than LAST."""

import numpy as np
import pytest
import torch

from oracle import ExtrapLS, ProjQR
from workloads import Grid, helmholtz_apply, prescribed_rhs
from workloads.cg import pcg

pytestmark = pytest.mark.gpu


def _run(g, steps, make_oracle, make_gpu, dt=1e-3):
    its = {"gpu": [], "ora": []}
    for side in ("gpu", "ora"):
        obj = make_gpu() if side == "gpu" else make_oracle()
        x_prev = torch.zeros(g.N, dtype=torch.float64)
        for n in range(steps):
            b = prescribed_rhs(g, n, dt)
            x0 = x_prev.clone()
            if obj is not None:
                if side == "gpu":
                    x0d = x0.cuda()
                    obj.form_guess(b.cuda(), x0d)
                    x0 = x0d.cpu()
                else:
                    x0 = torch.from_numpy(obj.form_guess(b.numpy(), x0.numpy()))
            x, it, _, _ = pcg(g, b, x0)
            its[side].append(it)
            if obj is not None:
                Ax = helmholtz_apply(g, x)
                if side == "gpu":
                    obj.update(x.cuda(), Ax.cuda())
                else:
                    obj.update(x.numpy(), Ax.numpy())
            x_prev = x
        if side == "gpu" and obj is not None:
            obj.close()
    return np.array(its["gpu"]), np.array(its["ora"])


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


METHODS = [("proj_qr", 8, 0), ("extrap_ls", 4, 2), ("extrap_ls", 8, 3), ("proj_classic", 4, 0),
           ("extrap_sparse", 8, 3)]


def _makers(g, method, M, p):
    from oracle import ExtrapSparse, ProjClassic
    from paper_2009_10863_b200 import InitialGuess

    mk_o = {"proj_qr": lambda: ProjQR(g.N, M), "extrap_ls": lambda: ExtrapLS(g.N, M, p),
            "proj_classic": lambda: ProjClassic(g.N, M), "extrap_sparse": lambda: ExtrapSparse(g.N, M, p)}[method]
    return mk_o, (lambda: InitialGuess(g.N, method, M, p))


# Downstream iterations on IDENTICAL systems: the oracle's closed loop drives the history (the
# CUDA library receives the same (x_n, A x_n) pairs); at every step CG runs from each side's
# guess for the same b_n.  Counts must agree within +-1 (north_star).
@pytest.mark.parametrize("method,M,p", METHODS)
def test_downstream_iterations_within_one(method, M, p):
    g = Grid(32, 2)
    mk_o, mk_g = _makers(g, method, M, p)
    ora, lib = mk_o(), mk_g()
    x_prev = torch.zeros(g.N, dtype=torch.float64)
    diffs = []
    for n in range(40):
        b = prescribed_rhs(g, n, 1e-3)
        x0o = torch.from_numpy(ora.form_guess(b.numpy(), x_prev.numpy()))
        x0g = x_prev.clone().cuda()
        lib.form_guess(b.cuda(), x0g)
        x, it_o, _, _ = pcg(g, b, x0o)
        _, it_g, _, _ = pcg(g, b, x0g.cpu())
        diffs.append(it_g - it_o)
        Ax = helmholtz_apply(g, x)
        ora.update(x.numpy(), Ax.numpy())
        lib.update(x.cuda(), Ax.cuda())
        x_prev = x
    lib.close()
    assert max(abs(d) for d in diffs) <= 1, diffs


# GPU-driven identical systems ("shadowed" closed loop): the CUDA path runs its own closed loop; the
# oracle receives the same (x_n, A x_n) pairs, so every step is an open-loop parity point.
@pytest.mark.parametrize("method,M,p", METHODS)
def test_shadowed_closed_loop(method, M, p):
    g = Grid(32, 2)
    mk_o, mk_g = _makers(g, method, M, p)
    ora, lib = mk_o(), mk_g()
    x_prev = torch.zeros(g.N, dtype=torch.float64)
    diffs, rels = [], []
    for n in range(40):
        b = prescribed_rhs(g, n, 1e-3)
        x0g = x_prev.clone().cuda()
        lib.form_guess(b.cuda(), x0g)
        x0g = x0g.cpu()
        x0o = torch.from_numpy(ora.form_guess(b.numpy(), x_prev.numpy()))
        rels.append(float(torch.linalg.vector_norm(x0g - x0o)) / max(float(torch.linalg.vector_norm(x0o)), 1e-300))
        x, it_g, _, _ = pcg(g, b, x0g)  # the CUDA path's guess drives the loop
        _, it_o, _, _ = pcg(g, b, x0o)
        diffs.append(it_g - it_o)
        Ax = helmholtz_apply(g, x)
        lib.update(x.cuda(), Ax.cuda())
        ora.update(x.numpy(), Ax.numpy())
        x_prev = x
    lib.close()
    assert max(rels) <= 1e-11, max(rels)
    assert max(abs(d) for d in diffs) <= 1, diffs


# Fully independent closed loops (each side feeds back its own solutions): north_star's +-1 per
# step, and the same steady-state mean.  See the module docstring / AMB-21 for why this is a
# property of the implementation pair (the oracle's own rounding-level envelope is wider).
@pytest.mark.parametrize("method,M,p", METHODS)
def test_closed_loop_iterations_within_one(method, M, p):
    g = Grid(32, 2)
    mk_o, mk_g = _makers(g, method, M, p)
    it_g, it_o = _run(g, 40, mk_o, mk_g)
    assert np.max(np.abs(it_g - it_o)) <= 1, (it_g.tolist(), it_o.tolist())
    assert abs(it_g[10:].mean() - it_o[10:].mean()) <= 0.5


def test_paper_ordering_of_methods():
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(32, 2)
    last, _ = _run(g, 40, lambda: None, lambda: None)
    qr, _ = _run(g, 40, lambda: ProjQR(g.N, 8), lambda: InitialGuess(g.N, "proj_qr", 8))
    ex, _ = _run(g, 40, lambda: ExtrapLS(g.N, 8, 3), lambda: InitialGuess(g.N, "extrap_ls", 8, 3))
    tail = slice(10, None)  # after the histories filled
    assert qr[tail].mean() < ex[tail].mean() < last[tail].mean(), (qr.mean(), ex.mean(), last.mean())


# Second workload: one time step of an INS-like solver
# = three velocity components solved with a Helmholtz operator of large shift (gamma/(nu dt)),
# guessed by EXTRAP, plus a pressure Poisson solve (sigma = 0), guessed by QR -- four history
# spaces, one batched guess call and one batched update call per step.  Downstream iterations of
# every field on identical systems within +-1 of the oracle; the pressure projection must beat
# LAST by a wide margin and the velocity extrapolation must not lose to LAST.
def test_velocity_pressure_fields_batched():
    from paper_2009_10863_b200 import InitialGuess, ig_form_guess_batch, ig_update_batch

    n, steps, dt = 32, 30, 1e-3
    gv = Grid(n, 2, sigma=1e3)  # velocity Helmholtz: shift gamma/(nu dt) dominates the Laplacian less than fully
    gp = Grid(n, 2, sigma=0.0)  # pressure Poisson
    grids = [gv, gv, gv, gp]
    specs = [("extrap_ls", 4, 2), ("extrap_ls", 4, 2), ("extrap_ls", 4, 2), ("proj_qr", 8, 0)]
    oras = [ExtrapLS(gv.N, 4, 2) for _ in range(3)] + [ProjQR(gp.N, 8)]
    libs = [InitialGuess(g.N, m, M, p) for g, (m, M, p) in zip(grids, specs)]
    offs = [0, 7, 13, 0]  # the velocity components see different (time-shifted) forcings
    x_prev = [torch.zeros(g.N, dtype=torch.float64) for g in grids]
    its = {"ora": [[] for _ in grids], "gpu": [[] for _ in grids], "last": [[] for _ in grids]}
    for t in range(steps):
        bs = [prescribed_rhs(g, t + o, dt) for g, o in zip(grids, offs)]
        x0g = [xp.clone().cuda() for xp in x_prev]
        ig_form_guess_batch(libs, [b.cuda() if m.startswith("proj") else None for b, (m, _, _) in zip(bs, specs)], x0g)
        xs, Axs = [], []
        for k, (g, b, o) in enumerate(zip(grids, bs, oras)):
            x0o = torch.from_numpy(o.form_guess(b.numpy(), x_prev[k].numpy()))
            x, it_o, _, _ = pcg(g, b, x0o)
            _, it_g, _, _ = pcg(g, b, x0g[k].cpu())
            _, it_l, _, _ = pcg(g, b, x_prev[k])
            its["ora"][k].append(it_o)
            its["gpu"][k].append(it_g)
            its["last"][k].append(it_l)
            Ax = helmholtz_apply(g, x)
            o.update(x.numpy(), Ax.numpy())
            xs.append(x)
            Axs.append(Ax)
            x_prev[k] = x
        ig_update_batch(libs, [x.cuda() for x in xs], [Ax.cuda() if m.startswith("proj") else None
                                                         for Ax, (m, _, _) in zip(Axs, specs)])
    for h in libs:
        h.close()
    for k in range(len(grids)):
        d = np.abs(np.array(its["gpu"][k]) - np.array(its["ora"][k]))
        assert d.max() <= 1, (k, its["gpu"][k], its["ora"][k])
    warm = slice(10, None)
    p_qr, p_last = np.mean(its["gpu"][3][warm]), np.mean(its["last"][3][warm])
    assert p_qr < 0.5 * p_last, (p_qr, p_last)
    for k in range(3):
        assert np.mean(its["gpu"][k][warm]) <= np.mean(its["last"][k][warm]), k
