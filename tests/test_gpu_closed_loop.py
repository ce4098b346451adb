"""Closed loop (BASELINE north_star): each side runs its own harness CG with its own guesses on
the configs[0] sequence (2D 32x32 Helmholtz, prescribed smooth RHS, 40 steps, INITRESID
eps = 1e-8, fallback LAST); per-step CG iteration counts of the CUDA path and the oracle must
agree within +-1.  Also checks the qualitative ordering the paper reports (§6.3):
projection needs fewer iterations than extrapolation, which needs fewer than LAST."""

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
        dev = "cuda" if side == "gpu" else "cpu"
        obj = make_gpu() if side == "gpu" else make_oracle()
        x_prev = torch.zeros(g.N, dtype=torch.float64, device=dev)
        for n in range(steps):
            b = prescribed_rhs(g, n, dt, device=dev)
            x0 = x_prev.clone()
            if obj is not None:
                if side == "gpu":
                    obj.form_guess(b, x0)
                else:
                    x0 = torch.from_numpy(obj.form_guess(b.numpy(), x0.numpy()))
            x, it, _, _ = pcg(g, b, x0)
            its[side].append(it)
            if obj is not None:
                Ax = helmholtz_apply(g, x)
                if side == "gpu":
                    obj.update(x, Ax)
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


@pytest.mark.parametrize("method,M,p", [("proj_qr", 8, 0), ("extrap_ls", 4, 2), ("extrap_ls", 8, 3),
                                        ("proj_classic", 4, 0)])
def test_closed_loop_iterations_within_one(method, M, p):
    from oracle import ProjClassic
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(32, 2)
    mk_o = {"proj_qr": lambda: ProjQR(g.N, M), "extrap_ls": lambda: ExtrapLS(g.N, M, p),
            "proj_classic": lambda: ProjClassic(g.N, M)}[method]
    it_g, it_o = _run(g, 40, mk_o, lambda: InitialGuess(g.N, method, M, p))
    assert np.max(np.abs(it_g - it_o)) <= 1, (it_g.tolist(), it_o.tolist())


def test_paper_ordering_of_methods():
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(32, 2)
    last, _ = _run(g, 40, lambda: None, lambda: None)
    qr, _ = _run(g, 40, lambda: ProjQR(g.N, 8), lambda: InitialGuess(g.N, "proj_qr", 8))
    ex, _ = _run(g, 40, lambda: ExtrapLS(g.N, 8, 3), lambda: InitialGuess(g.N, "extrap_ls", 8, 3))
    tail = slice(10, None)  # after the histories filled
    assert qr[tail].mean() < ex[tail].mean() < last[tail].mean(), (qr.mean(), ex.mean(), last.mean())
