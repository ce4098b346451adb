"""GPU: device-resident extrapolation window and captured multi-field time steps (SURVEY rows
f3/f4; include/ig.h "captured time steps").

* A handle with the device window (ig_set_device_ring) gives BITWISE the guesses of the host
  window at every fill (same kernels' arithmetic, same order), with copy and zero-copy pushes,
  and keeps its history across mode switches, reset and checkpoint/resume.
* One whole multi-field step -- pressure by QR(M) plus three velocity components by EXTRAP /
  SPEXTRAP, one history space per field (mixed schemes as Table 7,
  P:1643-1662) -- is captured ONCE into a CUDA graph and replayed every time step with the new
  data copied into the captured buffers: every guess matches the CPU oracle (north_star
  tolerance 1e-11), d matches, and the replay launches exactly the captured libig kernels.
"""

import copy

import numpy as np
import pytest
import torch

from oracle import ExtrapLS, ExtrapSparse, ProjClassic, ProjQR
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


@pytest.mark.parametrize("method,M,p", [("extrap_ls", 8, 3), ("extrap_ls", 5, 4), ("extrap_sparse", 12, 3),
                                         ("extrap_ls", 1, 0), ("extrap_ls", 32, 5)])
@pytest.mark.parametrize("zero_copy", [False, True])
def test_device_window_is_bitwise_the_host_window(method, M, p, zero_copy):
    from paper_2009_10863_b200 import InitialGuess

    N = 4097  # ragged: odd length, several CTAs
    gen = torch.Generator(device="cuda").manual_seed(10863 + M)
    hh = InitialGuess(N, method, M, p)
    hd = InitialGuess(N, method, M, p)
    hd.set_device_ring(True)
    for n in range(2 * M + 3):
        fb = torch.randn(N, dtype=torch.float64, device="cuda", generator=gen)
        x0h, x0d = fb.clone(), fb.clone()
        hh.form_guess(None, x0h)
        hd.form_guess(None, x0d)
        assert torch.equal(x0h, x0d), f"step {n}"
        assert hh.bytes()[0] == hd.bytes()[0]
        x = torch.randn(N, dtype=torch.float64, device="cuda", generator=gen)
        if zero_copy:
            sh, sd = hh.next_slot(), hd.next_slot()
            sh.copy_(x)
            sd.copy_(x)
            hh.update(sh)
            hd.update(sd)
            assert hd.bytes()[1] == 0
        else:
            hh.update(x)
            hd.update(x)
        assert hh.d == hd.d == min(n + 1, M)
    hh.close()
    hd.close()


def test_device_window_switch_reset_and_checkpoint():
    from paper_2009_10863_b200 import InitialGuess

    N, M, p = 3000, 6, 2
    ora = ExtrapLS(N, M, p)
    h = InitialGuess(N, "extrap_ls", M, p)
    rng = np.random.default_rng(7)
    xs = [rng.standard_normal(N) for _ in range(30)]
    image = None
    for n, x in enumerate(xs):
        if n % 4 == 1:
            h.set_device_ring(n % 8 == 1)  # alternate host / device window mid-run
        x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
        h.form_guess(None, x0)
        assert _rel(x0.cpu().numpy(), ora.form_guess(None, np.zeros(N))) <= TOL, n
        if n == 17:
            image = h.save_state()
            saved = copy.deepcopy(ora)
        ora.update(x)
        h.update(torch.from_numpy(x).cuda())
    # resume from step 17 into a device-window handle
    h.reset()
    h.set_device_ring(True)
    assert h.d == 0
    h.load_state(image)
    assert h.d == saved.fill
    x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    h.form_guess(None, x0)
    assert _rel(x0.cpu().numpy(), saved.form_guess(None, np.zeros(N))) <= TOL
    h.reset()
    assert h.d == 0
    x0 = torch.full((N,), 3.0, dtype=torch.float64, device="cuda")
    h.form_guess(None, x0)
    assert torch.all(x0 == 3.0)  # empty window: x0 untouched (AMB-13)
    h.close()


def test_capturing_a_host_window_call_is_refused():
    from paper_2009_10863_b200 import IGError, InitialGuess, ig_capture_begin, ig_capture_end, ig_graph_destroy

    N = 1000
    h = InitialGuess(N, "extrap_ls", 4, 2)
    h.update(torch.ones(N, dtype=torch.float64, device="cuda"))
    s = torch.cuda.Stream()
    h.set_stream(s)
    x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ig_capture_begin(s)
    with pytest.raises(IGError) as ei:
        h.form_guess(None, x0)
    ig_graph_destroy(ig_capture_end(s))
    assert "ig_set_device_ring" in str(ei.value)
    h.close()


@pytest.mark.parametrize("n_side", [33, 100])
def test_captured_multi_field_step_matches_the_oracle(n_side):
    """Pressure by QR(8) (and CLASSIC(5)), velocity u_x/u_y/u_z by EXTRAP(3,8) / EXTRAP(2,4) /
    SPEXTRAP(2,8) -- the mixed setting of Table 7 -- captured once as ONE graph
    (every field's guess, then every field's update), replayed each step."""
    from paper_2009_10863_b200 import (CapturedStep, InitialGuess, ig_form_guess_batch, ig_total_launches,
                                       ig_update_batch)

    g = Grid(n_side, 2)
    N = g.N
    specs = [("proj_qr", 8, 0), ("extrap_ls", 8, 3), ("extrap_ls", 4, 2), ("extrap_sparse", 8, 2),
             ("proj_classic", 5, 0)]
    mk = {"proj_qr": lambda M, p: ProjQR(N, M), "proj_classic": lambda M, p: ProjClassic(N, M),
          "extrap_ls": lambda M, p: ExtrapLS(N, M, p), "extrap_sparse": lambda M, p: ExtrapSparse(N, M, p)}
    oras = [mk[m](M, p) for m, M, p in specs]
    s = torch.cuda.Stream()
    igs = [InitialGuess(N, m, M, p, stream=s) for m, M, p in specs]
    for h, (m, _, _) in zip(igs, specs):
        if m.startswith("extrap"):
            h.set_device_ring(True)
    F = len(specs)
    seqs = [_seq(g, 22, dt=dt) for dt in (1e-2, 2e-2, 1e-2, 3e-2, 1e-2)]
    bufs = {k: [torch.zeros(N, dtype=torch.float64, device="cuda") for _ in range(F)] for k in ("b", "x0", "x", "Ax")}
    torch.cuda.synchronize()
    with CapturedStep(s) as step:
        ig_form_guess_batch(igs, bufs["b"], bufs["x0"])
        ig_update_batch(igs, bufs["x"], bufs["Ax"])
    per_replay = None
    for n in range(22):
        with torch.cuda.stream(s):
            for f in range(F):
                b, x, Ax = seqs[f][n]
                bufs["b"][f].copy_(torch.from_numpy(b))
                bufs["x0"][f].zero_()  # fallback (projection at d = 0, extrapolation at fill 0)
                bufs["x"][f].copy_(torch.from_numpy(x))
                bufs["Ax"][f].copy_(torch.from_numpy(Ax))
        l0 = ig_total_launches()
        step.replay()
        s.synchronize()
        launched = ig_total_launches() - l0
        assert launched > 0
        if n == 0:
            per_replay = launched
        assert launched == per_replay
        for f, o in enumerate(oras):
            b, x, Ax = seqs[f][n]
            ref = o.form_guess(b, np.zeros(N))
            e = _rel(bufs["x0"][f].cpu().numpy(), ref)
            assert e <= TOL, f"step {n} field {specs[f]}: {e:.3e}"
            o.update(x, Ax)
        for f, (h, o) in enumerate(zip(igs, oras)):
            assert h.d == (o.d if hasattr(o, "d") else o.fill), f"step {n} field {specs[f]}"
    # 2 projection form + 2 projection update kernels, 1 batched extrapolation form, 1 batched push
    assert per_replay == 6
    step.close()
    for h in igs:
        h.close()


def test_sync_calls_refused_during_capture():
    """A synchronising read of a device window during capture would invalidate the caller's
    capture: it is refused (IG_E_STATE) and the capture stays usable."""
    from paper_2009_10863_b200 import IGError, InitialGuess, ig_capture_begin, ig_capture_end, ig_graph_destroy
    from paper_2009_10863_b200 import ig_graph_launch

    N = 2000
    s = torch.cuda.Stream()
    h = InitialGuess(N, "extrap_ls", 4, 2, stream=s)
    h.set_device_ring(True)
    x = torch.ones(N, dtype=torch.float64, device="cuda")
    x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ig_capture_begin(s)
    with pytest.raises(IGError):
        _ = h.d
    with pytest.raises(IGError):
        h.set_device_ring(False)
    h.form_guess(None, x0)
    h.update(x)
    g = ig_capture_end(s)
    for _ in range(3):
        ig_graph_launch(g, s)
    s.synchronize()
    assert h.d == 3
    assert torch.equal(x0, torch.ones(N, dtype=torch.float64, device="cuda"))  # 2 pushes of ones -> guess 1
    ig_graph_destroy(g)
    h.close()


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_replays_interleaved_with_eager_calls(seed):
    """A captured step (guess + update of a QR field and two extrapolation fields) replayed at
    random points of a sequence that also makes eager calls, resets and window-mode switches on
    the same handles: the graph reads and advances the same device state, so every guess matches
    the oracle's at every point."""
    from paper_2009_10863_b200 import CapturedStep, InitialGuess, ig_form_guess_batch, ig_update_batch

    rng = np.random.default_rng(seed)
    g = Grid(40, 2)
    N = g.N
    specs = [("proj_qr", 6, 0), ("extrap_ls", 6, 2), ("extrap_sparse", 8, 2)]
    mk = {"proj_qr": lambda M, p: ProjQR(N, M), "extrap_ls": lambda M, p: ExtrapLS(N, M, p),
          "extrap_sparse": lambda M, p: ExtrapSparse(N, M, p)}
    oras = [mk[m](M, p) for m, M, p in specs]
    s = torch.cuda.Stream()
    hs = [InitialGuess(N, m, M, p, stream=s) for m, M, p in specs]
    for h in hs[1:]:
        h.set_device_ring(True)
    F = len(specs)
    seq = _seq(g, 30, dt=1e-2)
    bufs = {k: [torch.zeros(N, dtype=torch.float64, device="cuda") for _ in range(F)] for k in ("b", "x0", "x", "Ax")}
    torch.cuda.synchronize()
    with CapturedStep(s) as step:
        ig_form_guess_batch(hs, bufs["b"], bufs["x0"])
        ig_update_batch(hs, bufs["x"], bufs["Ax"])

    def check(got, f, ref, tag):
        nr = np.linalg.norm(ref)
        assert np.linalg.norm(got - ref) <= TOL * (nr if nr > 0 else 1.0), (seed, tag, specs[f])

    for it in range(40):
        b, x, Ax = seq[int(rng.integers(len(seq)))]
        op = rng.choice(["replay", "replay", "eager", "reset", "switch"])
        if op == "replay":
            # the graph was captured with device windows: make sure they are on
            for h in hs[1:]:
                h.set_device_ring(True)
            with torch.cuda.stream(s):
                for f in range(F):
                    bufs["b"][f].copy_(torch.from_numpy(b))
                    bufs["x0"][f].zero_()
                    bufs["x"][f].copy_(torch.from_numpy(x))
                    bufs["Ax"][f].copy_(torch.from_numpy(Ax))
            step.replay()
            s.synchronize()
            for f, o in enumerate(oras):
                check(bufs["x0"][f].cpu().numpy(), f, o.form_guess(b, np.zeros(N)), ("replay", it))
                o.update(x, Ax)
        elif op == "eager":
            f = int(rng.integers(F))
            x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
            with torch.cuda.stream(s):
                hs[f].form_guess(torch.from_numpy(b).cuda(), x0)
                hs[f].update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
            s.synchronize()
            check(x0.cpu().numpy(), f, oras[f].form_guess(b, np.zeros(N)), ("eager", it))
            oras[f].update(x, Ax)
        elif op == "reset":
            f = int(rng.integers(F))
            hs[f].reset()
            m, M, p = specs[f]
            oras[f] = mk[m](M, p)
        else:  # switch an extrapolation field's window to the host and back (history kept)
            f = 1 + int(rng.integers(F - 1))
            hs[f].set_device_ring(False)
            x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
            with torch.cuda.stream(s):
                hs[f].form_guess(None, x0)
            s.synchronize()
            check(x0.cpu().numpy(), f, oras[f].form_guess(None, np.zeros(N)), ("host window", it))
        for f, (h, o) in enumerate(zip(hs, oras)):
            assert h.d == (o.d if hasattr(o, "d") else o.fill), (seed, it, specs[f])
    step.close()
    for h in hs:
        h.close()
