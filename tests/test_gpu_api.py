"""GPU-side API behaviour: byte accounting, reset, launch policies, per-kernel profiling, errors."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import ExtrapLS, ProjQR
from workloads import Grid, manufactured_step

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _seq(g, steps, dt=1e-2):
    return [tuple(t.numpy() for t in manufactured_step(g, n, dt=dt)) for n in range(steps)]


def test_byte_accounting_follows_the_fused_schedule():
    """ig_bytes = DESIGN.md §7: form 2(d+1); update U1 (2M | d+1) + U2 (d+1) + U3; 8 bytes/value."""
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(20, 2)
    N, M = g.N, 5
    ig = InitialGuess(N, "proj_qr", M)
    vb = 8 * N
    d_before = 0
    for n, (b, x, Ax) in enumerate(_seq(g, 2 * M + 3)):
        x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
        ig.form_guess(torch.from_numpy(b).cuda(), x0)
        fb, _ = ig.bytes()
        assert fb == (2 * (d_before + 1) * vb if d_before > 0 else 0)
        ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
        _, ub = ig.bytes()
        rot = d_before == M
        de = M - 1 if rot else d_before
        expect = (2 * M if rot else de + 1) + (de + 1 if de > 0 else 0) + (1 + de + 1 + 2) + (2 * M - 1 if rot else de)
        assert ub == expect * vb, (n, ub / vb, expect)
        d_before = ig.d
    # steady state: (8M+4) values per element per step
    assert fb + ub == (8 * M + 4) * vb
    # against the paper's Table 1 (tests/golden/paper_values.txt): the guess moves
    # exactly 2(M+1)N values; the update moves at most the table's (10M+24)N minus the 9N operator
    # apply that is not part of the library (the fused Givens sweep saves the rest)
    assert fb == 2 * (M + 1) * vb
    assert ub <= (10 * M + 24 - 9) * vb
    ig.close()


def test_extrapolation_bytes_match_table_1():
    """EXTRAP(m, M): (M+1)N per step with the solver writing in place."""
    from paper_2009_10863_b200 import InitialGuess

    N, M, m = 5000, 8, 2  # EXTRAP(2,8): all weights nonzero
    ig = InitialGuess(N, "extrap_ls", M, m)
    assert all(w != 0.0 for w in ig.weights())
    for n in range(M + 2):
        slot = ig.next_slot()
        if n == 0:
            slot.zero_()
        ig.form_guess(None, slot)
        slot.add_(1.0)  # the "solver" writes its solution in place
        ig.update(slot)
    fb, ub = ig.bytes()
    assert fb == (M + 1) * 8 * N and ub == 0
    ig.close()


def test_reset_forgets_history():
    from paper_2009_10863_b200 import InitialGuess

    g = Grid(16, 2)
    seq = _seq(g, 10)
    ig, ie = InitialGuess(g.N, "proj_qr", 4), InitialGuess(g.N, "extrap_ls", 4, 2)
    for b, x, Ax in seq[:6]:
        ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
        ie.update(torch.from_numpy(x).cuda())
    ig.reset()
    ie.reset()
    assert ig.d == 0 and ie.d == 0
    op, oe = ProjQR(g.N, 4), ExtrapLS(g.N, 4, 2)
    for b, x, Ax in seq[6:]:
        for o, h in ((op, ig), (oe, ie)):
            x0 = torch.full((g.N,), 2.0, dtype=torch.float64, device="cuda")
            h.form_guess(torch.from_numpy(b).cuda(), x0)
            ref = o.form_guess(b, np.full(g.N, 2.0))
            assert np.linalg.norm(x0.cpu().numpy() - ref) <= 1e-11 * np.linalg.norm(ref)
            o.update(x, Ax)
            h.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
    ig.close()
    ie.close()


@pytest.mark.parametrize("flags", ["coop,pdl", "coop", "", "pdl"])
def test_launch_policies_give_identical_results(flags):
    """IG_LAUNCH selects cooperative launch and/or programmatic dependent launch; the arithmetic
    (and therefore every bit of the guesses) must not depend on it."""
    code = (
        "import numpy as np, torch, sys\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "from paper_2009_10863_b200 import InitialGuess\n"
        "from workloads import Grid, manufactured_step\n"
        "g = Grid(64, 2); ig = InitialGuess(g.N, 'proj_qr', 6); ie = InitialGuess(g.N, 'extrap_ls', 6, 2)\n"
        "out = []\n"
        "for n in range(14):\n"
        "    b, x, Ax = (t.cuda() for t in manufactured_step(g, n, dt=1e-2))\n"
        "    x0 = torch.zeros_like(b); ig.form_guess(b, x0); out.append(x0.cpu().numpy())\n"
        "    y0 = torch.zeros_like(b); ie.form_guess(None, y0); out.append(y0.cpu().numpy())\n"
        "    ig.update(x, Ax); ie.update(x)\n"
        "np.save(sys.argv[1], np.stack(out))\n"
    )
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        res = {}
        for f in (flags, "pdl"):
            path = os.path.join(td, f"out_{f or 'none'}.npy")
            env = dict(os.environ, IG_LAUNCH=f if f else "none")
            r = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True, text=True, timeout=300)
            assert r.returncode == 0, r.stderr
            res[f] = np.load(path)
        assert np.array_equal(res[flags], res["pdl"])  # bitwise identical (same grid, same order)


def test_profile_counts_launches():
    from paper_2009_10863_b200 import InitialGuess, ig_profile, ig_profile_read

    g = Grid(32, 2)
    ig = InitialGuess(g.N, "proj_qr", 4)
    ig_profile(ig.h, True)
    for b, x, Ax in _seq(g, 6):
        x0 = torch.zeros(g.N, dtype=torch.float64, device="cuda")
        ig.form_guess(torch.from_numpy(b).cuda(), x0)
        ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
    prof = ig_profile_read(ig.h)
    assert prof["update_fused"][1] == 6 and prof["form_fused"][1] == 6
    assert prof["update_fused"][0] > 0.0
    ig_profile(ig.h, False)
    ig.close()


def test_argument_errors_on_device():
    from paper_2009_10863_b200 import IGError, InitialGuess

    ig = InitialGuess(100, "proj_qr", 4)
    with pytest.raises(TypeError):
        ig.form_guess(torch.zeros(100, dtype=torch.float32, device="cuda"), torch.zeros(100, device="cuda"))
    with pytest.raises(IGError, match="Ax is NULL"):
        ig.update(torch.zeros(100, dtype=torch.float64, device="cuda"), None)
    ig.close()


@pytest.mark.parametrize("method,M,p", [("proj_qr", 6, 0), ("proj_classic", 4, 0), ("extrap_ls", 6, 3),
                                        ("extrap_sparse", 8, 2)])
def test_checkpoint_resume_is_bitwise(method, M, p):
    """Save the history mid-run, load it into a fresh handle: the resumed run reproduces the
    uninterrupted one bit for bit."""
    from paper_2009_10863_b200 import IGError, InitialGuess

    g = Grid(30, 2)
    seq = _seq(g, 2 * M + 6)
    a = InitialGuess(g.N, method, M, p)
    half = M + 2
    for b, x, Ax in seq[:half]:
        a.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
    img = a.save_state()
    bnew = InitialGuess(g.N, method, M, p)
    bnew.load_state(img)
    for b, x, Ax in seq[half:]:
        outs = []
        for h in (a, bnew):
            x0 = torch.zeros(g.N, dtype=torch.float64, device="cuda")
            h.form_guess(torch.from_numpy(b).cuda(), x0)
            outs.append(x0.cpu().numpy())
            h.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
        assert np.array_equal(outs[0], outs[1])
    other = InitialGuess(g.N + 1, method, M, p)
    with pytest.raises(IGError, match="state image is for"):
        other.load_state(img)
    for h in (a, bnew, other):
        h.close()


@pytest.mark.parametrize("fused", [True, False])
def test_non_finite_inputs_are_reported(fused):
    from paper_2009_10863_b200 import IGError, InitialGuess

    N = 4000
    ig = InitialGuess(N, "proj_qr", 4, fused=fused)
    x = torch.rand(N, dtype=torch.float64, device="cuda")
    ig.update(x, x + 1.0)
    bad = x.clone()
    bad[17] = float("nan")
    ig.update(bad, bad)
    with pytest.raises(IGError, match="non-finite"):
        ig.stats()
    ig.close()


def test_projection_fields_on_different_streams_are_ordered_and_correct():
    """Two projection fields on two streams (plus one on the first stream again), calls interleaved:
    full-grid persistent kernels from different streams are ordered by the library (they must not
    share the SMs), so no barrier can wait on CTAs the other grid holds; every guess matches its
    oracle and no watchdog fires."""
    import numpy as np

    from oracle import ProjQR
    from paper_2009_10863_b200 import InitialGuess
    from workloads import Grid, manufactured_step

    g = Grid(40, 2)
    N = g.N
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    specs = [(s1, 6, 1e-2), (s2, 8, 2e-2), (s1, 4, 3e-2)]
    igs = [InitialGuess(N, "proj_qr", M, stream=st) for st, M, _ in specs]
    oras = [ProjQR(N, M) for _, M, _ in specs]
    for n in range(20):
        for (st, M, dt), ig, ora in zip(specs, igs, oras):
            b, x, Ax = (t.numpy() for t in manufactured_step(g, n, dt=dt))
            with torch.cuda.stream(st):
                x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
                ig.form_guess(torch.from_numpy(b).cuda(), x0)
                ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
                got = x0.cpu().numpy()
            ref = ora.form_guess(b, np.zeros(N))
            assert np.linalg.norm(got - ref) <= 1e-11 * max(np.linalg.norm(ref), 1e-300), (n, M)
            ora.update(x, Ax)
    for ig, ora in zip(igs, oras):
        assert ig.stats()["d"] == ora.d  # stats() syncs and reports a watchdog trip as an error
        ig.close()


def test_non_finite_first_pair_is_not_admitted():
    """d = 0 and ||A x||^2 = Inf: the pair must not enter the history (ig.h: NaN/Inf sums leave it
    unadmitted) -- the next guess leaves the caller's fallback untouched (d == 0)
    and the event is reported as IG_E_STATE."""
    from paper_2009_10863_b200 import IGError, InitialGuess

    N = 3000
    for fused in (True, False):
        ig = InitialGuess(N, "proj_qr", 4, fused=fused)
        x = torch.rand(N, dtype=torch.float64, device="cuda")
        big = x.clone()
        big[5] = 1e200  # ||A x||^2 overflows to Inf, entries stay finite
        ig.update(x, big)
        fb = torch.full((N,), 3.0, dtype=torch.float64, device="cuda")
        ig.form_guess(torch.rand(N, dtype=torch.float64, device="cuda"), fb)
        assert torch.equal(fb.cpu(), torch.full((N,), 3.0, dtype=torch.float64)), fused
        with pytest.raises(IGError, match="non-finite"):
            ig.stats()
        ig.close()


def test_load_state_rejects_corrupt_headers():
    """ig_load_state validates the ring / dimension fields before touching the handle."""
    import struct

    from paper_2009_10863_b200 import IGError, InitialGuess

    g = Grid(20, 2)
    for method, M, p in (("extrap_ls", 5, 2), ("proj_qr", 5, 0)):
        a = InitialGuess(g.N, method, M, p)
        for b, x, Ax in _seq(g, M + 2):
            a.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
        img = bytearray(a.save_state())
        for off, val in ((20, M), (20, -1), (32, M + 1), (36, 2 * M + 3)):  # head, fill, nslab
            bad = bytearray(img)
            struct.pack_into("<i", bad, off, val)
            with pytest.raises(IGError, match="corrupt"):
                a.load_state(bytes(bad))
        a.load_state(bytes(img))  # the intact image still loads
        a.close()


def test_checkpoint_restore_with_peers_attached():
    """Load an OLDER image into live handles wired as virtual ranks of the in-kernel exchange: the
    exchange epochs must stay monotonic (ig_load_state keeps the live ones), so the resumed run
    matches the unsharded oracle restored at the same step, with identical decisions on all ranks."""
    import copy

    from paper_2009_10863_b200 import InitialGuess, attach_virtual_ranks, ig_set_grid_limit, shard_range

    G, M = 2, 5
    g = Grid(37, 2)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    ranges = [shard_range(g.N, G, r) for r in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    igs = [InitialGuess(hi - lo, "proj_qr", M, stream=streams[r]) for r, (lo, hi) in enumerate(ranges)]
    for ig in igs:
        ig_set_grid_limit(ig.h, max(1, nsm // G))
    attach_virtual_ranks([ig.h for ig in igs])
    ora = ProjQR(g.N, M)
    seq = _seq(g, 3 * M + 6)

    def step(n, check):
        b, x, Ax = seq[n]
        x0s = [torch.zeros(hi - lo, dtype=torch.float64, device="cuda") for lo, hi in ranges]
        ins = [tuple(torch.from_numpy(v[lo:hi].copy()).cuda() for v in (b, x, Ax)) for lo, hi in ranges]
        torch.cuda.synchronize()  # inputs resident before the ranks' streams read them
        for r in range(G):
            igs[r].form_guess(ins[r][0], x0s[r])
        for r in range(G):
            igs[r].update(ins[r][1], ins[r][2])
        torch.cuda.synchronize()
        got = torch.cat([t.cpu() for t in x0s]).numpy()
        ref = ora.form_guess(b, np.zeros(g.N))
        if check:
            assert np.linalg.norm(got - ref) <= 1e-11 * max(np.linalg.norm(ref), 1e-300), n
        ora.update(x, Ax)
        st = [ig.stats() for ig in igs]
        assert all(s["d"] == ora.d for s in st) and len({(s["admitted"], s["rho"]) for s in st}) == 1, n

    ck = M + 2
    for n in range(ck):
        step(n, True)
    imgs = [ig.save_state() for ig in igs]
    ora_ck = copy.deepcopy(ora)
    for n in range(ck, ck + M + 3):  # move the exchange epochs well past the image's
        step(n, True)
    for ig, img in zip(igs, imgs):
        ig.load_state(img)
    ora = ora_ck
    for n in range(ck, len(seq)):
        step(n, True)
    for ig in igs:
        ig.close()


def test_peers_force_the_fused_schedule():
    """A handle asked for the split schedule and then wired to peers runs the fused kernels (the
    only ones that read the exchange windows); asking for the split schedule afterwards fails."""
    from paper_2009_10863_b200 import IGError, InitialGuess, attach_virtual_ranks, ig_set_grid_limit, ig_set_schedule
    from paper_2009_10863_b200 import shard_range

    G, M = 2, 4
    g = Grid(33, 2)
    ranges = [shard_range(g.N, G, r) for r in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    igs = [InitialGuess(hi - lo, "proj_qr", M, stream=streams[r], fused=False) for r, (lo, hi) in enumerate(ranges)]
    for ig in igs:
        ig_set_grid_limit(ig.h, 16)
    attach_virtual_ranks([ig.h for ig in igs])
    with pytest.raises(IGError, match="fused schedule"):
        ig_set_schedule(igs[0].h, False)
    ora = ProjQR(g.N, M)
    for n, (b, x, Ax) in enumerate(_seq(g, 2 * M + 3)):
        x0s = [torch.zeros(hi - lo, dtype=torch.float64, device="cuda") for lo, hi in ranges]
        ins = [tuple(torch.from_numpy(v[lo:hi].copy()).cuda() for v in (b, x, Ax)) for lo, hi in ranges]
        torch.cuda.synchronize()  # inputs resident before the ranks' streams read them
        for r in range(G):
            igs[r].form_guess(ins[r][0], x0s[r])
        for r in range(G):
            igs[r].update(ins[r][1], ins[r][2])
        torch.cuda.synchronize()
        got = torch.cat([t.cpu() for t in x0s]).numpy()
        ref = ora.form_guess(b, np.zeros(g.N))
        assert np.linalg.norm(got - ref) <= 1e-11 * max(np.linalg.norm(ref), 1e-300), n
        ora.update(x, Ax)
    for ig in igs:
        ig.close()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("mode", ["default", "plain"])
def test_persistent_update_next_to_a_foreign_kernel(mode):
    """A foreign kernel on another stream holds most SMs (227 KB of shared memory per CTA, so no
    libig CTA fits beside it) for 1.5 s while ig_update is enqueued -- the situation of a solver,
    halo-exchange or NCCL kernel running concurrently with the guess machinery.
    Default (cooperative) launch: the driver starts the persistent grid only when all of its CTAs
    fit, so no grid barrier waits on CTAs that cannot run: no watchdog trip (0.5 s), oracle
    parity.  Plain launch: the resident CTAs wait at the first barrier for the rest -- the hazard
    the default removes (the 0.5 s watchdog must fire)."""
    from paper_2009_10863_b200 import IGError, InitialGuess, ig_set_launch, ig_set_watchdog
    from support import hog_lib  # tests/support (tests/ is on sys.path under pytest)

    hog = hog_lib()
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    g = Grid(256, 2)  # N = 65536
    seq = _seq(g, 6)
    ora = ProjQR(g.N, 4)
    ig = InitialGuess(g.N, "proj_qr", 4)
    if mode == "plain":
        ig_set_launch(ig.h, 0)
    ig_set_watchdog(ig.h, 0.5)
    for b, x, Ax in seq[:4]:  # history filled, kernels warm
        ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
        ora.update(x, Ax)
    torch.cuda.synchronize()
    started = torch.zeros(1, dtype=torch.int64, device="cuda")
    foreign = torch.cuda.Stream()
    nblk = nsm - 16
    rc = hog.hog_launch(nblk, 227 * 1024, int(1.5e9), started.data_ptr(), foreign.cuda_stream)
    assert rc == 0, rc
    while int(started.item()) < nblk:  # every foreign CTA holds its SM (item() syncs the default stream only)
        pass
    b, x, Ax = seq[4]
    x0 = torch.zeros(g.N, dtype=torch.float64, device="cuda")
    ig.form_guess(torch.from_numpy(b).cuda(), x0)
    ig.update(torch.from_numpy(x).cuda(), torch.from_numpy(Ax).cuda())
    if mode == "plain":
        with pytest.raises(IGError, match="watchdog"):
            ig.stats()
    else:
        st = ig.stats()
        ref = ora.form_guess(b, np.zeros(g.N))
        assert np.linalg.norm(x0.cpu().numpy() - ref) <= 1e-11 * np.linalg.norm(ref)
        ora.update(x, Ax)
        assert st["d"] == ora.d
    torch.cuda.synchronize()
    ig.close()
