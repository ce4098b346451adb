"""The multi-rank SPLIT schedule (one kernel per pass, all-gather of the per-rank partial sums
between kernels -- the path a handle takes with an NCCL communicator, ig_attach_comm) with G
ranks on ONE GPU.  NCCL refuses two ranks on one device, so the ranks are host threads of this
process wired by the in-process communicator (ig_comm_create_local: same all-gather layout, same
exchange points, device-to-device copies after each rank's event).  Each rank owns a contiguous
DOF shard (z-slab partition) and its own stream; the concatenated guesses must match
the UNSHARDED oracle within 1e-11, and every rank must take the same decisions
and hold a bitwise-identical R (rank-ordered sums of the gathered partials)."""

import threading

import numpy as np
import pytest
import torch

from oracle import ProjClassic, ProjQR
from workloads import Grid, manufactured_step

pytestmark = pytest.mark.gpu

TOL = 1e-11


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("G,M,method", [(2, 8, "proj_qr"), (3, 5, "proj_qr"), (2, 30, "proj_qr"),
                                        (4, 3, "proj_classic"), (8, 8, "proj_qr")])
def test_split_schedule_with_in_process_ranks_matches_unsharded_oracle(G, M, method):
    from paper_2009_10863_b200 import (InitialGuess, ig_comm_create_local, ig_comm_destroy, ig_copy_history,
                                       ig_local_group_create, ig_local_group_destroy, shard_range)

    g = Grid(29, 2)
    N = g.N
    steps = 3 * M + 4
    seq = [tuple(t.numpy() for t in manufactured_step(g, n, dt=1e-2)) for n in range(steps)]
    ora = (ProjQR if method == "proj_qr" else ProjClassic)(N, M)
    group = ig_local_group_create(G)
    comms = [ig_comm_create_local(group, r) for r in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    shards = [shard_range(N, G, r) for r in range(G)]
    igs = [InitialGuess(hi - lo, method, M, comm=comms[r], stream=streams[r])
           for r, (lo, hi) in enumerate(shards)]
    guesses = [[None] * steps for _ in range(G)]
    dims = [[None] * steps for _ in range(G)]
    errors = []

    def rank(r):
        try:
            lo, hi = shards[r]
            with torch.cuda.stream(streams[r]):
                for n, (b, x, Ax) in enumerate(seq):
                    x0 = torch.full((hi - lo,), -1.0, dtype=torch.float64, device="cuda")
                    igs[r].form_guess(torch.from_numpy(b[lo:hi]).cuda(), x0)
                    guesses[r][n] = x0.cpu().numpy()  # syncs this rank's stream
                    igs[r].update(torch.from_numpy(x[lo:hi]).cuda(), torch.from_numpy(Ax[lo:hi]).cuda())
                    dims[r][n] = igs[r].d
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append((r, repr(e)))

    threads = [threading.Thread(target=rank, args=(r,)) for r in range(G)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=240)
    assert not any(t.is_alive() for t in threads), "a rank hung"
    assert not errors, errors
    worst = 0.0
    for n, (b, x, Ax) in enumerate(seq):
        ref = ora.form_guess(b, np.full(N, -1.0))
        got = np.concatenate([guesses[r][n] for r in range(G)])
        worst = max(worst, _rel(got, ref))
        ora.update(x, Ax)
        assert len({dims[r][n] for r in range(G)}) == 1 and dims[0][n] == ora.d, n
    assert worst <= TOL, worst
    Rs = [ig_copy_history(h.h, M, hi - lo)[2] for h, (lo, hi) in zip(igs, shards)]
    for R in Rs[1:]:
        assert torch.equal(R, Rs[0])  # bitwise-identical small state on every rank
    for h in igs:
        h.close()
    for c in comms:
        ig_comm_destroy(c)
    ig_local_group_destroy(group)
