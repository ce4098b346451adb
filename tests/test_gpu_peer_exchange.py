"""In-kernel peer exchange (fused compute + collective) on ONE GPU with virtual ranks.

The multi-GPU path of the persistent projection kernels sums each reduction pass across ranks by
storing the rank-local partials into every rank's exchange window (NVLink peer memory between
GPUs) and acquiring per-rank epoch flags inside the kernel.  The pool gives one GPU, so G ranks
are emulated by G handles in one process on G streams, each owning a contiguous DOF shard and a
1/G share of the SMs (ig_set_grid_limit), wired with in-process window pointers.  The code path
(publish, system-scope fence + release, acquire, rank-ordered sum) is the one a multi-GPU run
executes; only the transport differs.  The concatenated guesses must match the UNSHARDED oracle
 within 1e-11 and all ranks must take identical decisions.
"""

import numpy as np
import pytest
import torch

from oracle import ProjClassic, ProjQR
from workloads import Grid, manufactured_step

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.timeout(300)
@pytest.mark.parametrize("G,M,method", [(2, 8, "proj_qr"), (3, 5, "proj_qr"), (2, 30, "proj_qr"), (4, 3, "proj_qr"),
                                         (2, 4, "proj_classic"), (8, 8, "proj_qr"), (8, 4, "proj_classic")])
def test_virtual_ranks_match_unsharded_oracle(G, M, method):
    """G = 8 is the largest exchange (MAXG, one 8-GPU NVLink node): every window slot and flag."""
    from paper_2009_10863_b200 import InitialGuess, attach_virtual_ranks, ig_set_grid_limit, shard_range

    g = Grid(41, 2)  # N = 1681: odd shards
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    ranges = [shard_range(g.N, G, r) for r in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    igs = [InitialGuess(hi - lo, method, M, stream=streams[r]) for r, (lo, hi) in enumerate(ranges)]
    for ig in igs:
        ig_set_grid_limit(ig.h, max(1, nsm // G))
    attach_virtual_ranks([ig.h for ig in igs])
    ora = (ProjQR if method == "proj_qr" else ProjClassic)(g.N, M)
    for n in range(2 * M + 6):
        b, x, Ax = (t.numpy() for t in manufactured_step(g, n, dt=1e-2))
        bs = [torch.from_numpy(b[lo:hi].copy()).cuda() for lo, hi in ranges]
        xs = [torch.from_numpy(x[lo:hi].copy()).cuda() for lo, hi in ranges]
        As = [torch.from_numpy(Ax[lo:hi].copy()).cuda() for lo, hi in ranges]
        x0s = [torch.zeros(hi - lo, dtype=torch.float64, device="cuda") for lo, hi in ranges]
        torch.cuda.synchronize()
        for r in range(G):  # all ranks' kernels run concurrently on their own streams
            igs[r].form_guess(bs[r], x0s[r])
        for r in range(G):
            igs[r].update(xs[r], As[r])
        torch.cuda.synchronize()
        got = torch.cat([t.cpu() for t in x0s]).numpy()
        ref = ora.form_guess(b, np.zeros(g.N))
        nr = np.linalg.norm(ref)
        assert np.linalg.norm(got - ref) <= 1e-11 * (nr if nr > 0 else 1.0), n
        ora.update(x, Ax)
        st = [ig.stats() for ig in igs]
        assert all(s["d"] == ora.d for s in st), (n, [s["d"] for s in st], ora.d)
        assert len({(s["admitted"], s["rho"]) for s in st}) == 1  # bitwise-identical decisions
    for ig in igs:
        ig.close()


@pytest.mark.timeout(120)
def test_watchdog_reports_a_missing_rank():
    """Failure detection: rank 1 never calls; rank 0's in-kernel exchange gives up after the
    watchdog time instead of hanging, and the host reports IG_E_STATE."""
    from paper_2009_10863_b200 import IGError, InitialGuess, attach_virtual_ranks, ig_set_grid_limit, ig_set_watchdog

    N = 1000
    igs = [InitialGuess(N, "proj_qr", 4) for _ in range(2)]
    for ig in igs:
        ig_set_grid_limit(ig.h, 8)
        ig_set_watchdog(ig.h, 0.2)
    attach_virtual_ranks([ig.h for ig in igs])
    x = torch.rand(N, dtype=torch.float64, device="cuda")
    igs[0].update(x, x)  # only rank 0 participates
    with pytest.raises(IGError, match="watchdog"):
        igs[0].stats()
    for ig in igs:
        ig.close()
