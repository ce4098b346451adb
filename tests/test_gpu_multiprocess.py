"""Two PROCESSES, one rank each, sharing the single GPU: the multi-process setup path of the in-kernel
peer exchange (CUDA IPC handles of the exchange windows traded through torch.distributed/gloo,
`peers_from_process_group`), then a sharded projection sequence whose concatenated guesses must
match the unsharded oracle within 1e-11, with identical decisions on both ranks.

On a multi-GPU node the same code maps each peer's window over NVLink; here both windows live on
one GPU, so each rank's persistent kernels get half of the SMs (`ig_set_grid_limit`) to run
concurrently with the other rank's."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, steps, out):
    import torch.distributed as dist

    from paper_2009_10863_b200 import InitialGuess, ig_set_grid_limit, peers_from_process_group, shard_range
    from workloads import Grid, manufactured_step

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = Grid(37, 2)
    lo, hi = shard_range(g.N, world, rank)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    ig = InitialGuess(hi - lo, "proj_qr", M)
    ig_set_grid_limit(ig.h, nsm // world)
    peers_from_process_group([ig.h])
    guesses, decisions = [], []
    for n in range(steps):
        b, x, Ax = (t.numpy() for t in manufactured_step(g, n, dt=1e-2))
        x0 = torch.zeros(hi - lo, dtype=torch.float64, device="cuda")
        ig.form_guess(torch.from_numpy(b[lo:hi].copy()).cuda(), x0)
        ig.update(torch.from_numpy(x[lo:hi].copy()).cuda(), torch.from_numpy(Ax[lo:hi].copy()).cuda())
        torch.cuda.synchronize()
        pieces = [None] * world
        dist.all_gather_object(pieces, x0.cpu().numpy())
        guesses.append(np.concatenate(pieces))
        st = ig.stats()
        decisions.append((st["d"], st["admitted"], st["rho"]))
    dist.barrier()
    ig.close()
    out[rank] = {"guesses": guesses if rank == 0 else None, "decisions": decisions}
    dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("M", [4, 8])
def test_two_processes_one_gpu_peer_exchange(M):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import ProjQR
    from workloads import Grid, manufactured_step

    world, steps = 2, 2 * M + 5
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), M, steps, out), nprocs=world, join=True,
                       start_method="spawn")
    assert out[0]["decisions"] == out[1]["decisions"]  # bitwise-identical d / admission / rho
    g = Grid(37, 2)
    ora = ProjQR(g.N, M)
    for n in range(steps):
        b, x, Ax = (t.numpy() for t in manufactured_step(g, n, dt=1e-2))
        ref = ora.form_guess(b, np.zeros(g.N))
        got = out[0]["guesses"][n]
        nr = np.linalg.norm(ref)
        assert np.linalg.norm(got - ref) <= 1e-11 * (nr if nr > 0 else 1.0), n
        ora.update(x, Ax)
        assert out[0]["decisions"][n][0] == ora.d
