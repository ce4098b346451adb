"""Multi-rank (N > 1) host logic on CPU with gloo, world size 2.

The CUDA library's multi-rank schedule is: contiguous DOF shards
(`shard_range`), per-rank partial sums of every reduction pass (form alpha; U1: c1 and ||Ax||^2;
U2: c2 and ||b1||^2), an ALL-GATHER of those partials, and a rank-ordered sum on every rank, so
that every control decision (admission, d, R, Givens) is bitwise identical across ranks.  This
test runs exactly that protocol over torch.distributed/gloo with a numpy model of the per-rank
arithmetic, and checks (1) the sharded guesses equal the unsharded oracle to
1e-12, (2) both ranks take identical decisions with bitwise-identical coefficients.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ProjQR
from paper_2009_10863_b200.ig import shard_range
from workloads import Grid, manufactured_step


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class ShardedProjQR:
    """Per-rank model of libig's split schedule: local slabs, replicated R and decisions."""

    def __init__(self, n_local, M, world, eps=1e-10):
        self.M, self.world, self.eps = M, world, eps
        self.Bt = np.zeros((n_local, M))
        self.Xt = np.zeros((n_local, M))
        self.R = np.zeros((M, M))
        self.d = 0
        self.pending = False
        self.gc = np.ones(M)
        self.gs = np.zeros(M)
        self.log = []

    def gsum(self, partial):
        t = torch.from_numpy(np.ascontiguousarray(partial, dtype=np.float64))
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t)
        s = parts[0].clone()
        for r in range(1, self.world):  # rank-ordered sum: identical on every rank
            s += parts[r]
        return s.numpy()

    def form_guess(self, b, x0):
        if self.d == 0:
            return x0.copy()
        alpha = self.gsum(self.Bt[:, :self.d].T @ b)
        self.log.append(("alpha", alpha.tobytes()))
        return self.Xt[:, :self.d] @ alpha

    def _plan(self):  # givens_plan: replicated small dense work
        M = self.M
        H = self.R[:M, 1:M].copy()
        for i in range(M - 1):
            a, b = H[i, i], H[i + 1, i]
            r = math.hypot(a, b)
            c, s = (1.0, 0.0) if r == 0 else (a / r, b / r)
            self.gc[i], self.gs[i] = c, s
            H[i:i + 2, :] = np.array([[c, s], [-s, c]]) @ H[i:i + 2, :]
        self.Rdn = np.zeros_like(self.R)
        self.Rdn[:M - 1, :M - 1] = np.triu(H[:M - 1, :])
        self.pending = True

    def update(self, x, Ax):
        M = self.M
        if self.pending:  # U1: rotate B~ (and later X~) with the pre-planned Givens
            for i in range(M - 1):
                c, s = self.gc[i], self.gs[i]
                for Y in (self.Bt, self.Xt):
                    Y[:, i], Y[:, i + 1] = c * Y[:, i] + s * Y[:, i + 1], -s * Y[:, i] + c * Y[:, i + 1]
            self.R = self.Rdn.copy()
            self.d = M - 1
            self.pending = False
        d = self.d
        p1 = self.gsum(np.concatenate([self.Bt[:, :d].T @ Ax, [Ax @ Ax]]))
        c1, nAx2 = p1[:d], p1[d]
        if d > 0:
            b1 = Ax - self.Bt[:, :d] @ c1
            p2 = self.gsum(np.concatenate([self.Bt[:, :d].T @ b1, [b1 @ b1]]))
            c2, nb12 = p2[:d], p2[d]
            nb = math.sqrt(max(nb12 - c2 @ c2, 0.0))
            adm = nb > self.eps * math.sqrt(nAx2)
        else:
            c2 = np.zeros(0)
            nb = math.sqrt(nAx2)
            adm = nb > 0
        self.log.append(("dec", p1.tobytes(), bool(adm), d))
        if adm:
            b2 = (Ax - self.Bt[:, :d] @ c1) - self.Bt[:, :d] @ c2
            xt = (x - self.Xt[:, :d] @ c1) - self.Xt[:, :d] @ c2
            self.R[:d, d] = c1 + c2
            self.R[d, d] = nb
            self.Bt[:, d] = b2 / nb
            self.Xt[:, d] = xt / nb
            self.d = d + 1
            if self.d == M:
                self._plan()


def _worker(rank, world, port, M, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = Grid(14, 3)
    lo, hi = shard_range(g.N, world, rank)
    model = ShardedProjQR(hi - lo, M, world)
    guesses = []
    for n in range(steps):
        b, x, Ax = (t.numpy() for t in manufactured_step(g, n, dt=1e-2))
        x0 = model.form_guess(b[lo:hi], np.zeros(hi - lo))
        pieces = [None] * world
        dist.all_gather_object(pieces, x0)
        guesses.append(np.concatenate(pieces))
        model.update(x[lo:hi], Ax[lo:hi])
    out[rank] = {"guesses": guesses if rank == 0 else None, "log": model.log, "d": model.d}
    dist.destroy_process_group()


@pytest.mark.parametrize("M", [3, 8])
def test_two_rank_sharded_projection_matches_oracle(M):
    world, steps = 2, 3 * M + 4
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), M, steps, out), nprocs=world, join=True,
                       start_method="spawn")
    r0, r1 = out[0], out[1]
    assert r0["log"] == r1["log"], "ranks must take bitwise-identical decisions"
    assert r0["d"] == r1["d"] == M
    g = Grid(14, 3)
    ora = ProjQR(g.N, M)
    for n in range(steps):
        b, x, Ax = (t.numpy() for t in manufactured_step(g, n, dt=1e-2))
        ref = ora.form_guess(b, np.zeros(g.N))
        got = r0["guesses"][n]
        nr = np.linalg.norm(ref)
        assert np.linalg.norm(got - ref) <= 1e-12 * (nr if nr > 0 else 1.0), n
        ora.update(x, Ax)


def test_slab_generator_concatenates_to_the_global_field():
    from workloads.gen import manufactured_step_slab

    parts = [manufactured_step_slab(8, 4, r, 2, 3) for r in range(2)]
    x_full = torch.cat([p[1] for p in parts])
    whole = manufactured_step_slab(8, 8, 0, 1, 3)
    # same global coordinates and noise -> identical x; A is block-diagonal across the cut
    assert torch.allclose(x_full, whole[1], rtol=0, atol=1e-15)
