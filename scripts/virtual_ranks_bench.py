#!/usr/bin/env python
"""Cost of the in-kernel peer exchange, measured on ONE GPU with G virtual ranks.

The C2 projection workload (128^3 DOFs, QR(8)) is split into G contiguous shards; each virtual
rank (own handle, own stream, 1/G of the SMs) runs its persistent kernels concurrently with the
others, and every reduction pass is summed across ranks through the exchange windows.  Compared
with the single-rank run on the same GPU this isolates the exchange + skew cost (the multi-GPU
run adds NVLink latency, ~1-2 us per exchange, instead of on-chip latency).

    python scripts/virtual_ranks_bench.py [--G 2] [--steps 100]
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2009_10863_b200 import InitialGuess, attach_virtual_ranks, ig_set_grid_limit, shard_range  # noqa: E402
from workloads.gen import manufactured_step_slab  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--G", type=int, default=2)
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    n, M, G = a.n, a.M, a.G
    N = n ** 3
    S = a.steps + M + 4
    pool = [manufactured_step_slab(n, n, 0, 1, k, device="cuda") for k in range(S)]
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    res = {}
    for g in (1, G):
        ranges = [shard_range(N, g, r) for r in range(g)]
        streams = [torch.cuda.Stream() for _ in range(g)]
        igs = [InitialGuess(hi - lo, "proj_qr", M, stream=streams[r]) for r, (lo, hi) in enumerate(ranges)]
        if g > 1:
            for ig in igs:
                ig_set_grid_limit(ig.h, nsm // g)
            attach_virtual_ranks([ig.h for ig in igs])
        x0s = [torch.zeros(hi - lo, dtype=torch.float64, device="cuda") for lo, hi in ranges]

        def step(k):
            b, x, Ax = pool[k]
            for r, (lo, hi) in enumerate(ranges):
                igs[r].form_guess(b[lo:hi], x0s[r])
            for r, (lo, hi) in enumerate(ranges):
                igs[r].update(x[lo:hi], Ax[lo:hi])

        for k in range(M + 4):
            step(k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in streams:
            s.wait_event(e0)
        for k in range(M + 4, S):
            step(k)
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            torch.cuda.current_stream().wait_event(e)
        e1.record()
        torch.cuda.synchronize()
        res[g] = e0.elapsed_time(e1) / a.steps * 1e3
        assert all(ig.d == M for ig in igs)
        for ig in igs:
            ig.close()
    by = (8 * M + 4) * 8 * N
    for g, us in res.items():
        print(f"G={g}: QR({M}) form+update {us:.1f} us/step, {by / (us * 1e-6) / 1e9:.0f} GB/s")
    print(f"exchange + skew overhead of {G} virtual ranks: {res[G] - res[1]:+.1f} us/step "
          f"({3} exchanges per step)")


if __name__ == "__main__":
    main()
