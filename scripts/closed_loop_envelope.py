#!/usr/bin/env python
"""How far apart can two CORRECT fully closed loops drift?  (oracle only; writes a test fixture)

SURVEY §8(c)'s closed-loop protocol runs each side's own CG from its own guesses and feeds its own
solutions back into its own history.  This script measures the oracle against ITSELF: the same
oracle closed loop (configs[0]: 2D 32x32 Helmholtz, prescribed smooth RHS, 40 steps, dt = 1e-3,
Jacobi-PCG INITRESID eps = 1e-8) is re-run with every guess multiplied
elementwise by (1 + delta * xi), xi ~ N(0, 1) seeded, i.e. a rounding-level perturbation like the
one a different (but equally correct) summation order produces.  Per method it records the
per-step spread of the CG iteration counts, the largest |difference| over all seeds, and the size
of the difference at the FIRST step where the two loops' counts differ.

Calls only oracle/ and workloads/ (no CUDA path):   python scripts/closed_loop_envelope.py
-> tests/golden/closed_loop_envelope.json (used by tests/test_gpu_closed_loop.py; DESIGN.md AMB-21)
"""

from __future__ import annotations

import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METHODS = [("proj_qr", 8, 0), ("extrap_ls", 4, 2), ("extrap_ls", 8, 3), ("proj_classic", 4, 0),
           ("extrap_sparse", 8, 3)]
DELTAS = [1e-16, 1e-15, 1e-14]
SEEDS = 32
STEPS, DT = 40, 1e-3


def closed_loop(method, M, p, delta, seed):
    import torch

    torch.set_num_threads(1)
    from oracle import ExtrapLS, ExtrapSparse, ProjClassic, ProjQR
    from workloads import Grid, helmholtz_apply, prescribed_rhs
    from workloads.cg import pcg

    g = Grid(32, 2)
    obj = {"proj_qr": lambda: ProjQR(g.N, M), "extrap_ls": lambda: ExtrapLS(g.N, M, p),
           "proj_classic": lambda: ProjClassic(g.N, M), "extrap_sparse": lambda: ExtrapSparse(g.N, M, p)}[method]()
    rng = np.random.default_rng(seed)
    x_prev = np.zeros(g.N)
    its = []
    for n in range(STEPS):
        b = prescribed_rhs(g, n, DT)
        x0 = np.array(obj.form_guess(b.numpy(), x_prev.copy()), dtype=np.float64)
        if delta:
            x0 = x0 * (1.0 + delta * rng.standard_normal(g.N))
        x, it, _, _ = pcg(g, b, torch.from_numpy(x0))
        its.append(int(it))
        obj.update(x.numpy(), helmholtz_apply(g, x).numpy())
        x_prev = x.numpy()
    return its


def main():
    out = {"what": __doc__.split("\n\n")[1].strip(), "config": "configs[0] 2D 32x32, 40 steps, dt 1e-3, INITRESID 1e-8",
           "seeds": SEEDS, "methods": {}}
    with ProcessPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for method, M, p in METHODS:
            key = f"{method}({M},{p})"
            base = closed_loop(method, M, p, 0.0, 0)
            rec = {"unperturbed": base}
            for delta in DELTAS:
                runs = list(ex.map(closed_loop, *zip(*[(method, M, p, delta, s) for s in range(SEEDS)])))
                d = np.array(runs) - np.array(base)[None, :]
                first = []
                for row in d:
                    nz = np.nonzero(row)[0]
                    first.append(int(abs(row[nz[0]])) if len(nz) else 0)
                rec[f"{delta:g}"] = {"max_abs_diff": int(np.abs(d).max()),
                                     "max_abs_diff_per_seed": np.abs(d).max(axis=1).astype(int).tolist(),
                                     "first_divergence_abs_diff": first,
                                     "per_step_max_abs_diff": np.abs(d).max(axis=0).astype(int).tolist(),
                                     "steady_mean_shift_max": float(np.abs(d[:, 10:].mean(axis=1)).max())}
                print(key, delta, rec[f"{delta:g}"]["max_abs_diff"], sorted(set(first)), flush=True)
            out["methods"][key] = rec
    path = os.path.join(ROOT, "tests", "golden", "closed_loop_envelope.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
