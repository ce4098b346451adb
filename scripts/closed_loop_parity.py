#!/usr/bin/env python
"""Closed-loop parity data (SURVEY §8(c) protocol, configs[0]): per-step CG iteration counts of the
CUDA path and the oracle for every method, three ways --

  open   : identical systems driven by the ORACLE's closed loop (both guesses solved from the same b_n)
  shadow : identical systems driven by the CUDA path's OWN closed loop (its guesses feed its CG, its
           solutions feed both histories): per-step guess difference and iteration difference
  closed : two independent closed loops (each side feeds back its own solutions)

Prints one JSON object per method.  GPU needed.   python scripts/closed_loop_parity.py
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import ExtrapLS, ExtrapSparse, ProjClassic, ProjQR  # noqa: E402
from paper_2009_10863_b200 import InitialGuess  # noqa: E402
from workloads import Grid, helmholtz_apply, prescribed_rhs  # noqa: E402
from workloads.cg import pcg  # noqa: E402

METHODS = [("proj_qr", 8, 0), ("extrap_ls", 4, 2), ("extrap_ls", 8, 3), ("proj_classic", 4, 0),
           ("extrap_sparse", 8, 3)]
ORA = {"proj_qr": lambda N, M, p: ProjQR(N, M), "extrap_ls": lambda N, M, p: ExtrapLS(N, M, p),
       "proj_classic": lambda N, M, p: ProjClassic(N, M), "extrap_sparse": lambda N, M, p: ExtrapSparse(N, M, p)}


def run(method, M, p, steps=40, dt=1e-3):
    g = Grid(32, 2)
    out = {"method": method, "M": M, "p": p}
    # shadow: the CUDA path drives
    lib, ora = InitialGuess(g.N, method, M, p), ORA[method](g.N, M, p)
    x_prev = torch.zeros(g.N, dtype=torch.float64)
    its_g, its_o, rel = [], [], []
    for n in range(steps):
        b = prescribed_rhs(g, n, dt)
        x0g = x_prev.clone().cuda()
        lib.form_guess(b.cuda(), x0g)
        x0g = x0g.cpu()
        x0o = torch.from_numpy(ora.form_guess(b.numpy(), x_prev.numpy()))
        rel.append(float(torch.linalg.vector_norm(x0g - x0o) / max(float(torch.linalg.vector_norm(x0o)), 1e-300)))
        x, it_g, _, _ = pcg(g, b, x0g)
        _, it_o, _, _ = pcg(g, b, x0o)
        its_g.append(it_g)
        its_o.append(it_o)
        Ax = helmholtz_apply(g, x)
        lib.update(x.cuda(), Ax.cuda())
        ora.update(x.numpy(), Ax.numpy())
        x_prev = x
    lib.close()
    out["shadow"] = {"gpu": its_g, "ora": its_o, "max_rel_guess_diff": max(rel)}
    # closed: independent loops
    res = {}
    for side in ("gpu", "ora"):
        obj = InitialGuess(g.N, method, M, p) if side == "gpu" else ORA[method](g.N, M, p)
        x_prev = torch.zeros(g.N, dtype=torch.float64)
        its = []
        for n in range(steps):
            b = prescribed_rhs(g, n, dt)
            if side == "gpu":
                x0 = x_prev.clone().cuda()
                obj.form_guess(b.cuda(), x0)
                x0 = x0.cpu()
            else:
                x0 = torch.from_numpy(obj.form_guess(b.numpy(), x_prev.numpy()))
            x, it, _, _ = pcg(g, b, x0)
            its.append(it)
            Ax = helmholtz_apply(g, x)
            if side == "gpu":
                obj.update(x.cuda(), Ax.cuda())
            else:
                obj.update(x.numpy(), Ax.numpy())
            x_prev = x
        if side == "gpu":
            obj.close()
        res[side] = its
    out["closed"] = res
    d = np.array(res["gpu"]) - np.array(res["ora"])
    out["closed_max_abs_diff"] = int(np.abs(d).max())
    out["shadow_max_abs_diff"] = int(np.abs(np.array(its_g) - np.array(its_o)).max())
    return out


if __name__ == "__main__":
    for m in METHODS:
        print(json.dumps(run(*m)), flush=True)
