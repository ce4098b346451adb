#!/usr/bin/env python
"""Bandwidth sweep (BASELINE configs[2]/[4]: C3 history sweep and C5 N x M sweep) on one GPU.

For each (N, M): QR(M) form+update and EXTRAP(floor(sqrt M), M) form+update (zero-copy push)
timed with CUDA events over K steps after history fill; effective GB/s from the algorithmic
bytes (QR (8M+4)*8N, EXTRAP (nnz(beta)+1)*8N), fraction of the measured copy roofline.  Inputs are
random per-step vectors from a pool of M+2 (a vector re-enters only after it left the window, so
every projection update is admitted and the full update path is timed).  Points whose per-step
working set fits in L2 are labelled (L2-resident, not an HBM measurement).

    python scripts/bench_sweep.py [--sizes 1e5,1e6,1e7,134217728] [--ms 1,2,4,8,16,30] [--steps 10]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2009_10863_b200 import InitialGuess  # noqa: E402

L2 = 126 * 2 ** 20


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def time_steps(fn, K):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for k in range(K):
        fn(k)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3  # us per step


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="100000,1000000,10000000,134217728")
    ap.add_argument("--ms", default="1,2,4,8,16,30")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--mem-gb", type=float, default=150.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--degree", type=int, default=None, help="EXTRAP degree (default floor(sqrt(M)), P:1527-1529)")
    a = ap.parse_args()
    P = peak()
    rows = []
    for N in [int(float(x)) for x in a.sizes.split(",")]:
        for M in [int(x) for x in a.ms.split(",")]:
            vb = 8 * N
            pool = M + 2
            need = (2 * M + 2 * pool + 2) * vb / 1e9
            if need > a.mem_gb:
                rows.append({"N": N, "M": M, "skipped": f"needs {need:.0f} GB"})
                continue
            g = torch.Generator(device="cuda").manual_seed(10863 + M)
            X = [torch.randn(N, dtype=torch.float64, device="cuda", generator=g) for _ in range(pool)]
            AX = [torch.randn(N, dtype=torch.float64, device="cuda", generator=g) for _ in range(pool)]
            x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
            hp = InitialGuess(N, "proj_qr", M)

            def qstep(k):
                hp.form_guess(AX[(k + 1) % pool], x0)
                hp.update(X[k % pool], AX[k % pool])

            for k in range(M + 2):
                qstep(k)
            tq = time_steps(lambda k: qstep(k + M + 2), a.steps)
            assert hp.d == M and hp.stats()["admitted"] == 1
            hp.close()
            del hp
            p = (int(math.isqrt(M)) if M > 1 else 0) if a.degree is None else a.degree
            p = min(p, M - 1)
            he = InitialGuess(N, "extrap_ls", M, p)

            def estep(k):
                slot = he.next_slot()
                he.form_guess(None, slot)  # solve in place from the guess: zero-copy push
                he.update(slot)

            for k in range(M + 1):
                estep(k)
            te = time_steps(estep, a.steps)
            nnz = sum(1 for w in he.weights() if w != 0.0)
            he.close()
            del he, X, AX, x0
            torch.cuda.empty_cache()
            bq, be = (8 * M + 4) * vb, (nnz + 1) * vb
            ws_q = (2 * M + 3) * vb
            r = {"N": N, "M": M, "qr_us": tq, "qr_gbs": bq / (tq * 1e-6) / 1e9, "qr_frac": bq / (tq * 1e-6) / 1e9 / P,
                 "extrap_p": p, "extrap_us": te, "extrap_gbs": be / (te * 1e-6) / 1e9,
                 "extrap_frac": be / (te * 1e-6) / 1e9 / P, "l2_resident": ws_q <= L2}
            rows.append(r)
            print(json.dumps(r), flush=True)
    md = ["| N | M | QR(M) us/step | QR GB/s | QR frac | EXTRAP(p,M) us/step | EXTRAP GB/s | EXTRAP frac | note |",
          "|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        if "skipped" in r:
            md.append(f"| {r['N']} | {r['M']} | – | – | – | – | – | – | {r['skipped']} |")
        else:
            md.append(f"| {r['N']} | {r['M']} | {r['qr_us']:.1f} | {r['qr_gbs']:.0f} | {r['qr_frac']:.3f} | "
                      f"{r['extrap_us']:.1f} (p={r['extrap_p']}) | {r['extrap_gbs']:.0f} | {r['extrap_frac']:.3f} | "
                      f"{'L2-resident, not an HBM measurement' if r['l2_resident'] else ''} |")
    txt = "\n".join(md)
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write(f"# Bandwidth sweep (1 B200, peak {P} GB/s measured copy)\n\n" + txt + "\n")


if __name__ == "__main__":
    main()
