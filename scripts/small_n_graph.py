#!/usr/bin/env python
"""Small-N fixed cost: eager calls vs a captured step (VERDICT r1 "widen f3/f4").

Below ~1e6 DOFs a step of the hot path is dominated by per-call host launch cost, not HBM.  This
times, per (N, M), on one GPU with CUDA events over K consecutive steps:
  * QR(M) form+update of one field;
  * EXTRAP(3 or M-1, M) form+push of one field (eager: zero-copy push into ig_next_slot; graph:
    device window, push by copy -- 2 more values/element);
  * the multi-field step of the paper's solver (Table 7 mix): pressure by
    QR(M) + u_x, u_y, u_z by EXTRAP(p, M), the batch calls (one batched extrapolation launch).
"eager" = the Python binding's calls per step (what bench_sweep.py times); "graph" = the same
calls captured once per input buffer set (a pool of M+2 sets, so every projection update stays on
the admission path, each a graph bound to its own buffers) and replayed with ONE ig_graph_launch
per step.  Inputs are random device vectors; the history is filled before timing.

    python scripts/small_n_graph.py [--sizes 1e5,3e5,1e6] [--ms 4,8,16] [--steps 200] [--out f.md]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2009_10863_b200 import (CapturedStep, InitialGuess, ig_form_guess_batch,  # noqa: E402
                                   ig_update_batch)


def time_steps(fn, K, s):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for k in range(K):
        fn(k)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="100000,300000,1000000")
    ap.add_argument("--ms", default="4,8,16")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    s = torch.cuda.Stream()
    rows = []
    for N in [int(float(x)) for x in a.sizes.split(",")]:
        for M in [int(x) for x in a.ms.split(",")]:
            p = min(3, M - 1)
            pool = M + 2
            g = torch.Generator(device="cuda").manual_seed(10863 + M)
            rnd = lambda: torch.randn(N, dtype=torch.float64, device="cuda", generator=g)  # noqa: E731
            X = [[rnd() for _ in range(4)] for _ in range(pool)]   # per set: x of 4 fields
            AX = [[rnd() for _ in range(4)] for _ in range(pool)]
            B = [[rnd() for _ in range(4)] for _ in range(pool)]
            X0 = [[torch.zeros(N, dtype=torch.float64, device="cuda") for _ in range(4)] for _ in range(pool)]
            r = {"N": N, "M": M, "p": p}
            with torch.cuda.stream(s):
                # --- QR(M), one field
                hq = InitialGuess(N, "proj_qr", M, stream=s)

                def q_eager(k):
                    hq.form_guess(B[k % pool][0], X0[k % pool][0])
                    hq.update(X[k % pool][0], AX[k % pool][0])

                for k in range(pool):
                    q_eager(k)
                r["qr_eager_us"] = time_steps(q_eager, a.steps, s)
                graphs = []
                for k in range(pool):
                    with CapturedStep(s) as st:
                        q_eager(k)
                    graphs.append(st)
                for k in range(pool):
                    graphs[k].replay()
                r["qr_graph_us"] = time_steps(lambda k: graphs[k % pool].replay(), a.steps, s)
                assert hq.d == M and hq.stats()["admitted"] == 1
                for st in graphs:
                    st.close()
                hq.close()
                # --- EXTRAP(p, M), one field
                he = InitialGuess(N, "extrap_ls", M, p, stream=s)

                def e_eager(k):
                    slot = he.next_slot()
                    he.form_guess(None, slot)
                    he.update(slot)

                for k in range(pool):
                    e_eager(k)
                r["extrap_eager_us"] = time_steps(e_eager, a.steps, s)
                he.set_device_ring(True)
                graphs = []
                for k in range(pool):
                    with CapturedStep(s) as st:
                        he.form_guess(None, X0[k][1])
                        he.update(X0[k][1])
                    graphs.append(st)
                for k in range(pool):
                    graphs[k].replay()
                r["extrap_graph_us"] = time_steps(lambda k: graphs[k % pool].replay(), a.steps, s)
                for st in graphs:
                    st.close()
                he.close()
                # --- multi-field step: p by QR(M), u_x/u_y/u_z by EXTRAP(p, M)
                hs = [InitialGuess(N, "proj_qr", M, stream=s)] + [InitialGuess(N, "extrap_ls", M, p, stream=s)
                                                                   for _ in range(3)]

                def mf_eager(k):
                    ig_form_guess_batch(hs, B[k % pool], X0[k % pool])
                    ig_update_batch(hs, [X[k % pool][0]] + X0[k % pool][1:],
                                    AX[k % pool])

                for k in range(pool):
                    mf_eager(k)
                r["multi_eager_us"] = time_steps(mf_eager, a.steps, s)
                for h in hs[1:]:
                    h.set_device_ring(True)
                graphs = []
                for k in range(pool):
                    with CapturedStep(s) as st:
                        mf_eager(k)
                    graphs.append(st)
                for k in range(pool):
                    graphs[k].replay()
                r["multi_graph_us"] = time_steps(lambda k: graphs[k % pool].replay(), a.steps, s)
                assert hs[0].d == M
                for st in graphs:
                    st.close()
                for h in hs:
                    h.close()
            for key in ("qr", "extrap", "multi"):
                r[f"{key}_speedup"] = r[f"{key}_eager_us"] / r[f"{key}_graph_us"]
            rows.append(r)
            print(json.dumps(r), flush=True)
            del X, AX, B, X0
            torch.cuda.empty_cache()
    md = ["| N | M | QR(M) eager us | QR graph us | x | EXTRAP(p,M) eager us | graph us | x | "
          "QR(M)+3xEXTRAP eager us | graph us | x |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        md.append(f"| {r['N']} | {r['M']} | {r['qr_eager_us']:.1f} | {r['qr_graph_us']:.1f} | {r['qr_speedup']:.2f} | "
                  f"{r['extrap_eager_us']:.1f} (p={r['p']}) | {r['extrap_graph_us']:.1f} | {r['extrap_speedup']:.2f} | "
                  f"{r['multi_eager_us']:.1f} | {r['multi_graph_us']:.1f} | {r['multi_speedup']:.2f} |")
    txt = "\n".join(md)
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write("# Small-N fixed cost: eager calls vs captured step (1 B200, scripts/small_n_graph.py)\n\n"
                    "Per-step time over consecutive steps (CUDA events), history full, every projection update "
                    "admitted. EXTRAP eager pushes zero-copy (ig_next_slot); the graph pushes by copy (device "
                    "window, +2 values/element). L2-resident sizes: these are latency, not HBM, measurements.\n\n"
                    + txt + "\n")


if __name__ == "__main__":
    main()
