#!/usr/bin/env python
"""Summarise ncu outputs into profiles/: launch list (gpu__time_duration per launch) and one
--set full capture per hot kernel (DRAM bytes, throughput, occupancy, registers).

    python scripts/summarize_ncu.py --launches gpurun_out/launches.csv --full gpurun_out/prof.ncu-rep \
        --bench gpurun_out/bench.log --tag r1 [--M 8 --N 2097152]

Writes profiles/<tag>_launches.csv (copied), profiles/<tag>_ncu_summary.md and merges per-launch
DRAM traffic into profiles/traffic.json keyed "<kernel>@M<M>N<N>" (read by bench.py).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_active.avg",
    "sm__cycles_elapsed.avg",
]

SHORT = {
    "k_form_dot": "form_dot", "k_form_combine": "form_combine", "k_u1": "u1", "k_u2": "u2", "k_u3": "u3",
    "k_extrap": "extrap", "k_copy": "copy", "k_form_fused": "form_fused", "k_update_fused": "update_fused",
}


def kernel_short(name: str) -> str:
    m = re.search(r"(k_[a-z0-9_]+)", name)
    return SHORT.get(m.group(1), m.group(1)) if m else name


def to_bytes(val: str, unit: str) -> float:
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return v * scale


def to_us(val: str, unit: str) -> float:
    v = float(val.replace(",", ""))
    return v * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)


def read_full(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": kernel_short(r[head.index("Kernel Name")]), "name": r[head.index("Kernel Name")]}
        for m in METRICS:
            if m in head:
                i = head.index(m)
                d[m] = (r[i], units[i])
        res.append(d)
    return res


def read_launches(path: str):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    head = rows[0]
    out = []
    for r in rows[1:]:
        if len(r) < len(head):
            continue
        d = dict(zip(head, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        out.append((kernel_short(d["Kernel Name"]), to_us(d["Metric Value"], d["Metric Unit"])))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--bench")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--M", type=int, default=None, help="default: the bench line's history_m (else 8)")
    ap.add_argument("--N", type=int, default=None, help="default: the bench line's dofs_per_gpu (else 128^3)")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    bench_line, nnz = None, None
    if a.bench and os.path.exists(a.bench):
        lines = [l for l in open(a.bench).read().splitlines() if l.startswith("{")]
        if lines:
            bench_line = json.loads(lines[-1])
    cfg = (bench_line or {}).get("config", {})
    N = a.N or cfg.get("dofs_per_gpu") or 128 ** 3
    M = a.M or cfg.get("history_m") or 8
    nnz = cfg.get("extrap_nnz") or M  # extrapolation streams the nonzero weights only
    md = [f"# ncu summary `{a.tag}` (B200, bench.py {cfg.get('workload', 'C2').split(':')[0]}: N = {N} DOFs, M = {M})", ""]
    vb = 8 * N
    alg = {"form_dot": (M + 1) * vb, "form_combine": (M + 1) * vb, "u1": 2 * M * vb, "u2": M * vb,
           "u3": (3 * M + 2) * vb, "extrap": (nnz + 1) * vb, "copy": 2 * vb, "form_fused": 2 * (M + 1) * vb,
           "update_fused": (6 * M + 2) * vb}
    if bench_line is not None:
        md += ["## bench.py line (same build)", "", "```json", json.dumps(bench_line, indent=1)[:6000], "```", ""]
        shutil.copy(a.bench, os.path.join(prof, f"{a.tag}_bench.json"))
    if a.launches and os.path.exists(a.launches):
        shutil.copy(a.launches, os.path.join(prof, f"{a.tag}_launches.csv"))
        L = read_launches(a.launches)
        tot = sum(t for _, t in L) or 1.0
        agg = {}
        for k, t in L:
            agg.setdefault(k, []).append(t)
        md += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, cold/serialised)", "",
               "| kernel | launches | mean us | share of listed time | algorithmic GB/s at mean |", "|---|---|---|---|---|"]
        for k, ts in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            mean = sum(ts) / len(ts)
            gbs = alg.get(k, 0) / (mean * 1e-6) / 1e9 if k in alg else float("nan")
            md.append(f"| {k} | {len(ts)} | {mean:.1f} | {sum(ts) / tot:.3f} | {gbs:.0f} |")
        md.append("")
    traffic = {}
    tpath = os.path.join(prof, "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    if a.full and os.path.exists(a.full):
        R = read_full(a.full)
        md += ["## `ncu --set full` captures (one launch each, steady state)", "",
               "| kernel | us | DRAM read MB | DRAM write MB | DRAM total / algorithmic | DRAM % peak | L2 hit % | warps active % | regs | grid |",
               "|---|---|---|---|---|---|---|---|---|---|"]
        seen = {}
        for d in R:
            k = d["kernel"]
            t = to_us(*d["gpu__time_duration.sum"])
            rd = to_bytes(*d["dram__bytes_read.sum"])
            wr = to_bytes(*d["dram__bytes_write.sum"])
            ratio = (rd + wr) / alg[k] if k in alg else float("nan")
            md.append(f"| {k} | {t:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {ratio:.3f} | "
                      f"{float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'][0]):.1f} | "
                      f"{float(d.get('lts__t_sector_hit_rate.pct', ('nan',))[0]):.1f} | "
                      f"{float(d['sm__warps_active.avg.pct_of_peak_sustained_active'][0]):.1f} | "
                      f"{d['launch__registers_per_thread'][0]} | {d['launch__grid_size'][0]} |")
            seen.setdefault(k, []).append(rd + wr)
        for k, v in seen.items():
            traffic[f"{k}@M{M}N{N}"] = sum(v) / len(v)
        json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
        md.append("")
        shutil.copy(a.full, os.path.join(prof, f"{a.tag}_full.ncu-rep"))
    open(os.path.join(prof, f"{a.tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    sys.exit(main())
