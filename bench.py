#!/usr/bin/env python
"""bench.py -- initial-guess form+update throughput on B200 (arXiv 2009.10863 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3|c2|c4]
                    [--scaling weak|strong] [--dry-run]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N ...

Headline workload (BASELINE.json configs[2], "C3", the configuration the metric is quoted on):
3D 512^3 7-point Poisson-like manufactured sequence, 2^27 = 134,217,728 fp64 DOFs per GPU,
projection QR(8) and extrapolation EXTRAP(3,8) on the same time steps.  One STEP = the whole hot
path once: QR form + QR update + EXTRAP form + EXTRAP update (push by copy) on that step's
(b_n, x_n, A x_n), all resident in HBM (1.07 GB vectors: every stream is an HBM stream, no L2
reuse between steps).  The line also carries the configs[1] point ("C2", 128^3 = 2^21 DOFs) under
"c2_l2_assisted": at 16.8 MB per vector L2 serves part of the update's re-reads, so that point is
NOT an HBM measurement (N < 2^24).  --config c4 selects configs[3] (2^28 DOFs/GPU,
QR(16)+EXTRAP(3,16)).

Scaling (N > 1 ranks, one per GPU): --scaling weak (default) gives every rank its own z-slab of
the config's size (global grid n x n x (nz*N)); --scaling strong splits the config's FIXED global
grid into N contiguous z-plane ranges (shard_range; sizes differ by at most one plane), so t(N)
can be compared with t(1): E(N) = t(1)/(N t(N)) (--t1-ms, or computed by the driver).  The
projection's global sums go through the in-kernel NVLink peer exchange (--exchange peer, default;
NCCL all-gather between kernels with --exchange nccl or when the GPUs lack P2P); extrapolation
never communicates.  --dry-run: no GPU work, prints the partition plan (CPU tests).

value = effective HBM GB/s of the whole job = (algorithmic bytes of all ranks) / (max-over-ranks
device time), algorithmic bytes per step and rank = [(8M+4) + (nnz(beta)+1) + 2] * 8 * N_rank
(DESIGN.md section 7).  ms_per_step is reported beside it.  Also on the JSON line: roofline (the
dominant kernel against the measured copy peak, plus read-only and nominal ceilings), kernels
(per-kernel event timing from a second pass), step_stats, fill_phase, clocks, e2e (host-buffer
batch calls, PCIe transfers inside the timed region), cpu_baseline (the CPU oracle).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "initial-guess form+update time/step & effective HBM GB/s (% of roofline), 1/2/4/8 B200"
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback (GB/s)
NOMINAL_HBM = 7700.0  # B200_PROFILING.md nominal HBM3e (HGX), for context
L2_BYTES = 126 * 2 ** 20


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=["c2", "c3", "c4"], default="c3",
                   help="c3 (default): configs[2] 512^3 (2^27 DOFs) QR(8)+EXTRAP(3,8); c2: configs[1] 128^3 "
                        "(L2-assisted); c4: configs[3] 2^28 DOFs/GPU QR(16)+EXTRAP(3,16)")
    p.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                   help="N>1: weak = a config-sized slab per rank; strong = the config's global grid split in z-slabs")
    p.add_argument("--t1-ms", type=float, default=None, help="strong scaling: t(1) in ms/step for E(N) = t(1)/(N t(N))")
    p.add_argument("--dry-run", action="store_true", help="no GPU work: print the partition plan (CPU tests)")
    p.add_argument("--no-c2", action="store_true", help="skip the extra C2 (L2-assisted) point of the default run")
    p.add_argument("--n", type=int, default=None, help="grid points per direction (per-GPU slab n^3), overrides --config")
    p.add_argument("--m", type=int, default=None, help="history size M (projection and extrapolation)")
    p.add_argument("--degree", type=int, default=3, help="extrapolation degree")
    p.add_argument("--e2e-steps", type=int, default=20)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="budget of the oracle cpu_baseline sample")
    p.add_argument("--cpu-seconds-1t", type=float, default=6.0, help="budget of the one-core oracle sample")
    p.add_argument("--same-gpu", action="store_true",
                   help="TEST MODE: all ranks on GPU 0 (gloo plumbing, 1/N of the SMs each) to exercise the N>1 path")
    p.add_argument("--exchange", choices=["peer", "nccl"], default="peer",
                   help="N>1 projection sums: in-kernel NVLink peer exchange (fused) or NCCL between kernels")
    a = p.parse_args()
    # (nx, ny, nz per GPU, M): the z extent is per rank (contiguous z-slabs, weak scaling)
    shape = {"c2": (128, 128, 128, 8), "c3": (512, 512, 512, 8), "c4": (512, 512, 1024, 16)}[a.config]
    a.n_override = a.n is not None
    if a.n is not None:
        shape = (a.n, a.n, a.n, shape[3])
    a.nxy, a.nz = shape[0], shape[2]
    a.n = a.nxy
    if a.m is None:
        a.m = shape[3]
    a.cfg_name = {"c2": "C2 configs[1]", "c3": "C3 configs[2]", "c4": "C4 configs[3]"}[a.config]
    return a


def partition(args, world: int, rank: int):
    """(nz_global, z0, z1): this rank's contiguous z-plane range (SURVEY §8(e) DOF shards)."""
    from paper_2009_10863_b200.ig import shard_range

    if args.scaling == "weak":  # every rank holds args.nz planes of an n x n x (nz*world) grid
        return args.nz * world, rank * args.nz, (rank + 1) * args.nz
    lo, hi = shard_range(args.nz, world, rank)  # the fixed n x n x nz grid, planes split evenly
    if hi <= lo:
        raise SystemExit(f"--scaling strong: {args.nz} z-planes cannot be split over {world} ranks")
    return args.nz, lo, hi


def l2_label(N: int) -> str | None:
    """per-vector sizes below 2^24 doubles are partly served by the 126 MB L2."""
    return "L2-assisted (N < 2^24), not an HBM measurement" if N < (1 << 24) else None


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


def read_only_ceiling(dev):
    """In-run read-only HBM ceiling: dots are pure reads and can exceed the copy
    rate.  torch.sum over a 2.1 GB fp64 vector, best of 5 (a measuring stick, not the product)."""
    import torch

    try:
        t = torch.ones(1 << 28, dtype=torch.float64, device=dev)
    except RuntimeError:
        return None
    best = None
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t.sum()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    del t
    torch.cuda.empty_cache()
    return 8 * (1 << 28) / (best * 1e-3) / 1e9


def bytes_per_step(M: int, N: int, nnz: int | None = None):
    """Algorithmic fp64 traffic of one steady step.  nnz = extrapolation weights
    that are nonzero (only those solutions are streamed; M for a dense scheme)."""
    vb = 8 * N
    nnz = M if nnz is None else nnz
    proj = (8 * M + 4) * vb  # form 2(M+1) + U1 2M + U2 M + U3 3M+2
    extrap = (nnz + 1) * vb + 2 * vb  # combine of the nonzero-weight solutions + write x0, push by copy
    per_kernel = {"form_dot": (M + 1) * vb, "form_combine": (M + 1) * vb, "u1": 2 * M * vb, "u2": M * vb,
                  "u3": (3 * M + 2) * vb, "extrap": (nnz + 1) * vb, "copy": 2 * vb,
                  "form_fused": 2 * (M + 1) * vb, "update_fused": (6 * M + 2) * vb}
    return proj, extrap, per_kernel


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.same_gpu:
        local = 0
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl" if (torch.cuda.is_available() and not args.same_gpu) else "gloo")
    return world, rank, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ------------------------------------------------------------------------------------------ oracle arm
def oracle_sample_run(n: int, M: int, degree: int, nz: int, steps: int, budget_s: float | None, fill: int):
    """Time the CPU oracle (as it stands) on a contiguous z-slab sample of the C2 grid.

    Returns (seconds per step, bytes per step, steps timed, N_sample)."""
    import numpy as np

    from oracle import ExtrapLS, ProjQR
    from workloads.gen import manufactured_step_slab

    world_equiv = n // nz
    N = n * n * nz
    op, oe = ProjQR(N, M), ExtrapLS(N, M, degree)

    def gen(k):
        return tuple(t.numpy() for t in manufactured_step_slab(n, nz, 0, world_equiv, k))

    x_prev = np.zeros(N)
    for k in range(fill):  # history fill, untimed
        b, x, Ax = gen(k)
        op.form_guess(b, x_prev)
        op.update(x, Ax)
        oe.form_guess(b, x_prev)
        oe.update(x)
        x_prev = x
    tot, done = 0.0, 0
    k = fill
    while done < steps and (budget_s is None or tot < budget_s):
        b, x, Ax = gen(k)
        t0 = time.perf_counter()
        op.form_guess(b, x_prev)
        op.update(x, Ax)
        oe.form_guess(b, x_prev)
        oe.update(x)
        tot += time.perf_counter() - t0
        x_prev = x
        done += 1
        k += 1
    nnz = int(np.count_nonzero(oe.weights()))
    pb, eb, _ = bytes_per_step(M, N, nnz)
    return tot / max(done, 1), pb + eb, done, N


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info

        th = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if th:
            return max(th)
    except Exception:
        pass
    return os.cpu_count()


def run_reference(args, world, rank):
    """--impl reference: the oracle timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    n, M, p = args.nxy, args.m, args.degree
    N_full = n * n * args.nz
    # the same contiguous z-slab sample as our arm's cpu_baseline (2^21 DOFs, 8 planes at C3), thinned
    # only when K is large so the whole --steps K --warmup W run stays within a few minutes
    nz = max(1, min(args.nz, (1 << 21) // (n * n)))
    if args.steps > 200:
        nz = max(1, nz * 200 // args.steps)
    # warm-up steps double as history fill; each timed step is one oracle step on the sample
    sps, bps, done, Ns = oracle_sample_run(n, M, p, nz, args.steps, None, max(args.warmup, M + 1))
    gbs = bps / sps / 1e9
    sample = (f"{nz} of {args.nz} z-planes of the {n}x{n}x{args.nz} {args.cfg_name} grid ({Ns} DOFs), "
              f"QR({M}) + EXTRAP({p},{M}) oracle steps, {done} timed after {max(args.warmup, M + 1)} fill steps")
    out = {"metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": sps * 1e3 * (N_full / Ns), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": f"{args.cfg_name}: 3D {n}x{n}x{args.nz} 7-point Helmholtz manufactured sequence "
                                  f"per GPU, QR({M}) + EXTRAP({p},{M})",
                      "sample": sample, "ms_per_step_note": "sample time scaled to the full grid"},
           "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cpu_cores(), "kind": "oracle", "sample": sample},
           "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------ our arm
def measure(args, world, rank, local, full: bool):
    """Time K steps of the hot path on this rank's slab; returns the JSON fields of one config.
    full=False (the extra C2 point): headline value, kernels and roofline only."""
    import torch

    from paper_2009_10863_b200 import (InitialGuess, comm_from_process_group, ig_form_guess_batch_host,
                                       ig_form_guess_host, ig_profile, ig_profile_read, ig_total_launches,
                                       ig_update_batch_host, ig_update_host, peers_from_process_group)
    from workloads.gen import manufactured_step_zrange

    n, M, p = args.nxy, args.m, args.degree
    nzg, z0, z1 = partition(args, world, rank)
    nz = z1 - z0
    N = n * n * nz
    N_total = n * n * (nzg if args.scaling == "strong" else args.nz * world)
    K, W = args.steps, args.warmup
    prefill = max(0, M + 1 - W)  # untimed history fill when W is too short to reach the steady state
    S = prefill + W + K
    dev = torch.device("cuda", local)

    # ---- inputs resident in HBM before the timed region: one fresh (b, x, Ax) per step, or --
    # when S steps of inputs would not fit next to the history (c3/c4) -- a pool of P = M+2
    # distinct steps cycled (a pair re-enters only after it left the M-window: still admitted)
    vec_gb = 8 * N / 1e9
    cap_gb = 0.85 * torch.cuda.get_device_properties(dev).total_memory / 1e9
    hist_gb = (3 * M + 4) * vec_gb  # QR slabs 2M, EXTRAP ring M, x0 buffers
    if 3 * S * vec_gb + hist_gb < cap_gb:
        P, regen = S, False
    elif 3 * (M + 2) * vec_gb + hist_gb < cap_gb:
        P, regen = M + 2, False
    else:
        # configs[3] (2^28 DOFs per GPU, M = 16): the history alone is ~110 GB, no input pool
        # fits.  Inputs are regenerated into fixed buffers between steps, OUTSIDE the timed
        # windows: every step is bracketed by its own events and the K windows are summed.
        P, regen = 1, True
    ro_gbs = read_only_ceiling(dev) if (rank == 0 and full) else None

    def gen(k):
        return manufactured_step_zrange(n, nzg, z0, z1, k, device=dev)

    pool = [gen(k) for k in range(P)]
    torch.cuda.synchronize()

    comm = comm_from_process_group() if (world > 1 and args.exchange == "nccl") else None
    hp = InitialGuess(N, "proj_qr", M, comm=comm)
    if world > 1 and args.exchange == "peer":
        if args.same_gpu:  # ranks share one GPU: each persistent kernel gets 1/world of the SMs
            from paper_2009_10863_b200 import ig_set_grid_limit

            ig_set_grid_limit(hp.h, torch.cuda.get_device_properties(dev).multi_processor_count // world)
        try:
            peers_from_process_group([hp.h])
            print(f"[bench] rank {rank}/{world}: in-kernel peer exchange attached (CUDA IPC windows of "
                  f"{world} ranks, NVLink P2P), {N} DOFs = z-planes [{z0}, {z1}) of {nzg}", file=sys.stderr, flush=True)
        except RuntimeError as e:  # no P2P between the GPUs: fall back to NCCL between kernels
            print(f"[bench] peer exchange unavailable ({e}); using NCCL", file=sys.stderr, flush=True)
            args.exchange = "nccl"
            hp.close()
            hp = InitialGuess(N, "proj_qr", M, comm=comm_from_process_group())
    if world > 1 and args.exchange == "nccl":
        print(f"[bench] rank {rank}/{world}: NCCL communicator attached, {N} DOFs = z-planes [{z0}, {z1}) of {nzg}",
              file=sys.stderr, flush=True)
    he = InitialGuess(N, "extrap_ls", M, p)
    x0p = torch.zeros(N, dtype=torch.float64, device=dev)
    x0e = torch.zeros(N, dtype=torch.float64, device=dev)

    def refill(k):  # regen mode: step k's inputs into the single pool slot (untimed)
        for dst, src in zip(pool[0], gen(k)):
            dst.copy_(src)
            del src

    def step(k):
        b, x, Ax = pool[k % P]
        hp.form_guess(b, x0p)
        hp.update(x, Ax)
        he.form_guess(None, x0e)
        he.update(x)

    for k in range(prefill + W):
        if regen:
            refill(k)
        step(k)
    torch.cuda.synchronize()
    assert hp.d == M, f"projection history not full after warm-up (d={hp.d})"

    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    l0 = ig_total_launches()
    with sampler:
        if not regen:
            e0.record(stream)
            th0 = time.perf_counter()
            for k in range(prefill + W, S):
                step(k)
            host_us = (time.perf_counter() - th0) / K * 1e6  # host enqueue cost per step (async launches)
            e1.record(stream)
            torch.cuda.synchronize()
            t_local = e0.elapsed_time(e1)
        else:
            t_local, host_us, launches_regen, step_ms = 0.0, 0.0, 0, []
            for k in range(prefill + W, S):
                refill(k)
                barrier(world)
                torch.cuda.synchronize()
                l1 = ig_total_launches()
                e0.record(stream)
                step(k)
                e1.record(stream)
                torch.cuda.synchronize()
                launches_regen += ig_total_launches() - l1
                step_ms.append(e0.elapsed_time(e1))
                t_local += step_ms[-1]
    barrier(world)
    launches = ig_total_launches() - l0 if not regen else launches_regen
    t_ms = max_over_ranks(t_local, world)
    st = hp.stats()
    fb, ub = hp.bytes()
    nnz = sum(1 for w in he.weights() if w != 0.0)
    pb, eb, per_kernel = bytes_per_step(M, N, nnz)
    assert fb + ub == pb, f"library byte count {fb + ub} != analytic {pb}"
    efb, eub = he.bytes()
    assert efb + eub == eb, f"library extrapolation byte count {efb + eub} != analytic {eb}"
    assert st["admitted"] == 1

    step_bytes = pb + eb  # this rank's
    pbT, ebT, _ = bytes_per_step(M, N_total, nnz)
    job_bytes = pbT + ebT  # all ranks (bytes are linear in the slab length)
    value = job_bytes * K / (t_ms * 1e-3) / 1e9
    ms_per_step = t_ms / K

    # ---- per-kernel CUDA-event timing over a second K-step pass (same inputs, cycled)
    ig_profile(hp.h, True)
    ig_profile(he.h, True)
    for k in range(prefill + W, S):
        if regen:
            refill(k + K)  # fresh steps (a repeated pair would take the rejection path)
        step(k)
    torch.cuda.synchronize()
    prof = ig_profile_read(hp.h)
    prof_e = ig_profile_read(he.h)
    for kk in ("extrap", "copy"):
        prof[kk] = prof_e[kk]
    ig_profile(hp.h, False)
    ig_profile(he.h, False)
    kernels = {}
    step_kernel_ms = sum(v[0] for v in prof.values()) / K
    for name, (ms, cnt) in prof.items():
        if cnt:
            avg = ms / cnt
            kernels[name] = {"avg_us": avg * 1e3, "launches": cnt, "gbs": per_kernel[name] / (avg * 1e-3) / 1e9,
                             "share": (ms / K) / step_kernel_ms}
    dom = max(kernels, key=lambda k: kernels[k]["avg_us"] * kernels[k]["launches"])
    peak, peak_src = peak_hbm()
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            key = f"{dom}@M{M}N{N}"
            if key in tj:
                traffic = tj[key]
                src = tj.get("_source", {}).get(key, "ncu --set full")
                traffic_src = f"profiles/traffic.json[{key}] (dram__bytes_read.sum + dram__bytes_write.sum, {src})"
        except Exception:
            pass
    roofline = {"bound": "hbm", "kernel": f"k_{dom}", "achieved": kernels[dom]["gbs"], "peak": peak, "unit": "GB/s",
                "frac": kernels[dom]["gbs"] / peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": per_kernel[dom], "traffic_source": traffic_src,
                "traffic_over_algorithmic": (traffic / per_kernel[dom]) if traffic else None,
                "step_frac": (step_bytes / (ms_per_step * 1e-3) / 1e9) / peak,
                "frac_nominal": kernels[dom]["gbs"] / NOMINAL_HBM}
    if full:
        roofline["ceilings_gbs"] = {"copy_measured": peak, "read_only_measured": ro_gbs, "nominal": NOMINAL_HBM,
                                    "read_only_how": "torch.sum over 2^28 fp64 (2.1 GB), best of 5, CUDA events"}
    res = {"value": value, "ms_per_step": ms_per_step, "N": N, "N_total": N_total, "z": (z0, z1, nzg), "M": M,
           "p": p, "nnz": nnz, "P": P, "regen": regen, "prefill": prefill, "step_bytes": step_bytes,
           "launches": launches, "roofline": roofline, "kernels": kernels, "clocks": sampler.summary(),
           "proj_state": {"d": st["d"], "rho_last": st["rho"]}, "host_us": host_us}
    if not full:
        hp.close()
        he.close()
        return res

    # ---- per-step distribution: a third pass with an event between consecutive steps (regen
    # mode: the headline's own per-step windows)
    if not regen:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
        evs[0].record(stream)
        for j, k in enumerate(range(prefill + W, S)):
            step(k)
            evs[j + 1].record(stream)
        torch.cuda.synchronize()
        step_ms = [evs[j].elapsed_time(evs[j + 1]) for j in range(K)]
    q = statistics.quantiles(step_ms, n=10) if len(step_ms) >= 2 else [step_ms[0]] * 9
    res["step_stats"] = {"median_us": statistics.median(step_ms) * 1e3, "p10_us": q[0] * 1e3, "p90_us": q[-1] * 1e3,
                         "steps": len(step_ms), "how": "per-step CUDA events (separate pass)" if not regen
                         else "the headline's per-step windows"}

    # ---- end to end through the public host-buffer API (H2D of inputs and D2H of guesses timed)
    # M+1 distinct host steps: a pair re-enters only after it left the M-window (admission path)
    PH = M + 1
    if regen or PH > len(pool) or 3 * PH * vec_gb > 40.0:
        res["e2e"] = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": 4 * 8 * N, "d2h_bytes_per_step": 2 * 8 * N,
                      "unavailable": "M+1 distinct pinned host input steps (to stay on the admission path) exceed 40 GB"}
    else:
        host = [tuple(t.cpu().pin_memory() for t in pool[(prefill + W + j) % len(pool)]) for j in range(PH)]
        x0h_p = torch.zeros(N, dtype=torch.float64).pin_memory()
        x0h_e = torch.zeros(N, dtype=torch.float64).pin_memory()
        KE = max(1, args.e2e_steps)
        # one untimed call pair per handle: allocates the staging buffers outside the timed region
        b, x, Ax = host[PH - 1]
        ig_form_guess_batch_host([hp, he], [b, None], [x0h_p, x0h_e])
        ig_form_guess_host(hp.h, b, x0h_p)

        def e2e_run(batch: bool):
            barrier(world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for j in range(KE):
                b, x, Ax = host[j % PH]
                if batch:  # one time step of the two fields: guesses, (the host solve), updates
                    ig_form_guess_batch_host([hp, he], [b, None], [x0h_p, x0h_e])
                    ig_update_batch_host([hp, he], [x, x], [Ax, None])
                else:
                    ig_form_guess_host(hp.h, b, x0h_p)
                    ig_update_host(hp.h, x, Ax)
                    ig_form_guess_host(he.h, None, x0h_e)
                    ig_update_host(he.h, x, None)
            torch.cuda.synchronize()
            return max_over_ranks(time.perf_counter() - t0, world)

        te1 = e2e_run(False)
        te = e2e_run(True)
        res["e2e"] = {"value": job_bytes * KE / te / 1e9, "unit": "GB/s", "ms_per_step": te / KE * 1e3,
                      "h2d_bytes_per_step": 4 * 8 * N, "d2h_bytes_per_step": 2 * 8 * N, "steps": KE,
                      "h2d_vectors": "QR: b, x, Ax (the fallback x0 is not uploaded once d > 0); EXTRAP: x",
                      "api": "ig_form_guess_batch_host/ig_update_batch_host (pinned host buffers, one call per "
                             "time step for both fields; transfers of the fields overlap)",
                      "single_calls": {"value": job_bytes * KE / te1 / 1e9, "ms_per_step": te1 / KE * 1e3,
                                       "api": "ig_form_guess_host/ig_update_host, one call per field"}}
        del host

    # ---- fill phase (reported separately from the steady state): both histories
    # reset, the first M+1 steps timed one by one (projection d = 0..M, extrapolation fill 0..M)
    res["fill_phase"] = None
    if not regen:
        hp.reset()
        he.reset()
        torch.cuda.synchronize()
        f_us, f_bytes = [], []
        for j in range(M + 1):
            e0.record(stream)
            step(prefill + W + j)
            e1.record(stream)
            torch.cuda.synchronize()
            f_us.append(e0.elapsed_time(e1) * 1e3)
            (a, b_), (c, d_) = hp.bytes(), he.bytes()
            f_bytes.append(a + b_ + c + d_)
        res["fill_phase"] = {"steps": M + 1, "us_per_step": [round(v, 1) for v in f_us],
                             "gbs_per_step": [round(bb / (u * 1e-6) / 1e9) for bb, u in zip(f_bytes, f_us)],
                             "bytes_per_step": f_bytes, "total_us": sum(f_us)}
    hp.close()
    he.close()
    return res


def cpu_baseline(args, n, M, p, N):
    """The CPU oracle (as it stands) on rank 0 at N=1: a bounded z-slab sample of the workload."""
    nz_cpu = args.nz if N <= (1 << 22) else max(1, (1 << 21) // (n * n))  # big configs: a 2M-DOF z-slab sample
    sps, bps, done, Ns = oracle_sample_run(n, M, p, nz_cpu, 10 ** 6, args.cpu_seconds, M + 1)
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=1):  # the same oracle on one host core
        sps1, bps1, done1, _ = oracle_sample_run(n, M, p, nz_cpu, 10 ** 6, args.cpu_seconds_1t, M + 1)
    return {"value": bps / sps / 1e9, "unit": "GB/s", "cores": cpu_cores(), "kind": "oracle",
            "one_core": {"value": bps1 / sps1 / 1e9, "unit": "GB/s", "cores": 1, "steps": done1},
            "ms_per_step": sps * 1e3,
            "sample": f"{Ns} DOFs ({'full grid' if Ns == N else f'{nz_cpu}-plane z-slab sample of the {n}x{n}x{args.nz} grid'}), "
                      f"{done} steady oracle steps (QR({M})+EXTRAP({p},{M})) after {M + 1} fill steps, "
                      f"~{args.cpu_seconds:.0f} s budget; GB/s = the step's algorithmic bytes / oracle time"}


def run_ours(args, world, rank, local):
    import copy

    import torch

    n, M, p = args.nxy, args.m, args.degree
    r = measure(args, world, rank, local, full=True)
    torch.cuda.empty_cache()
    c2 = None
    if args.config == "c3" and world == 1 and not args.no_c2 and not args.n_override and args.m == 8:
        a2 = copy.copy(args)
        a2.config, a2.nxy, a2.n, a2.nz, a2.m, a2.cfg_name = "c2", 128, 128, 128, 8, "C2 configs[1]"
        a2.steps, a2.warmup = max(args.steps, 200), max(args.warmup, 10)
        r2 = measure(a2, world, rank, local, full=False)
        torch.cuda.empty_cache()
        c2 = {"value": r2["value"], "unit": "GB/s", "ms_per_step": r2["ms_per_step"], "steps": a2.steps,
              "label": l2_label(r2["N"]),
              "workload": f"C2 configs[1]: 3D 128x128x128 7-point Helmholtz manufactured sequence, QR(8) + EXTRAP(3,8)",
              "dofs": r2["N"], "roofline": r2["roofline"], "kernels": r2["kernels"], "gpu_launches": r2["launches"],
              "clocks": r2["clocks"]}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, n, M, p, r["N"])
    if rank != 0:
        return
    N, P, nzg = r["N"], r["P"], r["z"][2]
    strong = args.scaling == "strong"
    if strong:
        workload = (f"{args.cfg_name}: 3D {n}x{n}x{nzg} 7-point manufactured sequence (fixed global grid, "
                    f"{r['N_total']} DOFs) split over {world} GPU(s) in z-slabs, QR({M}) + EXTRAP({p},{M})")
    else:
        workload = (f"{args.cfg_name}: 3D {n}x{n}x{args.nz} 7-point manufactured sequence per GPU, "
                    f"QR({M}) + EXTRAP({p},{M})")
    l2 = l2_label(N)
    cfg = {"workload": workload, "dofs_per_gpu": N, "global_dofs": r["N_total"], "input_pool_steps": P,
           "timing": ("K per-step event windows summed; inputs regenerated between steps outside the windows "
                      "(history + inputs exceed HBM)") if r["regen"] else "one event window over K steps",
           "history_m": M, "degree": p, "prefill_steps": r["prefill"], "bytes_per_step_per_gpu": r["step_bytes"],
           "bytes_model": "QR (8M+4)*8N + EXTRAP (nnz(beta)+1)*8N + push copy 2*8N", "extrap_nnz": r["nnz"],
           "l2": l2 if l2 else (("fresh inputs every step" if P == args.steps + args.warmup + r["prefill"]
                                 else f"inputs cycled over {P} steps (1 step re-enters after {P - 1} others)")
                                + f"; every vector {8 * N / 1e9:.2f} GB > L2 126 MB: HBM measurement"),
           "parallelism": f"dof-shard{world}" if world > 1 else "single",
           "exchange": (args.exchange if world > 1 else "none"),
           "mode": "TEST: all ranks on one GPU" if args.same_gpu else "one rank per GPU"}
    if strong:
        cfg["slab_planes"] = [list(partition(args, world, q)[1:]) for q in range(world)]
    out = {"metric": METRIC, "value": r["value"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
           "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
           "gpu_launches": r["launches"], "roofline": r["roofline"], "kernels": r["kernels"],
           "step_stats": r["step_stats"], "fill_phase": r["fill_phase"], "clocks": r["clocks"], "e2e": r["e2e"],
           "cpu_baseline": cpu, "c2_l2_assisted": c2, "proj_state": r["proj_state"],
           "host_enqueue_us_per_step": r["host_us"]}
    if strong:
        out["strong_scaling"] = {"t_ms_per_step": r["ms_per_step"], "t1_ms_per_step": args.t1_ms,
                                 "efficiency": (args.t1_ms / (world * r["ms_per_step"])) if args.t1_ms else None,
                                 "definition": "E(N) = t(1) / (N t(N)) at a fixed global grid (SURVEY §8(d))"}
    print(json.dumps(out), flush=True)


def run_dry(args, world, rank):
    """--dry-run: the partition plan only (no GPU): every rank's z-planes, gathered to rank 0."""
    import torch.distributed as dist

    nzg, z0, z1 = partition(args, world, rank)
    mine = [rank, z0, z1, args.nxy * args.nxy * (z1 - z0)]
    allp = [None] * world
    if world > 1:
        dist.all_gather_object(allp, mine)
    else:
        allp = [mine]
    if rank == 0:
        print(json.dumps({"dry_run": True, "scaling": args.scaling, "n_gpus": world, "config": args.config,
                          "nz_global": nzg, "grid": [args.nxy, args.nxy, nzg],
                          "global_dofs": args.nxy * args.nxy * nzg,
                          "slabs": [{"rank": q, "z0": a, "z1": b, "dofs": d} for q, a, b, d in allp]}), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        # the reference arm is the CPU oracle on rank 0 only: no process group, no GPU; the other
        # ranks of a torchrun launch exit 0 without work
        world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
        run_reference(args, world, rank)
        return
    world, rank, local = dist_setup(args)
    if args.dry_run:
        run_dry(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
