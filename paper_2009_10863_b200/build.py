"""Build libig.so in-tree with nvcc for sm_100a (B200).  ``python -m paper_2009_10863_b200.build``.

Static cudart (the .so does not depend on torch's CUDA runtime); NCCL is dlopen'ed at run time.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "libig")
LIB = os.path.join(PKG, "libig.so")

SOURCES = ["kern_proj.cu", "kern_fused.cu", "kern_extrap.cu", "coeffs.cpp", "api.cpp"]
HEADERS = [os.path.join(CSRC, "ig_internal.h"), os.path.join(CSRC, "proj_common.cuh"), os.path.join(INCLUDE, "ig.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{CSRC}"]
# Debug build (`python -m paper_2009_10863_b200.build --trace`): per-CTA %globaltimer stamps in the
# fused update (scripts/trace_phases.py).  The default build has no variants.
TRACE_FLAGS = ["-DIG_TRACE=1"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, trace: bool = False, extra_flags=(), out: str | None = None) -> str:
    """extra_flags / out: experiment builds (A/B of table entries) into another library file."""
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    flags = FLAGS + (TRACE_FLAGS if trace else []) + list(extra_flags)
    lib_path = out or LIB
    # objects built with other flags (e.g. an IG_TRACE=1 debug build) are never reused
    stamp = os.path.join(BUILD, "flags.txt")
    want = " ".join(ARCH + flags)
    have = open(stamp).read() if os.path.exists(stamp) else None
    if have != want:
        force = True
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + HEADERS):
            lang = [] if src.endswith(".cu") else ["-x", "cu"] if False else []
            jobs.append((s, o, [nvcc, *ARCH, *flags, *lang, "-c", s, "-o", o]))

    def run(job):
        s, o, cmd = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stdout}\n{r.stderr}")
        log = os.path.join(BUILD, os.path.basename(s) + ".ptxas.txt")
        with open(log, "w") as f:
            f.write(r.stderr)
        return s

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for s in ex.map(run, jobs):
            if verbose:
                print("compiled", os.path.relpath(s, ROOT))
    if force or jobs or _stale(lib_path, objs):
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", lib_path, *objs, "-ldl", "-lpthread", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print("linked", os.path.relpath(lib_path, ROOT))
    with open(stamp, "w") as f:
        f.write(want)
    return lib_path


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv, trace="--trace" in sys.argv)
