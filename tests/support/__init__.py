"""Test-only native helpers (built on demand with nvcc; never part of the product library)."""

from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
BUILD = os.path.join(ROOT, "build", "test_support")


def _build(name: str) -> str:
    src = os.path.join(HERE, f"{name}.cu")
    out = os.path.join(BUILD, f"lib{name}.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        os.makedirs(BUILD, exist_ok=True)
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared", "-Xcompiler", "-fPIC",
                        "-o", out, src], check=True, capture_output=True)
    return out


def hog_lib():
    """ctypes handle of libhog.so: hog_launch(blocks, smem_bytes, ns, started_dev_ptr, stream)."""
    lib = ctypes.CDLL(_build("hog"))
    lib.hog_launch.restype = ctypes.c_int
    lib.hog_launch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, ctypes.c_void_p, ctypes.c_void_p]
    return lib
