"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NONE of the method's arithmetic (no projection, no
Gram--Schmidt, no extrapolation weights).  It only draws the inputs: smooth
time-varying right-hand sides / solutions on 1D/2D/3D grids, counter-hash
noise, and the harness operator A = -Delta_h + sigma I (a 3/5/7-point
Helmholtz stencil) that turns a solution x into the A x the projection update
consumes.  The recipe is stated in DESIGN.md "Input recipe".
"""

from .gen import (  # noqa: F401
    Grid,
    SEED,
    counter_uniform,
    helmholtz_apply,
    helmholtz_diag,
    smooth_field,
    manufactured_step,
    prescribed_rhs,
)
