"""CPU oracle for arXiv 2009.10863 (initial guesses for sequences of linear systems).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
under ``oracle/``.  The product path (``paper_2009_10863_b200``) never imports it
and shares no code with it: no kernels, headers, helpers, tables or constants.

The oracle is a plain, slow, obviously-correct fp64 transcription of the paper:

* ``proj_qr.ProjQR``      -- Algorithm 2 "Rolling QR" (§2), literal
  per-pass classical Gram--Schmidt, explicit norms, explicit Givens sweep.
* ``proj_qr.ProjClassic`` -- Algorithm 1 "Classic" (§2).
* ``extrap_ls.ExtrapLS``  -- Eq. EXTRAPEXPN with least-squares
  weights Eq. LSQRCOEFFS (§3.2) computed in EXACT rational
  arithmetic (``fractions.Fraction``) and rounded once to the nearest double.
* ``extrap_ls.naive_weights`` -- Theorem 3.1, Eq. NAIVEEXTRAPCOEFFS.
* ``sparse.sparse_weights``   -- Eq. CPQRCOEFFS (§3.3) (NEXT row f2).

Every function is pinned by ``tests/test_oracle_*.py`` to something other than
itself (paper-printed values, closed forms, brute-force least squares,
invariants); see DESIGN.md "Oracle pins".
"""

from .proj_qr import ProjQR, ProjClassic  # noqa: F401
from .extrap_ls import (  # noqa: F401
    ExtrapLS,
    ls_weights_exact,
    ls_weights,
    naive_weights,
    warmup_weights,
    lebesgue,
)
from .sparse import ExtrapSparse, cpqr_pivots_exact, sparse_weights, sparse_weights_exact  # noqa: F401
