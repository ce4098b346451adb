#!/usr/bin/env python
"""Build experiment variants of libig (table overrides as -D flags) for scripts/r2_ab.sh.

    python scripts/build_variants.py name1:"-DIG_T_U_2=8 -DIG_T_U2_2=12" name2:"..."
-> paper_2009_10863_b200/libig_<name>.so (and restores the default build afterwards)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2009_10863_b200.build import PKG, build  # noqa: E402

for spec in sys.argv[1:]:
    name, _, flags = spec.partition(":")
    out = os.path.join(PKG, f"libig_{name}.so")
    build(force=True, extra_flags=flags.split(), out=out)
    print("built", out, flags, flush=True)
build(force=True)
