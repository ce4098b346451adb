#!/bin/bash
# per-column coefficients in registers also for the M = 13..14 bucket (creg14) vs M <= 12 only (base)
mkdir -p gpurun_out
for v in base creg14; do cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  for pt in 1000000:13 20000000:14; do echo "$v $(timeout 300 python scripts/r3/dump_guesses.py ${pt%%:*} ${pt##*:} x 2>&1 | tail -1)"; done
done
VARIANTS="base creg14" POINTS="134217728:13,14 20000000:13 1000000:13,14" REPS=2 SWEEP_STEPS=10 bash scripts/r2_ab.sh
cp paper_2009_10863_b200/libig_base.so paper_2009_10863_b200/libig.so
