#!/bin/bash
# per-column coefficients in registers for the M = 9..12 buckets (creg) vs shared memory (base)
mkdir -p gpurun_out
for v in base creg; do cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  for pt in 1000000:9 1000000:12 20000000:10; do echo "$v $(timeout 300 python scripts/r3/dump_guesses.py ${pt%%:*} ${pt##*:} x 2>&1 | tail -1)"; done
done
VARIANTS="base creg" POINTS="134217728:9,10,11,12 20000000:9,12 1000000:9,10,12 300000:9" REPS=2 SWEEP_STEPS=10 bash scripts/r2_ab.sh
cp paper_2009_10863_b200/libig_base.so paper_2009_10863_b200/libig.so
