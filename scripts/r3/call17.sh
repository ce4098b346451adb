#!/bin/bash
# two-set rolling pass 3 also for the M = 17..20 one-copy kernel (r3x, 40 B spill) vs split pass 3 (base)
mkdir -p gpurun_out
for v in base r3x; do cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  for pt in 1000000:20 300000:17; do echo "$v $(timeout 300 python scripts/r3/dump_guesses.py ${pt%%:*} ${pt##*:} x 2>&1 | tail -1)"; done
done
VARIANTS="base r3x" POINTS="300000:20 1000000:17,20 3000000:20 10000000:20" REPS=2 SWEEP_STEPS=20 bash scripts/r2_ab.sh
cp paper_2009_10863_b200/libig_base.so paper_2009_10863_b200/libig.so
