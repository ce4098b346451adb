#!/bin/bash
# traces: planner CTA (cur) vs 1aceb2c at C2 (n=128, M=8) and n=100 M=30
mkdir -p gpurun_out
for wt in 1aceb2c cur; do
  if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
  (cd $D && python -m paper_2009_10863_b200.build --trace > /dev/null 2>&1 && for c in 128:8 100:30 100:8; do
     n=${c%%:*}; m=${c##*:}; echo "=== $wt n=$n M=$m"; for r in 1 2 3; do TRACE_N=$n TRACE_M=$m timeout 600 python scripts/trace_phases.py 2>&1 | head -11 | grep -E "pass|barrier|exit|reduce"; echo; done; done)
done
