#!/bin/bash
# phase traces at 2^27 M=16: current vs d0db641 (the M=16 update regression)
mkdir -p gpurun_out
for wt in cur d0db641; do
  if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
  (cd $D && python -m paper_2009_10863_b200.build --trace > /dev/null 2>&1 && for c in 512:16 512:8; do
     n=${c%%:*}; m=${c##*:}; echo "=== $wt n=$n M=$m"; TRACE_N=$n TRACE_M=$m timeout 600 python scripts/trace_phases.py 2>&1 | head -12; done)
done
