#!/bin/bash
mkdir -p gpurun_out
python -m paper_2009_10863_b200.build --trace > gpurun_out/build_trace.log 2>&1 || { tail gpurun_out/build_trace.log; exit 1; }
for c in 100:30 100:8 46:8; do n=${c%%:*}; m=${c##*:}
  for L in coop plain,pdl; do IG_LAUNCH=$L TRACE_N=$n TRACE_M=$m timeout 300 python scripts/r3/gap_trace.py 2>&1 | tail -9; done
done
