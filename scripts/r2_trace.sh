#!/bin/bash
# per-CTA phase traces of the fused kernels (debug --trace build) at the sizes named by TRACE_CASES
mkdir -p gpurun_out
python -m paper_2009_10863_b200.build --trace > gpurun_out/build_trace.log 2>&1 || { tail gpurun_out/build_trace.log; exit 1; }
CASES=${TRACE_CASES:-100:30 100:16}
for c in $CASES; do
  n=${c%%:*}; m=${c##*:}
  echo "=== n=$n (N=$((n*n*n))) M=$m"
  TRACE_N=$n TRACE_M=$m timeout 300 python scripts/trace_phases.py 2>&1 | tail -25
done
python -m paper_2009_10863_b200.build --force > /dev/null 2>&1  # leave the default build behind
