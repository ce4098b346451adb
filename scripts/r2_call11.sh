#!/bin/bash
# pass-3 slowdown experiments: claim-loop form, dynamic tail fraction
mkdir -p gpurun_out
cp paper_2009_10863_b200/libig.so /tmp/libig_default.so
cp /tmp/libig_default.so paper_2009_10863_b200/libig_cur.so
for v in tr_cur tr_claim tr_t4 tr_t16; do
  cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  for c in 128:8 100:30; do n=${c%%:*}; m=${c##*:}; echo "=== $v n=$n M=$m"
    for r in 1 2; do TRACE_N=$n TRACE_M=$m timeout 600 python scripts/trace_phases.py 2>&1 | head -11 | grep -E "barrier2|pass3"; done; done
done
for rep in 1 2; do for v in cur claim t4 t16; do
  cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  echo "== $v"; timeout 600 python scripts/bench_sweep.py --sizes 1000000,2097152,10000000 --ms 8,30 --steps 30 2>&1 | grep '^{' | python scripts/probes/sweep_short.py
done; done
cp /tmp/libig_default.so paper_2009_10863_b200/libig.so
