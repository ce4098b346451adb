#!/bin/bash
# pass-2 b1 = Ax - B~c1 as two interleaved partial sums for the M<=32 bucket (ss) vs default; + GPU tests of HEAD
mkdir -p gpurun_out
cp paper_2009_10863_b200/libig.so /tmp/libig_default.so
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do for v in def ss; do
  cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  echo "== $v"; timeout 900 python scripts/bench_sweep.py --sizes 100000,1000000,3000000,10000000,134217728 --ms 24,30 --steps 20 2>&1 | grep '^{' | python scripts/probes/sweep_short.py
done; done
cp /tmp/libig_default.so paper_2009_10863_b200/libig.so
