#!/bin/bash
# one-copy pass-3 loop threshold: MC>=32 (def) vs MC>=16 (oc16) vs MC>=8 (oc8)
mkdir -p gpurun_out
cp paper_2009_10863_b200/libig.so /tmp/libig_default.so
for rep in 1 2; do for v in def oc16 oc8; do
  cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  echo "== $v"; timeout 900 python scripts/bench_sweep.py --sizes 100000,1000000,10000000,134217728 --ms 8,12,16 --steps 20 2>&1 | grep '^{' | python scripts/probes/sweep_short.py
  timeout 600 python bench.py --steps 40 --warmup 20 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read().splitlines()[-1]); print('C3 $v', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, 'C2', round(d['c2_l2_assisted']['ms_per_step']*1e3,1))"
done; done
cp /tmp/libig_default.so paper_2009_10863_b200/libig.so
