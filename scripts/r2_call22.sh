#!/bin/bash
# MC=16 bucket: X~ loads split from the B~ part (s16), + one-copy pass 3 below 2^24 (s16oc)
mkdir -p gpurun_out
cp paper_2009_10863_b200/libig.so /tmp/libig_default.so
for rep in 1 2; do for v in def s16 s16oc; do
  cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  echo "== $v"; timeout 900 python scripts/bench_sweep.py --sizes 1000000,10000000,134217728 --ms 12,16 --steps 20 2>&1 | grep '^{' | python scripts/probes/sweep_short.py
done; done
for v in def s16 s16oc; do
  cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  timeout 900 python bench.py --config c4 --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read().splitlines()[-1]); print('C4 $v', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
cp /tmp/libig_default.so paper_2009_10863_b200/libig.so
