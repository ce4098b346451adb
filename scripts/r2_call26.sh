#!/bin/bash
# one-copy pass 3 as separate kernel instantiations (OC) for M>8 below 2^24 vs HEAD (runtime branch in M<=32 only)
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do for wt in head cur; do
  if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
  echo "== $wt"; (cd $D && timeout 900 python scripts/bench_sweep.py --sizes 100000,1000000,3000000,10000000,134217728 --ms 12,16,30 --steps 20 2>&1 | grep '^{' | python /root/repo/scripts/probes/sweep_short.py)
  (cd $D && timeout 900 python bench.py --config c4 --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read().splitlines()[-1]); print('C4 $wt', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])")
done; done
