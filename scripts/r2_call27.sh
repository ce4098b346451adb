#!/bin/bash
# planner CTA writes the control block (CTA 0 has no epilogue) vs HEAD
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do for wt in head cur; do
  if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
  echo "== $wt"; (cd $D && timeout 900 python scripts/bench_sweep.py --sizes 100000,300000,1000000,134217728 --ms 4,8,16,30 --steps 30 2>&1 | grep '^{' | python /root/repo/scripts/probes/sweep_short.py)
  (cd $D && timeout 600 python bench.py --steps 40 --warmup 20 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read().splitlines()[-1]); print('C3 $wt', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, 'C2', round(d['c2_l2_assisted']['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['c2_l2_assisted']['kernels'].items()})")
done; done
