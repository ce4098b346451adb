#!/bin/bash
# A/B: planner CTA (cur) vs previous commit (1aceb2c), same box
mkdir -p gpurun_out
PTS="--sizes 100000,1000000,2097152,10000000 --ms 8,16,30 --steps 30"
for rep in 1 2; do
  for wt in 1aceb2c cur; do
    if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
    echo "== rep $rep $wt"; (cd $D && timeout 600 python scripts/bench_sweep.py $PTS 2>&1 | grep '^{' | python /root/repo/scripts/probes/sweep_short.py)
    (cd $D && timeout 600 python bench.py --config c2 --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read().splitlines()[-1]); print('C2 $wt', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})")
  done
done
