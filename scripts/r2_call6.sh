#!/bin/bash
# bisect the M=16 update regression at C3 (per-kernel event times)
mkdir -p gpurun_out
for rep in 1 2; do
  for wt in d0db641 7087008 103285a cur; do
    if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
    (cd $D && timeout 600 python bench.py --config c3 --m 16 --steps 10 --warmup 4 --no-cpu-baseline --no-c2 --e2e-steps 1 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read().splitlines()[-1]); print('$wt', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})")
  done
done
