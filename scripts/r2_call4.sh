#!/bin/bash
# per-kernel A/B at C3 with M=16 (current vs d0db641) + phase traces at small/mid N
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
  for wt in cur d0db641; do
    if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
    (cd $D && timeout 600 python bench.py --config c3 --m 16 --steps 20 --warmup 5 --no-cpu-baseline --no-c2 --e2e-steps 1 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read().splitlines()[-1]); print('$wt', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})")
  done
done
TRACE_CASES="46:8 46:30 100:8 100:16 100:30 215:16 215:30" bash scripts/r2_trace.sh
