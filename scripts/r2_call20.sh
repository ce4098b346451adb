#!/bin/bash
# grid barrier: red.release + acquire spin (bar) vs fence+atomic+nanosleep (def)
mkdir -p gpurun_out
cp paper_2009_10863_b200/libig.so /tmp/libig_default.so
for rep in 1 2; do for v in def bar; do
  cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  echo "== $v"; timeout 900 python scripts/bench_sweep.py --sizes 100000,300000,1000000 --ms 4,8,30 --steps 50 2>&1 | grep '^{' | python scripts/probes/sweep_short.py
  timeout 600 python bench.py --config c2 --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read().splitlines()[-1]); print('C2 $v', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done; done
cp /tmp/libig_default.so paper_2009_10863_b200/libig.so
