#!/bin/bash
# noinline planner (small call interface) vs 1aceb2c: sweep, C2/C3 bench, traces
mkdir -p gpurun_out
for rep in 1 2; do for wt in 1aceb2c cur; do
  if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
  echo "== $wt"; (cd $D && timeout 600 python scripts/bench_sweep.py --sizes 100000,1000000,2097152,10000000 --ms 8,16,30 --steps 30 2>&1 | grep '^{' | python /root/repo/scripts/probes/sweep_short.py)
  (cd $D && timeout 600 python bench.py --steps 40 --warmup 20 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read().splitlines()[-1]); print('C3 $wt', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, 'C2', round(d['c2_l2_assisted']['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['c2_l2_assisted']['kernels'].items()})")
done; done
cp paper_2009_10863_b200/libig.so /tmp/libig_default.so
cp paper_2009_10863_b200/libig_tr.so paper_2009_10863_b200/libig.so
for c in 128:8 100:30 512:16; do n=${c%%:*}; m=${c##*:}; echo "=== tr n=$n M=$m"; TRACE_N=$n TRACE_M=$m timeout 600 python scripts/trace_phases.py 2>&1 | head -11; done
cp /tmp/libig_default.so paper_2009_10863_b200/libig.so
