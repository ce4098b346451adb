#!/bin/bash
# A/B of prebuilt library variants (paper_2009_10863_b200/libig_<v>.so): sweep points + C2/C3 bench.
# VARIANTS="base new" POINTS="1000000:16,30 134217728:1,2" REPS=2
mkdir -p gpurun_out
for rep in $(seq 1 ${REPS:-1}); do
for v in ${VARIANTS}; do
  cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  for pt in ${POINTS}; do
    n=${pt%%:*}; ms=${pt##*:}
    timeout 600 python scripts/bench_sweep.py --sizes $n --ms $ms --steps ${SWEEP_STEPS:-20} 2>&1 | grep '^{' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$v', 'N',d['N'],'M',d['M'],'qr_us',round(d['qr_us'],1),'frac',round(d['qr_frac'],3),'ex_us',round(d['extrap_us'],1),'exfrac',round(d['extrap_frac'],3))"
  done
  for cfg in ${BENCH_CFGS}; do
    timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-c2 --e2e-steps 1 > gpurun_out/ab_${cfg}_$v.log 2>&1
    echo "$v $cfg: $(python -c "import json; d=json.loads([l for l in open('gpurun_out/ab_${cfg}_$v.log') if l.startswith('{')][-1]); print(round(d['value']), round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})")"
  done
done
done
