#!/bin/bash
# ncu --set full capture of the hot kernels at the bench configuration (one launch each, steady state).
mkdir -p gpurun_out
OUT=${OUT:-gpurun_out/prof}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_u3|k_form_dot|k_form_combine|k_u1|k_u2|k_extrap}" \
  -s ${SKIP:-60} -c ${COUNT:-6} -o ${OUT} -f \
  python bench.py --steps 3 --warmup 12 --e2e-steps 1 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
tail -2 gpurun_out/ncu_full.log
