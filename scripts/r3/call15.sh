#!/bin/bash
# exact M = 5 bucket (mc5) vs M = 5 in the 6-column bucket (base)
mkdir -p gpurun_out
cp paper_2009_10863_b200/libig_mc5.so paper_2009_10863_b200/libig.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "open_loop_c1 or buckets_multi or misaligned" 2>&1 | tail -2
VARIANTS="base mc5" POINTS="134217728:5,6 20000000:5 1000000:5 300000:5" REPS=2 SWEEP_STEPS=10 bash scripts/r2_ab.sh
cp paper_2009_10863_b200/libig_mc5.so paper_2009_10863_b200/libig.so
