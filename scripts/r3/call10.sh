#!/bin/bash
# finer history buckets (6, 10, 14, 20, 28 added): parity with them, A/B against 1/2/4/8/12/16/24/32
mkdir -p gpurun_out
cp paper_2009_10863_b200/libig_fine.so paper_2009_10863_b200/libig.so
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_sequences.py -q -x -p no:cacheprovider -k "open_loop_c1 or planner or 2p24 or orthonormality or rejection or sequence or alias or zero or graph" 2>&1 | tail -3
VARIANTS="base fine" POINTS="134217728:5,6,9,10,13,14,17,19,20,25,28 1000000:5,9,13,17,25 20000000:9,13,17" REPS=2 SWEEP_STEPS=10 bash scripts/r2_ab.sh
cp paper_2009_10863_b200/libig_fine.so paper_2009_10863_b200/libig.so
