#!/bin/bash
# M = 9..12 bucket (MC = 12): parity with it, A/B against the 16-column code
mkdir -p gpurun_out
cp paper_2009_10863_b200/libig_mc12.so paper_2009_10863_b200/libig.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_sequences.py -q -x -p no:cacheprovider -k "open_loop_c1 or planner or 2p24 or orthonormality or rejection or sequence or alias or zero or graph" 2>&1 | tail -3
VARIANTS="base mc12" POINTS="300000:9,12 1000000:9,10,12 3000000:12 20000000:9,12 134217728:12" REPS=2 SWEEP_STEPS=20 bash scripts/r2_ab.sh
cp paper_2009_10863_b200/libig_mc12.so paper_2009_10863_b200/libig.so
