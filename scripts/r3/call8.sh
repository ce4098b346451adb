#!/bin/bash
# M = 17..24 bucket (MC = 24) in the fused kernels: parity with it, A/B against the 32-column code
mkdir -p gpurun_out
cp paper_2009_10863_b200/libig_mc24.so paper_2009_10863_b200/libig.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_sequences.py -q -x -p no:cacheprovider -k "open_loop_c1 or planner or 2p24 or orthonormality or rejection or sequence or alias or zero or graph" 2>&1 | tail -3
VARIANTS="base mc24" POINTS="300000:20 1000000:17,20,24 3000000:24 20000000:17,20,24,25 134217728:20,24" REPS=2 SWEEP_STEPS=20 bash scripts/r2_ab.sh
cp paper_2009_10863_b200/libig_mc24.so paper_2009_10863_b200/libig.so
