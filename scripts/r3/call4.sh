#!/bin/bash
# rolling pass 3 (one register set, OC kernels): bitwise A/B, parity with the variant, sweep A/B
mkdir -p gpurun_out
for v in base r3a; do cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  for pt in 1000000:16 1000000:30 3000000:30 300000:17 1000000:9; do echo "$v $(timeout 300 python scripts/r3/dump_guesses.py ${pt%%:*} ${pt##*:} x 2>&1 | tail -1)"; done
done
cp paper_2009_10863_b200/libig_r3a.so paper_2009_10863_b200/libig.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_sequences.py -q -x -p no:cacheprovider -k "open_loop_c1 or planner or 2p24 or orthonormality or rejection or sequence" 2>&1 | tail -2
VARIANTS="base r3b r3a" POINTS="300000:16,30 1000000:12,16,24,30 3000000:16,30 10000000:16,30" REPS=2 SWEEP_STEPS=30 bash scripts/r2_ab.sh
cp paper_2009_10863_b200/libig_base.so paper_2009_10863_b200/libig.so
