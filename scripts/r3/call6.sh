#!/bin/bash
# rolling form kernel (M > 8 below 2^24): bitwise A/B, parity, sweep A/B
mkdir -p gpurun_out
for v in base rf; do cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  for pt in 1000000:16 1000000:30 300000:12 3000000:17; do echo "$v $(timeout 300 python scripts/r3/dump_guesses.py ${pt%%:*} ${pt##*:} x 2>&1 | tail -1)"; done
done
cp paper_2009_10863_b200/libig_rf.so paper_2009_10863_b200/libig.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_sequences.py -q -x -p no:cacheprovider -k "open_loop_c1 or planner or 2p24 or orthonormality or rejection or sequence or alias or zero" 2>&1 | tail -2
VARIANTS="base rf" POINTS="300000:12,16,30 1000000:12,16,24,30 3000000:16,30 10000000:16,30" REPS=2 SWEEP_STEPS=30 bash scripts/r2_ab.sh
cp paper_2009_10863_b200/libig_base.so paper_2009_10863_b200/libig.so
