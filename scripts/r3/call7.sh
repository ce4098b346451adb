#!/bin/bash
# rolling prefetch for the large-vector M = 17..32 kernels (form RF + update passes 1-2): A/B
mkdir -p gpurun_out
for v in base big; do cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  for pt in 20000000:30 20000000:20; do echo "$v $(timeout 300 python scripts/r3/dump_guesses.py ${pt%%:*} ${pt##*:} x 2>&1 | tail -1)"; done
done
cp paper_2009_10863_b200/libig_big.so paper_2009_10863_b200/libig.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "full_size" 2>&1 | tail -2
VARIANTS="base big" POINTS="20000000:17,24,30 30000000:30 134217728:24,30" REPS=2 SWEEP_STEPS=20 bash scripts/r2_ab.sh
cp paper_2009_10863_b200/libig_base.so paper_2009_10863_b200/libig.so
