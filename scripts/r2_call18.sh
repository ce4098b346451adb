#!/bin/bash
# one-copy pass-3 loop for the M<=32 bucket below 2^24 (runtime branch): tests + sweep vs 5f8e36f
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do for wt in 5f8e36f cur; do
  if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
  echo "== $wt"; (cd $D && timeout 900 python scripts/bench_sweep.py --sizes 100000,1000000,10000000,134217728 --ms 17,24,30 --steps 20 2>&1 | grep '^{' | python /root/repo/scripts/probes/sweep_short.py)
done; done
