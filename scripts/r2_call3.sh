#!/bin/bash
# round-2 call: new GPU tests (device window, captured steps, 2^24 parity), small-N graph timing,
# A/B of the M=16 large-N regression (current coop / current plain / d0db641 / f3e42b5), traces
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py -k "graph or 2p24 or capturable" -q -rf -x -p no:cacheprovider > gpurun_out/pytest_graph.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_graph.log
tail -n 15 gpurun_out/pytest_graph.log
timeout 900 python scripts/small_n_graph.py --out gpurun_out/r2b_small_n_graph.md > gpurun_out/small_n.log 2>&1; echo "small_n rc=$?"
tail -n 12 gpurun_out/small_n.log
PTS="--sizes 1000000,10000000,134217728 --ms 8,16,30 --steps 20"
for rep in 1 2; do
  echo "== rep $rep cur-coop";  timeout 600 python scripts/bench_sweep.py $PTS 2>&1 | grep '^{' | python scripts/probes/sweep_short.py
  echo "== rep $rep cur-plain"; IG_LAUNCH=plain,pdl timeout 600 python scripts/bench_sweep.py $PTS 2>&1 | grep '^{' | python scripts/probes/sweep_short.py
  for wt in d0db641 f3e42b5; do
    echo "== rep $rep $wt"; (cd build/wt_$wt && timeout 600 python scripts/bench_sweep.py $PTS 2>&1 | grep '^{' | python ../../scripts/probes/sweep_short.py)
  done
done
