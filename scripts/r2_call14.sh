#!/bin/bash
# round-2 evidence on the final planner build (TAG r2c) + extras
export TAG=r2c
T0=$SECONDS; bash scripts/evidence.sh; echo "evidence wall $((SECONDS-T0)) s"
mkdir -p gpurun_out/profiles_new
timeout 900 python scripts/small_n_graph.py --out gpurun_out/profiles_new/r2c_small_n_graph.md > gpurun_out/small_n.log 2>&1; tail -n 12 gpurun_out/small_n.log
T0=$SECONDS; python bench.py > gpurun_out/bench_default2.log 2>&1; echo "bench default wall $((SECONDS-T0)) s rc=$?"
timeout 900 python bench.py --config c4 --steps 10 --warmup 4 --no-c2 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?"; tail -c 600 gpurun_out/bench_c4.log
