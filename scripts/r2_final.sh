#!/bin/bash
# final round-2 evidence (TAG r2d): tests, smoke, bench (+reference arm), ncu launch list + full,
# sweep, sanitizers; closed-loop parity record; small-N graph table; C4 bench; C5 half-decade sweep
export TAG=${TAG:-r2d}
T0=$SECONDS; bash scripts/evidence.sh; echo "evidence wall $((SECONDS-T0)) s"
mkdir -p gpurun_out/profiles_new
timeout 900 python scripts/closed_loop_parity.py > gpurun_out/profiles_new/${TAG}_closed_loop_parity.jsonl 2> gpurun_out/cl.err; echo "closed loop rc=$?"
timeout 900 python scripts/small_n_graph.py --out gpurun_out/profiles_new/${TAG}_small_n_graph.md > gpurun_out/small_n.log 2>&1; echo "small-n rc=$?"
timeout 900 python bench.py --config c4 --steps 10 --warmup 4 --no-c2 > gpurun_out/profiles_new/${TAG}_bench_c4.json 2> gpurun_out/c4.err; echo "c4 rc=$?"
timeout 2400 python scripts/bench_sweep.py --sizes 100000,300000,1000000,3000000,10000000,30000000,134217728,500000000,1000000000 --ms 1,2,4,8,16,30 --steps 10 --out gpurun_out/profiles_new/${TAG}_sweep_c5.md > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"
