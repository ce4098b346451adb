#!/bin/bash
# planner-CTA build: GPU tests, C3 bench, sweep points, small-N graph, traces
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 6 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 40 --warmup 20 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c3.log 2>&1
python -c "
import json
for l in open('gpurun_out/bench_c3.log'):
    if l.startswith('{'):
        d=json.loads(l); print('C3', round(d['ms_per_step']*1e3,1), round(d['value']), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, 'c2', round(d['c2_l2_assisted']['ms_per_step']*1e3,1))"
timeout 900 python scripts/bench_sweep.py --sizes 100000,1000000,10000000,134217728 --ms 8,16,30 --steps 20 2>&1 | grep '^{' | python scripts/probes/sweep_short.py
timeout 900 python scripts/small_n_graph.py --ms 8,30 > gpurun_out/small_n.log 2>&1; tail -n 8 gpurun_out/small_n.log
TRACE_CASES="46:30 100:30 100:16 512:16" bash scripts/r2_trace.sh
