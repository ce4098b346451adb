#!/bin/bash
# per-pass traces of k_update_fused at M = 30 / 16 across N (where does mid-N lose?), then the default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
TRACE_CASES="100:30 144:30 215:30 512:30 100:16 144:16 215:16" bash scripts/r2_trace.sh > gpurun_out/r3_trace1.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r3_bench1.json 2> gpurun_out/r3_bench1.err; echo bench rc $?
tail -c 600 gpurun_out/r3_bench1.json
