#!/bin/bash
# One gpurun call: GPU tests, smoke, a short bench, and the ncu launch list of a short bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "from paper_2009_10863_b200.build import build; build(verbose=True)" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -rf ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "${NCU}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 3 --warmup 10 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
fi
for f in pytest_gpu smoke bench; do tail -n 3 gpurun_out/$f.log; done
