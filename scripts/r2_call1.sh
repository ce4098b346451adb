#!/bin/bash
# round-2 GPU call: build, GPU tests, closed-loop parity data, launch-mode A/B at C2 and C3
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 15 gpurun_out/pytest_gpu.log
timeout 600 python scripts/closed_loop_parity.py > gpurun_out/cl_parity.jsonl 2> gpurun_out/cl_parity.err
echo "cl rc=$?"
for cfg in c2 c3; do
  for mode in plain,pdl coop,pdl plain,pdl coop,pdl; do
    IG_LAUNCH=$mode timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_${cfg}_${mode}.log 2>&1
    echo "$cfg $mode: $(python -c "import json; d=json.loads([l for l in open('gpurun_out/ab_${cfg}_${mode}.log') if l.startswith('{')][-1]); print(round(d['value']), round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})")"
  done
done
