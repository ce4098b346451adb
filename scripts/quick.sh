#!/bin/bash
# quick loop: GPU parity tests (fast subset unless FULL=1) + bench (+ optional ncu).
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
if [ -z "${NOTEST}" ]; then timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/pytest_gpu.log; fi
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python - <<'PY'
import json
lines=open('gpurun_out/bench.log').read().splitlines()
try:
    d=json.loads([l for l in lines if l.startswith('{')][-1])
    print('VALUE', round(d['value']), 'ms/step', round(d['ms_per_step']*1e3,1),'us', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'step_frac', round(d['roofline']['step_frac'],3))
    for k,v in d['kernels'].items(): print('  ', k, round(v['avg_us'],1), 'us', round(v['gbs']), 'GB/s')
except Exception as e:
    print('bench parse failed', e); print('\n'.join(lines[-20:]))
PY
if [ -n "${NCU}" ]; then KREGEX="${KREGEX}" SKIP=${SKIP:-30} COUNT=${COUNT:-3} bash scripts/ncu_full.sh; fi
