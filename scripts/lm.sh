python -c "from paper_2009_10863_b200.build import build; build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for mode in "coop,pdl" "coop" "pdl" "none"; do
  IG_LAUNCH=$mode timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/b_$mode.log 2>&1
  echo "$mode: $(python -c "import json,sys; d=json.loads([l for l in open('gpurun_out/b_$mode.log') if l.startswith('{')][-1]); print(round(d['value']), round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})")"
done
