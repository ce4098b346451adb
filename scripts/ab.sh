# A/B two prebuilt libig variants on the C2 bench (no rebuild on the box)
for v in ${VARIANTS}; do
  cp paper_2009_10863_b200/libig_$v.so paper_2009_10863_b200/libig.so
  for rep in 1 2; do
    timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/b_$v.log 2>&1
    echo "$v rep$rep: $(python -c "import json; d=json.loads([l for l in open('gpurun_out/b_$v.log') if l.startswith('{')][-1]); print(round(d['value']), round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})")"
  done
done
