#!/bin/bash
# post-r2g build (register coefficients for M = 9..12): full GPU tests, smoke, history sweeps (TAG r2h)
export TAG=${TAG:-r2h}
mkdir -p gpurun_out/profiles_new
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 1 --no-c2 > gpurun_out/profiles_new/${TAG}_bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 1500 python scripts/bench_sweep.py --sizes 134217728 --ms $(seq -s, 1 30) --steps 10 --out gpurun_out/profiles_new/${TAG}_sweep_c3_m1_30.md > gpurun_out/c3m.log 2>&1; echo "c3 m-sweep rc=$?"
timeout 2400 python scripts/bench_sweep.py --sizes 100000,300000,1000000,3000000,10000000,30000000,134217728,500000000,1000000000 --ms 1,2,4,8,16,30 --steps 10 --out gpurun_out/profiles_new/${TAG}_sweep_c5.md > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"
