#!/bin/bash
# Full evidence run for one round tag: tests, smoke, bench (default args), launch list, ncu full.
TAG=${TAG:-r1}
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference ${BENCH_ARGS} > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
# launch list: 4 steady steps (warm-up launches skipped), cold-cache serialised
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 80 -c 16 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 40 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
KREGEX="k_update_fused|k_form_fused|k_extrap|k_copy" SKIP=40 COUNT=4 bash scripts/ncu_full.sh
python scripts/summarize_ncu.py --launches gpurun_out/launches.csv --full gpurun_out/prof.ncu-rep --bench gpurun_out/bench.log --tag ${TAG} > gpurun_out/summary.log 2>&1
# only this tag's files travel back (gpurun_out is capped at 64 MiB)
mkdir -p gpurun_out/profiles_new
cp profiles/${TAG}_* profiles/traffic.json gpurun_out/profiles_new/ 2>/dev/null
rm -f gpurun_out/prof.ncu-rep
for f in pytest_gpu smoke bench bench_ref; do tail -n 2 gpurun_out/$f.log; done
timeout 1200 python scripts/bench_sweep.py --out gpurun_out/profiles_new/${TAG}_sweep.md > gpurun_out/sweep.log 2>&1
bash scripts/sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1
cp gpurun_out/sanitize_summary.txt gpurun_out/profiles_new/${TAG}_sanitize_summary.txt
