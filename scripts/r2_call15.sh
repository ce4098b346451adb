#!/bin/bash
# A/B: one-copy pass-3 trip loop for the M <= 32 bucket (cur) vs 5f8e36f
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_sequences.py -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do for wt in 5f8e36f cur; do
  if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
  echo "== $wt"; (cd $D && timeout 900 python scripts/bench_sweep.py --sizes 100000,1000000,10000000,134217728 --ms 17,24,30 --steps 20 2>&1 | grep '^{' | python /root/repo/scripts/probes/sweep_short.py)
done; done
timeout 600 ncu --set full --clock-control none -k regex:k_update_fused -s 40 -c 1 -o gpurun_out/u32_cur -f python scripts/probes/qr_steps.py 1000000 30 44 > /dev/null 2>&1
ncu -i gpurun_out/u32_cur.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio 2>/dev/null | tail -1
