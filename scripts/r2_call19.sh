#!/bin/bash
# ncu: M=16 bucket pass-1 slowdown (254-register build 103285a vs 252-register 5f8e36f) at 2^24
mkdir -p gpurun_out
for wt in 103285a 5f8e36f; do
  (cd build/wt_$wt && timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_update_fused -s 40 -c 1 -o /root/repo/gpurun_out/m16_${wt} -f python /root/repo/scripts/probes/qr_steps.py 16777216 16 44 > /dev/null 2>&1; echo "$wt rc=$?")
done
