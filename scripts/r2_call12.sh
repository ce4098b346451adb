#!/bin/bash
# ncu full of k_update_fused at N=1e6 M=30 and C2-size M=8: 1aceb2c vs current
mkdir -p gpurun_out
for wt in 1aceb2c cur; do
  if [ $wt = cur ]; then D=.; else D=build/wt_$wt; fi
  for c in 1000000:30 2097152:8; do n=${c%%:*}; m=${c##*:}
    (cd $D && timeout 600 ncu --set full --clock-control none -k regex:k_update_fused -s 40 -c 1 -o /root/repo/gpurun_out/u_${wt}_${n}_${m} -f python /root/repo/scripts/probes/qr_steps.py $n $m 44 > /root/repo/gpurun_out/ncu_${wt}_${n}_${m}.log 2>&1; echo "$wt $n $m rc=$?")
  done
done
