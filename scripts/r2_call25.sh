#!/bin/bash
# torchrun paths on ONE GPU (two ranks time-sharing it, --same-gpu): weak and strong scaling lines
mkdir -p gpurun_out
for sc in strong weak; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 2 --same-gpu --scaling $sc --config c2 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tr_$sc.log 2> gpurun_out/tr_$sc.err
  echo "$sc rc=$?"; grep '^{' gpurun_out/tr_$sc.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['scaling'], d['n_gpus'], d['config'].get('global_dofs'), d['config'].get('dofs_per_gpu'), round(d['ms_per_step'],3), round(d['value']), d['config'].get('exchange'), d.get('strong_scaling'))"
  grep -i "peer\|nccl\|exchange" gpurun_out/tr_$sc.err | head -3
done
