#!/bin/bash
# final round-2 evidence (TAG r2g): everything scripts/r2_final.sh records, plus the C3 history
# sweep m = 1..30 at 2^27 DOFs (the metric's configuration)
export TAG=${TAG:-r2g}
T0=$SECONDS
bash scripts/r2_final.sh
timeout 1500 python scripts/bench_sweep.py --sizes 134217728 --ms $(seq -s, 1 30) --steps 10 --out gpurun_out/profiles_new/${TAG}_sweep_c3_m1_30.md > gpurun_out/c3m.log 2>&1; echo "c3 m-sweep rc=$?"
echo "final wall $((SECONDS-T0)) s"
