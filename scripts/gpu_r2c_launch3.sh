#!/bin/bash
# Launch lists of configs 3, 2, 1 (per-kernel durations inside a step).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c_l3
mkdir -p $O
for C in 3 2 1; do
CMD="python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > $O/plain_c$C.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c$C.csv $CMD > $O/ncu_c$C.log 2>&1
done
