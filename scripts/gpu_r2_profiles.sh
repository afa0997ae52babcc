#!/bin/bash
# Round-2 evidence for the headline kernel: drift record (back-to-back launches with clocks), the
# ncu launch list of the default bench command, and one ncu --set full capture of k_sketch_tma.
cd $GRAFT_REPO_ROOT
O=gpurun_out/pr
mkdir -p $O
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 20 > $O/drift_clocks.csv &
SMI=$!
timeout 600 python scripts/step_drift.py 5 > $O/drift_c5.txt 2>&1
kill $SMI
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launch.log 2>&1
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD1 > $O/plain1.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_sketch_tma -s 1 -c 1 -o $O/prof_c5 $CMD1 > $O/ncu_full.log 2>&1
