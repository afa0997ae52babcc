set -x
CMD="python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sketch -s 1 -c 1 -o gpurun_out/prof_ws_c4 $CMD > gpurun_out/ncu_ws_c4.log 2>&1; echo "ncu exit $?"
tail -3 gpurun_out/ncu_ws_c4.log
