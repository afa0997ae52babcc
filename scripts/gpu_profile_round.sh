# Round profile capture: bench JSON, launch list, full ncu of the top kernel (cfg5 and cfg4).
set -x
mkdir -p gpurun_out
CMD5="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full_c5.json 2> gpurun_out/bench_full_c5.err; echo "bench exit $?"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
CLK=$!
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_clk.json 2>&1
kill $CLK
timeout 900 $CMD5 > gpurun_out/plain_c5.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv $CMD5 > gpurun_out/ncu_launch.log 2>&1; echo "launch exit $?"
timeout 900 $CMD5 > gpurun_out/plain_c5b.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_sketch_ws -s 2 -c 1 -o gpurun_out/prof_ws_c5 $CMD5 > gpurun_out/ncu_full_c5.log 2>&1; echo "full exit $?"
