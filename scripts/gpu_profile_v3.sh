# Round-1 profile capture for kernel v3: bench JSON (config 5, default flags), clocks,
# launch list, one ncu --set full of k_sketch_tma (config 5) and of config 4.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/p_bench_c5.json 2> gpurun_out/p_bench_c5.err; echo "bench exit $?"
timeout 600 python bench.py --config 4 --steps 20 --warmup 5 > gpurun_out/p_bench_c4.json 2> gpurun_out/p_bench_c4.err; echo "bench4 exit $?"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/p_clocks.csv &
CLK=$!
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p_bench_c5_clk.json 2>&1
kill $CLK
CMD5="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 $CMD5 > gpurun_out/p_plain_c5.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p_launches_c5.csv $CMD5 > gpurun_out/p_ncu_launch.log 2>&1; echo "launch exit $?"
CMD5B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 $CMD5B > gpurun_out/p_plain_c5b.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_sketch_tma -s 1 -c 1 -o gpurun_out/p_prof_c5 $CMD5B > gpurun_out/p_ncu_full_c5.log 2>&1; echo "full exit $?"
CMD4="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD4 > gpurun_out/p_plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sketch_tma -s 1 -c 1 -o gpurun_out/p_prof_c4 $CMD4 > gpurun_out/p_ncu_full_c4.log 2>&1; echo "full4 exit $?"
