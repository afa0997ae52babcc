set -x
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 exit $?"
cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 exit $?"
cat gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
timeout 600 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sketch_tiles -s 1 -c 1 -o gpurun_out/prof_c4 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c4.log 2>&1; echo "ncu exit $?"
tail -5 gpurun_out/ncu_c4.log
