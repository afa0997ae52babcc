#!/bin/bash
# FP64 TMA kernel: parity tests, DADD microbenchmark, config-4 timing, bench line in FP64 mode.
cd $GRAFT_REPO_ROOT
./scripts/mb_dadd > gpurun_out/r2_mb_dadd.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_sketch.py -x -q -k "fp64 or dense_random or row_shard or binding or rows_finish" > gpurun_out/r2_f64_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2_f64_pytest.log
timeout 300 python scripts/fp64_mode_time.py > gpurun_out/r2_f64_time.json 2>&1
timeout 600 python bench.py --config 4 --accum fp64 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench_c4_f64.json 2> gpurun_out/r2_bench_c4_f64.err
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err
