timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest.log
SRHT_LIB=libsrht_dbg.so timeout 300 python scripts/ws_trace.py 1048576 512 8192 2>&1 | tee gpurun_out/trace_c4.txt
SRHT_LIB=libsrht_dbg.so timeout 300 python scripts/ws_experiments.py 1048576 512 8192 2>&1 | tee gpurun_out/exp_c4.txt
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 exit $?"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 exit $?"
