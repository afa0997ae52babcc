timeout 1800 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/pytest.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest.log
for c in 4 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "c$c exit $?"; done
SRHT_LIB=libsrht_dbg.so timeout 300 python scripts/ws_experiments.py 1048576 512 8192 0,32,1,33,3,35 2>&1 | tee gpurun_out/exp_c4.txt
