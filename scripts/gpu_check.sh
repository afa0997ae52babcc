set -x
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest.log 2>&1; echo "pytest exit $?"
tail -30 gpurun_out/pytest.log
timeout 300 python __graft_entry__.py smoke
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 exit $?"; cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 exit $?"; cat gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
