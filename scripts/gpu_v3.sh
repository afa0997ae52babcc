# Kernel v3 bring-up on one B200: parity tests, then config 4/5 bench lines for v3 and v2.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v3_pytest.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/v3_pytest.log
for k in v3 v2; do
  SRHT_KERNEL=$k timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v3_bench_c4_$k.json 2> gpurun_out/v3_bench_c4_$k.err; echo "c4 $k exit $?"
  tail -c 600 gpurun_out/v3_bench_c4_$k.json; tail -3 gpurun_out/v3_bench_c4_$k.err
  SRHT_KERNEL=$k timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v3_bench_c5_$k.json 2> gpurun_out/v3_bench_c5_$k.err; echo "c5 $k exit $?"
  tail -c 600 gpurun_out/v3_bench_c5_$k.json; tail -3 gpurun_out/v3_bench_c5_$k.err
done
