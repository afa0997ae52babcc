# Kernel v3 iteration: fast parity subset, trace, config 5/4 bench lines.
set -x
timeout 900 python -m pytest tests/test_gpu_sketch.py -q -x > gpurun_out/q_pytest.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/q_pytest.log
timeout 300 python scripts/v3_trace.py 67108864 127 16384 > gpurun_out/v3_trace_c5.txt 2>&1; cat gpurun_out/v3_trace_c5.txt
for c in 5 4; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_bench_c$c.json 2> gpurun_out/q_bench_c$c.err; echo "c$c exit $?"
python -c "import json; d=json.loads(open('gpurun_out/q_bench_c$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('cfg $c', r['kernel'], 'GB/s %.0f frac %.3f kernel_ms %.3f step_ms %.3f' % (d['value'], r['frac'], r['kernel_ms'], d['ms_per_step']))"
done
