# Kernel v3 iteration: fast parity subset + config 5/4 bench lines.
set -x
timeout 300 python -m pytest tests/test_gpu_sketch.py -q -x > gpurun_out/q_pytest.log 2>&1 || { echo "pytest failed"; tail -5 gpurun_out/q_pytest.log; exit 1; }; tail -2 gpurun_out/q_pytest.log
for rep in 1 2; do for c in 5 4; do
timeout 120 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_bench_c$c.json 2> gpurun_out/q_bench_c$c.err; echo "c$c exit $?"
python -c "import json; d=json.loads(open('gpurun_out/q_bench_c$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('cfg $c', r['kernel'], 'GB/s %.0f frac %.3f kernel_ms %.3f step_ms %.3f' % (d['value'], r['frac'], r['kernel_ms'], d['ms_per_step']), d['clocks'])"
done; done
