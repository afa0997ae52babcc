# Kernel v2 (fallback for unaligned columns): parity subset and config-5/4 timing.
SRHT_KERNEL=v2 timeout 300 python -m pytest tests/test_gpu_sketch.py -q -x -k "v2 or dense" > gpurun_out/v2_pytest.log 2>&1; tail -1 gpurun_out/v2_pytest.log
for c in 5 4; do
SRHT_KERNEL=v2 timeout 120 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v2_c$c.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/v2_c$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('v2 cfg $c', r['kernel'], 'kernel_ms %.3f frac %.3f' % (r['kernel_ms'], r['frac']))"
done
