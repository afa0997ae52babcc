# Plan-time slab length: dense parity / shard / row-shard tests, config 4 and 5 bench lines.
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -q -x -k "dense or shard or repeatable or config or fp64 or host" > gpurun_out/sl_pytest.log 2>&1 || { echo "pytest failed"; grep -E "Error|assert|FAILED" gpurun_out/sl_pytest.log | head; exit 1; }
tail -1 gpurun_out/sl_pytest.log
for c in 4 5 4 5; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sl_c$c.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/sl_c$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('cfg $c step_ms %.4f kernel_ms %.4f frac %.3f' % (d['ms_per_step'], r['kernel_ms'], r['frac']))"
done
