# Kernel v1 (CSC / batched / small N): parity tests and config 1-3 bench lines.
timeout 900 python -m pytest tests -m gpu -q -x -k "csc or batched or small or config or plan or tiny or sparse or v1 or shard" > gpurun_out/v1_pytest.log 2>&1 || { echo "pytest failed"; tail -15 gpurun_out/v1_pytest.log; exit 1; }
tail -1 gpurun_out/v1_pytest.log
for c in 2 3 1; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v1_c$c.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/v1_c$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('cfg $c', r.get('kernel'), 'step_ms %.4f kernel_ms %.4f frac %.3f' % (d['ms_per_step'], r.get('kernel_ms', 0), r['frac']))"
done
