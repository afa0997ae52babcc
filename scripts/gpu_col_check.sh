# Whole-column kernel (N = 2^13): parity subset, config-2 timing against the tiled kernel.
timeout 900 python -m pytest tests -m gpu -q -x -k "dense_random or csc or batched or config or bernoulli or fp64 or end_to_end" > gpurun_out/col_pytest.log 2>&1 || { echo "pytest failed"; grep -E "Error|assert|FAILED" gpurun_out/col_pytest.log | head -20; exit 1; }
tail -1 gpurun_out/col_pytest.log
for v in 1 0 1 0; do
SRHT_V1_COL=$v timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/col_c2.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/col_c2.json').read().strip().splitlines()[-1]); r=d['roofline']; print('col=$v cfg 2', r['kernel'], 'kernel_ms %.4f frac %.3f' % (r['kernel_ms'], r['frac']))"
done
