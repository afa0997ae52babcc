# Kernel v1 A/B: config 2/3 kernel times per library (SRHT_LIB=<lib>).
for lib in "$@"; do for c in 2 3; do
SRHT_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v1ab_$c.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/v1ab_$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$lib cfg $c kernel_ms %.4f' % r.get('kernel_ms', 0))"
done; done
