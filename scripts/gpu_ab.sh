# A/B of experiment builds: SRHT_LIB=<lib> for each lib given as arguments.
set -x
for lib in "$@"; do
  SRHT_LIB=$lib timeout 600 python -m pytest tests/test_gpu_sketch.py -q -x > gpurun_out/ab_pytest_$lib.log 2>&1; echo "$lib pytest exit $?"; tail -1 gpurun_out/ab_pytest_$lib.log
  for c in 5 4; do
    SRHT_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${lib}_$c.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/ab_${lib}_$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$lib cfg $c', 'GB/s %.0f frac %.3f kernel_ms %.3f' % (d['value'], r['frac'], r['kernel_ms']), d['clocks']['sm_mhz'])"
  done
done
