# Kernel v3 iteration: fast parity subset, config 5/4 bench lines, whole-run trace.
bash scripts/gpu_v3_quick.sh > gpurun_out/q_quick.log 2>&1 || { tail -8 gpurun_out/q_quick.log; exit 1; }
tail -2 gpurun_out/q_pytest.log
for c in 5 4; do python -c "import json; d=json.loads(open('gpurun_out/q_bench_c$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('cfg $c', r['kernel'], 'GB/s %.0f frac %.3f kernel_ms %.3f step_ms %.3f' % (d['value'], r['frac'], r['kernel_ms'], d['ms_per_step']), d['clocks'])"; done
timeout 300 python scripts/v3_trace.py 67108864 127 16384 raw > gpurun_out/v3_trace_c5.txt 2>&1; tail -12 gpurun_out/v3_trace_c5.txt
timeout 300 python scripts/step_drift.py 5 > gpurun_out/drift.txt 2>&1; python - <<'PY'
import re
t = open('gpurun_out/drift.txt').read()
for name in ("gap 0.5 s", "back to back"):
    m = re.search(name + r": \[([^\]]*)\]", t)
    if m:
        a = [float(x) for x in m.group(1).split(',')]
        print("%s: first5 %.3f  last50 %.3f ms" % (name, sum(a[:5]) / 5, sum(a[-50:]) / min(50, len(a))))
PY
