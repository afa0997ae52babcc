# Secondary evidence: Algorithm-1 stage timings (configs 1, 2, 4) and bench lines for configs 1-3.
for c in 1 2 4; do timeout 600 python scripts/pipeline_bench.py $c > gpurun_out/s_pipeline_c$c.json 2>&1; done
for c in 1 2 3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/s_bench_c$c.json 2> gpurun_out/s_bench_c$c.err; done
tail -n1 gpurun_out/s_pipeline_c*.json | cut -c1-200; tail -n1 gpurun_out/s_bench_c*.json | cut -c1-150
