#!/bin/bash
# Round-2 measurement sweep: full GPU tests, smoke, bench lines for every config and mode,
# Algorithm-1 stage timings.
cd $GRAFT_REPO_ROOT
O=gpurun_out/sw
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config 5 --accum fp64 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c5_fp64.json 2> $O/bench_c5_fp64.err
for C in 4 3 2 1; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-e2e > $O/bench_c$C.json 2> $O/bench_c$C.err
done
timeout 600 python bench.py --config 4 --accum fp64 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c4_fp64.json 2> $O/bench_c4_fp64.err
for C in 1 2 4; do timeout 600 python scripts/pipeline_bench.py $C > $O/pipe$C.json 2>&1; done
