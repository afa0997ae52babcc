#!/bin/bash
# Round-2 third-session sweep (bank dealing + refill quarters by RPT): GPU tests, smoke, A/B against
# the session-start library, bench lines for every config and mode, Algorithm-1 stages, drift,
# the ncu launch list and one full capture of k_sketch_tma (config 5), the config-4 end-to-end gate.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c_sw
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for rep in 1 2; do for L in libsrht.so libprev.so; do
  SRHT_LIB=$L timeout 300 python scripts/ab_time.py 5,4 >> $O/ab.jsonl 2>> $O/ab.err
done; done
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config 5 --accum fp64 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c5_fp64.json 2> $O/bench_c5_fp64.err
for C in 4 3 2 1; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-e2e > $O/bench_c$C.json 2> $O/bench_c$C.err
done
timeout 600 python bench.py --config 4 --accum fp64 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c4_fp64.json 2> $O/bench_c4_fp64.err
for C in 1 2 4; do timeout 600 python scripts/pipeline_bench.py $C > $O/pipe$C.json 2>&1; done
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap --format=csv -lms 20 > $O/drift_clocks.csv &
SMI=$!
timeout 600 python scripts/step_drift.py 5 > $O/drift_c5.txt 2>&1
kill $SMI
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launch.log 2>&1
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD1 > $O/plain1.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_sketch_tma -s 1 -c 1 -o $O/prof_c5 $CMD1 > $O/ncu_full.log 2>&1
ncu -i $O/prof_c5.ncu-rep --page raw --csv > $O/prof_c5_raw.csv 2>/dev/null
ncu -i $O/prof_c5.ncu-rep --page details > $O/prof_c5_details.txt 2>/dev/null
rm -f $O/prof_c5.ncu-rep
timeout 900 python scripts/e2e_gate.py 4 > $O/e2e_c4.json 2> $O/e2e_c4.err
