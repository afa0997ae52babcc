# Gram kernel: parity tests and Algorithm-1 stage timings (configs 2 and 4).
timeout 600 python -m pytest tests/test_gpu_sketch.py -q -x -k "gram or nnls or end_to_end" > gpurun_out/gr_pytest.log 2>&1 || { echo "pytest failed"; tail -20 gpurun_out/gr_pytest.log; exit 1; }
tail -1 gpurun_out/gr_pytest.log
for c in 2 4; do timeout 600 python scripts/pipeline_bench.py $c 2>&1 | tail -1 | cut -c1-330; done
