# GPU NNLS: parity tests and Algorithm-1 stage timings (configs 4 and 2).
timeout 600 python -m pytest tests/test_gpu_sketch.py -q -x -k "nnls or gram or end_to_end" > gpurun_out/nn_pytest.log 2>&1 || { echo "pytest failed"; tail -20 gpurun_out/nn_pytest.log; exit 1; }
tail -1 gpurun_out/nn_pytest.log
timeout 600 python scripts/pipeline_bench.py 4 > gpurun_out/pipe4.json 2>&1; tail -2 gpurun_out/pipe4.json
timeout 600 python scripts/pipeline_bench.py 2 > gpurun_out/pipe2.json 2>&1; tail -2 gpurun_out/pipe2.json
timeout 600 python scripts/pipeline_bench.py 4 > gpurun_out/pipe4b.json 2>&1; tail -1 gpurun_out/pipe4b.json | cut -c1-260
