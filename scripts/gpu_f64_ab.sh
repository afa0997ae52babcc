# FP64 parity mode: parity tests and config-4 time per library.
for lib in "$@"; do
SRHT_LIB=$lib timeout 600 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -q -x -k "fp64" > gpurun_out/f64_pytest.log 2>&1 || { echo "$lib pytest failed"; grep -E "Error|assert|FAILED" gpurun_out/f64_pytest.log | head -5; }
tail -1 gpurun_out/f64_pytest.log
SRHT_LIB=$lib timeout 300 python scripts/fp64_mode_time.py 2>&1 | tail -1 | sed "s/^/$lib /"
done
