# v1 slab-length heuristic: parity subset and config 3 / 1 / 2 timing against the previous rule.
timeout 900 python -m pytest tests -m gpu -q -x -k "csc or batched or config or fp64 or shard or dense_random" > gpurun_out/mi_pytest.log 2>&1 || { echo "pytest failed"; grep -E "Error|assert|FAILED" gpurun_out/mi_pytest.log | head; exit 1; }
tail -1 gpurun_out/mi_pytest.log
bash scripts/gpu_v1_ab.sh libsrht.so libmi0.so
