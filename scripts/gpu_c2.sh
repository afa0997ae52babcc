#!/bin/bash
# Config-2 whole-column kernel: parity tests, then the bench line for each build variant.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -x -q -k "csc or config2 or dense_random or batched or fuzz" > gpurun_out/c2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c2_pytest.log
for L in libsrht.so libcolb4.so libcolb5.so libcolb6.so; do
  SRHT_LIB=$L timeout 300 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/c2_$L.json 2>/dev/null
done
