#!/bin/bash
# Kernel-v3 A/B: parity of the default build, then config 5 / 4 bench lines per variant (alternating).
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sketch.py -q -x -k "dense_random or integer or tma or single_nonzero or shards or fuzz or row_shard" > gpurun_out/v3ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/v3ab_pytest.log
for rep in 1 2; do
for L in $LIBS; do
  SRHT_LIB=$L timeout 300 python bench.py --config 5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v3ab_${L}_c5_$rep.json 2>/dev/null
  SRHT_LIB=$L timeout 300 python bench.py --config 4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/v3ab_${L}_c4_$rep.json 2>/dev/null
done
done
