#!/bin/bash
# Config-2 whole-column kernel A/B: pruned last three row bits (default) vs full round C (cp0) vs
# 5 CTAs per SM without spills (cm5); parity of the batched / column-kernel paths first.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab6
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -q -x -k "column_kernel or batched or config2 or csc" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for L in libsrht.so libcp0.so libcm5.so; do
  SRHT_LIB=$L timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/c2_${L}_$rep.json 2> $O/c2_${L}_$rep.err
done; done
