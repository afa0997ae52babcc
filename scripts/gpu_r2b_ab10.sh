#!/bin/bash
# Config-3 tiled kernel A/B (run-summed CSC scatter vs shared atomics) + CSC parity.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab10
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -q -x -k "csc or config3 or config1 or batched or duplicate" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for L in libsrht.so libprev.so; do
  SRHT_LIB=$L timeout 300 python bench.py --config 3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $O/c3_${L}_$rep.json 2> $O/c3_${L}_$rep.err
done; done
