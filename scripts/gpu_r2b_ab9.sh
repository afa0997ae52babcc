#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab9
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -q -x -k "column_kernel or batched or config2 or csc" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for L in libsrht.so libcse0.so; do
  SRHT_LIB=$L timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/c2_${L}_$rep.json 2> $O/c2_${L}_$rep.err
done; done
