#!/bin/bash
# Gram: CTAs ordered by kind of block pair (heaviest first), uniform K-splits; libprev.so = row-major order.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c_ab4
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py -q -x -k "gram" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for L in libsrht.so libprev.so libgo12.so libgo16.so libgo6.so; do
  echo "$L" >> $O/gram4.log; SRHT_LIB=$L timeout 300 python scripts/gram_probe.py 4 20 2>&1 | tail -10 >> $O/gram4.log
done; done
