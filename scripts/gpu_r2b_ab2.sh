#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do
for L in libsrht.so libv3a.so libv3u.so libv3b.so; do
  SRHT_LIB=$L timeout 300 python scripts/ab_time.py 5,4 >> $O/ab.jsonl 2>> $O/ab.err
done
done
