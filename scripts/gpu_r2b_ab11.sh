#!/bin/bash
# Knock-out: kernel v3 without the consumers' frame flips (results wrong; timing only).
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab11
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_sketch.py -q -x -k "column_kernel or shared_gather" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for L in libsrht.so libkonf.so; do
  SRHT_LIB=$L timeout 300 python scripts/ab_time.py 5 >> $O/ab.jsonl 2>> $O/ab.err
done; done
