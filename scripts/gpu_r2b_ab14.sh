#!/bin/bash
# Kernel-v3 parameter re-sweep after the shared-gather change (L2 prefetch distance, quarters
# copied by the refill, register split) + the new rpt/8 parity cases.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab14
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py -q -x -k "dense_random_parity or shared_gather" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for L in libsrht.so libpfd2.so libpfd4.so libnref2.so libr160.so; do
  SRHT_LIB=$L timeout 300 python scripts/ab_time.py 5,4 >> $O/ab.jsonl 2>> $O/ab.err
done; done
