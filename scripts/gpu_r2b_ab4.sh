#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab4
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for L in libsrht.so libgblk0.so; do for C in 2 4; do SRHT_LIB=$L timeout 300 python scripts/gram_probe.py $C 5 > $O/gram_${L}_c$C.log 2>&1; done; done
for rep in 1 2; do
for L in libsrht.so libqe0.so; do
  SRHT_LIB=$L timeout 300 python scripts/ab_time.py 5,4 >> $O/ab.jsonl 2>> $O/ab.err
done
done
