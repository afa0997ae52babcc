#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab3
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for L in libp2.so; do SRHT_LIB=$L timeout 600 python -m pytest tests/test_gpu_sketch.py -q -x > $O/pytest_$L.log 2>&1; echo "rc=$?" >> $O/pytest_$L.log; done
for rep in 1 2; do
for L in libsrht.so libp1.so libp2.so libp3.so; do
  SRHT_LIB=$L timeout 300 python scripts/ab_time.py 5,4 >> $O/ab.jsonl 2>> $O/ab.err
done
done
