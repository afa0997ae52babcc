#!/bin/bash
# Gram FP32 double-buffered staging (libsrht) vs FP64 single buffer (libgold): A/B + parity tests.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2d_gram
mkdir -p $O
for rep in 1 2 3; do for L in libsrht.so libgold.so libgc4.so libgc16.so; do for C in 4 2; do
  SRHT_LIB=$L timeout 300 python scripts/gram_ab.py $C 30 >> $O/ab.txt 2>&1; done; done; done
timeout 900 python -m pytest tests -m gpu -q -k "gram or nnls or pipeline or config" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python scripts/pipeline_bench.py 4 > $O/pipeline_c4.json 2>&1
timeout 300 python scripts/pipeline_bench.py 2 > $O/pipeline_c2.json 2>&1
echo done
