#!/bin/bash
# Config-4 Gram (k_gram_mma): 5 / 6 CTAs per SM (register caps 96 / 80, some spills) against 4
# (libsrht, which now also carries the 2-CTA config-2 kernel); GPU Gram/NNLS tests; pipelines.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2d_gram3
mkdir -p $O
for rep in 1 2 3; do for L in libsrht.so libgmm5.so libgmm6.so; do
  SRHT_LIB=$L timeout 300 python scripts/gram_ab.py 4 30 >> $O/ab.txt 2>&1; done; done
timeout 900 python -m pytest tests -m gpu -q -k "gram or nnls or pipeline" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python scripts/pipeline_bench.py 2 > $O/pipeline_c2.json 2>&1
timeout 300 python scripts/pipeline_bench.py 4 > $O/pipeline_c4.json 2>&1
echo done
