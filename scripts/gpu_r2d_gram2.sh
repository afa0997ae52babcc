#!/bin/bash
# Config-2 Gram (k_gram_mma_small): 2 CTAs per SM at 128 registers (libgm2, libgm2s single buffer)
# against the kept 1 CTA per SM (libsrht); digests must match.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2d_gram2
mkdir -p $O
for rep in 1 2 3; do for L in libsrht.so libgm2.so libgm2s.so; do
  SRHT_LIB=$L timeout 300 python scripts/gram_ab.py 2 20 >> $O/ab.txt 2>&1; done; done
SRHT_LIB=libgm2.so timeout 600 python -m pytest tests -m gpu -q -k "gram" > $O/pytest_gm2.log 2>&1; echo "rc=$?" >> $O/pytest_gm2.log
echo done
