#!/bin/bash
# Kernel-v3 parameter re-check after the bank dealing (launched alone / back to back, configs 5 and 4).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c_ab3
mkdir -p $O
for rep in 1 2; do for L in libsrht.so libpfd4.so libnref2.so libch16.so libch4.so; do
  SRHT_LIB=$L timeout 300 python scripts/ab_time.py 5,4 >> $O/ab.jsonl 2>> $O/ab.err
done; done
