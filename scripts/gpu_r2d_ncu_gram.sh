#!/bin/bash
# Config-4 Gram: launch list (k_gram_mma vs k_gram_reduce) and one full capture of k_gram_mma.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2d_ncu_gram
mkdir -p $O
timeout 300 python scripts/gram_ab.py 4 10 > $O/plain.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python scripts/gram_ab.py 4 6 > $O/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_mma -s 4 -c 1 \
  -o $O/gram_c4 python scripts/gram_ab.py 4 6 > $O/ncu2.log 2>&1
ncu -i $O/gram_c4.ncu-rep --page details --csv > $O/gram_c4_details.csv 2>&1
ncu -i $O/gram_c4.ncu-rep --page raw --csv > $O/gram_c4_raw.csv 2>&1
echo done
