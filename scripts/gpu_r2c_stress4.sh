#!/bin/bash
# ab_time.py 5,4 in fresh processes with the stage of any failure named (AB_SYNC=1).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c_st4
mkdir -p $O
for i in $(seq 1 ${NPROC:-60}); do
  echo "== $i" >> $O/log.txt
  AB_SYNC=1 timeout 300 python scripts/ab_time.py 5,4 > /dev/null 2> $O/err_cur.txt; rc=$?
  echo "rc=$rc" >> $O/log.txt
  if [ $rc != 0 ]; then grep progress $O/err_cur.txt | tail -1 >> $O/log.txt; grep -E "Error" $O/err_cur.txt | head -2 >> $O/log.txt; fi
done
