#!/bin/bash
# Which configuration's first sketches fail: ab_time.py 5,4 and ab_time.py 4 in fresh processes.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c_st3
mkdir -p $O
for i in $(seq 1 ${NPROC:-30}); do
  for C in 5,4 4; do
    echo "== $i $C" >> $O/log.txt
    timeout 300 python scripts/ab_time.py $C > /dev/null 2> $O/err_cur.txt; rc=$?
    echo "rc=$rc" >> $O/log.txt
    grep -E "progress|Error|error" $O/err_cur.txt | tail -3 >> $O/log.txt
  done
done
