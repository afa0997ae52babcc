#!/bin/bash
# Gather-bank dealing A/B (libsrht.so: row-major bank dealing; libprev.so: round-robin dealing).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c_ab1
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_configs.py -q -x -k "dense or shared_gather or config4 or config5 or tma" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2 3; do for L in libsrht.so libprev.so; do
  SRHT_LIB=$L timeout 300 python scripts/ab_time.py 5,4 >> $O/ab.jsonl 2>> $O/ab.err
done; done
for L in libsrht.so libprev.so; do
  SRHT_LIB=$L timeout 600 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum -k regex:k_sketch_tma -s 3 -c 1 python scripts/ab_time.py 4 > $O/ncu_$L.txt 2>&1
done
