#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab13
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py -q -x -k "gram or nnls" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for L in libsrht.so libgcv0.so; do for C in 2 4; do SRHT_LIB=$L timeout 300 python scripts/gram_probe.py $C 5 > $O/gram_${L}_c${C}_$rep.log 2>&1; done; done; done
timeout 600 ncu --metrics sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__shared_mem_config_size -k regex:k_gram_mma_small -s 2 -c 1 python scripts/gram_probe.py 2 3 > $O/ncu_occ.log 2>&1
