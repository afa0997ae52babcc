#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab5
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sketch.py -q -x -k "gram or nnls" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for L in libsrht.so libgdb0.so; do for C in 2 4; do SRHT_LIB=$L timeout 300 python scripts/gram_probe.py $C 5 > $O/gram_${L}_c${C}_$rep.log 2>&1; done; done; done
timeout 600 python scripts/pipeline_bench.py 2 > $O/pipe2.json 2>&1
timeout 600 python scripts/pipeline_bench.py 4 > $O/pipe4.json 2>&1
