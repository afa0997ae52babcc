#!/bin/bash
# Profiles: config-4 Gram (k_gram_mma + k_gram_reduce), config-2 Gram, config-3 tiled kernel.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c_prof1
mkdir -p $O
timeout 300 python scripts/gram_probe.py 4 10 > $O/gram4.log 2>&1
timeout 300 python scripts/gram_probe.py 2 5 > $O/gram2.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:k_gram -s 2 -c 2 -o $O/gram4 python scripts/gram_probe.py 4 2 > $O/ncu_gram4.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:k_sketch_tiles -s 3 -c 1 -o $O/tiles3 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_tiles3.log 2>&1
