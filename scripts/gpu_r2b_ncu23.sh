#!/bin/bash
# ncu --set full of the config-2 column kernel and the config-3 tiled kernel (after plain runs).
cd $GRAFT_REPO_ROOT
O=gpurun_out/n23
mkdir -p $O
for C in ${CFGS:-2 3}; do
  K=$([ $C = 2 ] && echo k_sketch_col || echo k_sketch_tiles)
  CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 600 $CMD > $O/plain_c$C.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $O/prof_c$C $CMD > $O/ncu_c$C.log 2>&1
  ncu -i $O/prof_c$C.ncu-rep --page raw --csv > $O/prof_c${C}_raw.csv 2>/dev/null
  ncu -i $O/prof_c$C.ncu-rep --page details > $O/prof_c${C}_details.txt 2>/dev/null
  ncu -i $O/prof_c$C.ncu-rep --page source --csv --print-source sass > $O/prof_c${C}_src.csv 2>/dev/null
  rm -f $O/prof_c$C.ncu-rep
done
