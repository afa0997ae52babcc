#!/bin/bash
# Profiles after the shared-gather change: ncu --set full of k_sketch_tma (config 5), clock64
# trace of CTA 0 (config-5 shape, trace build variant), ncu of the Gram kernels (configs 2, 4).
cd $GRAFT_REPO_ROOT
O=gpurun_out/prof
mkdir -p $O
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD1 > $O/plain1.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_sketch_tma -s 1 -c 1 -o $O/prof_c5 $CMD1 > $O/ncu_full.log 2>&1
ncu -i $O/prof_c5.ncu-rep --page raw --csv > $O/prof_c5_raw.csv 2>/dev/null
ncu -i $O/prof_c5.ncu-rep --page source --csv --print-source sass > $O/prof_c5_src.csv 2>/dev/null
rm -f $O/prof_c5.ncu-rep
timeout 300 python scripts/v3_trace.py 67108864 127 16384 > $O/trace_c5.txt 2>&1
for C in 2 4; do
  timeout 300 python scripts/gram_probe.py $C 3 > $O/gram_plain_c$C.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_mma -s 2 -c 1 -o $O/gram_c$C python scripts/gram_probe.py $C 3 > $O/ncu_gram_c$C.log 2>&1
  ncu -i $O/gram_c$C.ncu-rep --page raw --csv > $O/gram_c${C}_raw.csv 2>/dev/null
  ncu -i $O/gram_c$C.ncu-rep --page details > $O/gram_c${C}_details.txt 2>/dev/null
  rm -f $O/gram_c$C.ncu-rep
done
