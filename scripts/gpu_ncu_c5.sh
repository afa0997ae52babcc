# One ncu --set full capture of k_sketch_tma on config 5 (after a clean run of the same command).
mkdir -p gpurun_out
CMD5B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 $CMD5B > gpurun_out/n_plain_c5.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_sketch_tma -s 1 -c 1 -o gpurun_out/n_prof_c5 $CMD5B > gpurun_out/n_ncu_full_c5.log 2>&1; echo "full exit $?"
