# Kernel v3: parity tests, config-5 bench, then one ncu --set full capture of k_sketch_tma.
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/v3_pytest.log 2>&1; echo "pytest exit $?"; tail -8 gpurun_out/v3_pytest.log
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/v3_plain_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sketch_tma -s 1 -c 1 -o gpurun_out/v3_prof_c5 $B > gpurun_out/v3_ncu_c5.log 2>&1; echo "ncu exit $?"; tail -3 gpurun_out/v3_ncu_c5.log
