# A/B of experiment builds plus the whole-run v3 trace (config 5).
bash scripts/gpu_ab.sh "$@"
timeout 600 python scripts/v3_trace.py 67108864 127 16384 > gpurun_out/v3_trace_c5.txt 2>&1; echo "trace exit $?"; cat gpurun_out/v3_trace_c5.txt
