set -x
timeout 300 python scripts/v3_trace.py > gpurun_out/v3_trace_c4.txt 2>&1; echo "exit $?"; cat gpurun_out/v3_trace_c4.txt
timeout 600 python scripts/v3_trace.py 67108864 127 16384 > gpurun_out/v3_trace_c5.txt 2>&1; echo "exit $?"; cat gpurun_out/v3_trace_c5.txt
