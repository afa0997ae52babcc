# Power vs kernel time per knock-out mode: nvidia-smi at 20 ms alongside scripts/power_modes.py.
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw.instant,clocks_event_reasons.active --format=csv,noheader -lms 20 > gpurun_out/pw_clk.csv &
CLK=$!
SRHT_LIB=libsrht_dbg.so timeout 600 python scripts/power_modes.py 0,1,4,5 > gpurun_out/pw_modes.txt 2>&1
kill $CLK
