# Power of plain TMA streaming (scripts/mb_power.cu), nvidia-smi at 20 ms alongside.
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw.instant,clocks_event_reasons.active --format=csv,noheader -lms 20 > gpurun_out/pwmb_clk.csv &
CLK=$!
timeout 120 ./scripts/mb_power > gpurun_out/pwmb.txt 2>&1
kill $CLK
