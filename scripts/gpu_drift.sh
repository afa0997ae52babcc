# Kernel-time drift under sustained load, with fast clock / power sampling alongside.
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,power.draw.instant,temperature.gpu,temperature.memory,clocks_event_reasons.active --format=csv -lms 20 > gpurun_out/drift_clk.csv &
CLK=$!
sleep 1
timeout 300 python scripts/step_drift.py 5 > gpurun_out/drift.txt 2>&1
sleep 0.5
kill $CLK
