# Config 2 (batched CSC): bench line and one ncu --set full capture of its tile kernel.
mkdir -p gpurun_out
timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err; echo "bench exit $?"
CMD="python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/c2_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sketch_col -s 1 -c 1 -o gpurun_out/c2_prof $CMD > gpurun_out/c2_ncu.log 2>&1; echo "ncu exit $?"
