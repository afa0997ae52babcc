set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; free -g; nproc
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest1.log 2>&1; echo "pytest exit $?"
tail -40 gpurun_out/pytest1.log
timeout 300 python __graft_entry__.py smoke
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -5
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -5
