#!/bin/bash
# Session re-entry baseline: full GPU tests, smoke, default bench line, drift record.
cd $GRAFT_REPO_ROOT
O=gpurun_out/base
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 300 python scripts/step_drift.py 5 > $O/drift_c5.txt 2>&1
