timeout 1800 python -m pytest tests -m gpu -q -x --timeout 1200 --durations=10 > gpurun_out/pytest.log 2>&1; echo "pytest exit $?"
tail -25 gpurun_out/pytest.log
