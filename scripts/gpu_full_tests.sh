set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/full_pytest.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/full_pytest.log
