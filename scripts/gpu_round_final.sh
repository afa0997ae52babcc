# Full GPU test suite, then the round's profile capture (scripts/gpu_profile_v3.sh) and the
# sustained-load drift / power evidence.
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/full_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/full_pytest.log
bash scripts/gpu_profile_v3.sh
bash scripts/gpu_drift.sh
