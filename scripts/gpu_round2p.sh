set -u
D=gpurun_out/r02p; mkdir -p $D
timeout 1500 python -m pytest tests/test_forces.py -q -m gpu > $D/pytest_forces.log 2>&1; echo "pytest rc $?"; tail -15 $D/pytest_forces.log
