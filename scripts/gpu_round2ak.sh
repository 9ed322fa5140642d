set -u
O=gpurun_out/r02ak; mkdir -p $O
timeout 1500 python -m pytest tests/test_forces.py -q -m gpu -x 2>&1 | tail -4 | tee $O/pytest_forces.txt
