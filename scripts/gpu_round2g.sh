set -u
D=gpurun_out/r02g; mkdir -p $D
timeout 900 python -m pytest tests/test_forces.py -q > $D/forces.log 2>&1; tail -3 $D/forces.log
timeout 1800 python -m pytest tests -q -m gpu > $D/pytest.log 2>&1; tail -5 $D/pytest.log
ANKH_B200_LIB=$PWD/paper_2212_08284_b200/variants/libankh_b200_checked.so timeout 2400 python -m pytest tests -q -m gpu -x > $D/pytest_checked.log 2>&1; tail -5 $D/pytest_checked.log
