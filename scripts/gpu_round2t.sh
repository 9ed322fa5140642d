set -u
D=gpurun_out/r02t; mkdir -p $D
ANKH_B200_LIB=$PWD/paper_2212_08284_b200/variants/libankh_b200_checked.so timeout 2700 python -m pytest tests -q -m gpu -k "not L16" > $D/pytest_checked.log 2>&1; echo "checked pytest rc $?"; tail -3 $D/pytest_checked.log; grep -c "ANKH_DASSERT\|guard" $D/pytest_checked.log
