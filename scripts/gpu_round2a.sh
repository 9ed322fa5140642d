set -u
D=gpurun_out/r02a; mkdir -p $D
timeout 1200 python -m pytest tests -x -q -m gpu > $D/pytest.log 2>&1; tail -3 $D/pytest.log
timeout 900 compute-sanitizer --tool memcheck --leak-check no python scripts/sanitize_case.py 0 1 > $D/memcheck.log 2>&1; echo "memcheck rc $?"; tail -5 $D/memcheck.log
