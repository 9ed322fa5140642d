set -u
O=gpurun_out/r02an; mkdir -p $O
timeout 1500 python -m pytest tests/test_forces.py tests/test_dropin_cpp.py -q -m gpu -x 2>&1 | tail -4 | tee $O/pytest_forces.txt
timeout 300 python scripts/forces_step.py --reps 3 --field > $O/field.txt 2>&1; cat $O/field.txt
