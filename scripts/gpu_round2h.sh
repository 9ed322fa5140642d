set -u
D=gpurun_out/r02h; mkdir -p $D
timeout 900 python -m pytest tests/test_forces.py -q > $D/forces.log 2>&1; tail -3 $D/forces.log
timeout 300 python scripts/forces_step.py --config 3 --reps 3 > $D/forces_step.txt 2>&1; cat $D/forces_step.txt
ANKH_B200_LIB=$PWD/paper_2212_08284_b200/variants/libankh_b200_checked.so timeout 2400 python -m pytest tests -q -m gpu > $D/pytest_checked.log 2>&1; tail -5 $D/pytest_checked.log
timeout 900 python bench.py --no-cpu-baseline > $D/bench.json 2> $D/bench.err; tail -c 3000 $D/bench.json
