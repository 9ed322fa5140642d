set -u
O=gpurun_out/r02aa; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > $O/pytest_gpu.txt
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python scripts/forces_step.py --reps 3 > $O/forces_step.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/forces_launches.csv python scripts/forces_step.py --reps 1 > $O/forces_ncu.log 2>&1
tail -3 $O/pytest_gpu.txt; tail -c 600 $O/bench_c3.json; cat $O/forces_step.txt
