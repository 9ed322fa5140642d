# closing check of the final tree: full GPU suite, smoke, the bench lines
set -u
O=gpurun_out/r02aq; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -6 > $O/pytest_gpu.txt; tail -3 $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" >> $O/pytest_gpu.txt 2>&1; tail -1 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 300 $O/bench_c4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/forces_launches.csv python scripts/forces_step.py --reps 1 --field > $O/forces_ncu.log 2>&1
