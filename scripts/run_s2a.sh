D=gpurun_out/s2a; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/smi.txt
timeout 1200 python -m pytest tests -x -q -m gpu > $D/pytest.log 2>&1; tail -3 $D/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -2 $D/smoke.log
timeout 600 python bench.py > $D/bench.json 2> $D/bench.err; cat $D/bench.json | cut -c1-600
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > $D/bench_ref.json 2> $D/bench_ref.err; cut -c1-300 $D/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu.log 2>&1; echo ncu $?
