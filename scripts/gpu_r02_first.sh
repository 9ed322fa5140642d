# round-2 re-entry: tests, default bench, reference arm, profiles (outputs in gpurun_out/r02a)
set -u
D=gpurun_out/r02a; mkdir -p $D
nvidia-smi -L > $D/smi.txt
timeout 1500 python -m pytest tests -q -m gpu > $D/pytest.log 2>&1; tail -3 $D/pytest.log
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; tail -c 400 $D/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > $D/bench_ref.json 2> $D/bench_ref.err; tail -c 200 $D/bench_ref.json
bash scripts/profile_round.sh r02a
