# round-end evidence: default bench line, reference arm, config 4 line, ncu captures
set -u
D=gpurun_out/${1:-final}; mkdir -p $D
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; tail -c 600 $D/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > $D/bench_ref.json 2> $D/bench_ref.err; tail -c 300 $D/bench_ref.json
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err; tail -c 400 $D/bench_c4.json
bash scripts/profile_round.sh ${1:-final}
