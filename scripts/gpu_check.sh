# one-shot GPU verification used during development (outputs in gpurun_out/$1)
set -u
D=gpurun_out/${1:-check}
mkdir -p $D
for L in 3 4 5; do timeout 300 python scripts/svd_accuracy.py --order $L 2>&1 | tail -1; done
python scripts/plan_timing.py --config 3 --config 4 > $D/plan_timing.log 2>&1; grep -E "jacobi|factors|build" $D/plan_timing.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $D/bench.json 2>$D/bench.err; head -c 300 $D/bench.json; echo
timeout 1500 python -m pytest tests -x -q -m gpu > $D/pytest.log 2>&1; tail -2 $D/pytest.log
