# one-shot GPU verification used during development (outputs in gpurun_out/$1)
set -u
D=gpurun_out/${1:-check}
mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "instances_match or svd" > $D/new_tests.log 2>&1; tail -2 $D/new_tests.log
python scripts/plan_timing.py --config 3 --config 4 > $D/plan_timing.log 2>&1; grep -E "instances|pack|upload|m2l  |build" $D/plan_timing.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $D/bench.json 2>$D/bench.err; head -c 300 $D/bench.json; echo
timeout 1500 python -m pytest tests -x -q -m gpu > $D/pytest.log 2>&1; tail -2 $D/pytest.log
