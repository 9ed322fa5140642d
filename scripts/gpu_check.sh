# one-shot GPU verification used during development (outputs in gpurun_out/$1)
set -u
D=gpurun_out/${1:-check}
mkdir -p $D
timeout 1500 python -m pytest tests -x -q -m gpu > $D/pytest.log 2>&1; tail -2 $D/pytest.log
ANKH_STREAM_INPUT=1 timeout 1500 python -m pytest tests -x -q -m gpu > $D/pytest_stream.log 2>&1; tail -2 $D/pytest_stream.log
