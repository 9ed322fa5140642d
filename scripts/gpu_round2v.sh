set -u
D=gpurun_out/r02v; mkdir -p $D
timeout 900 python -m pytest tests/test_fft_engine.py -q -m gpu -x > $D/pytest_fft.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed|Error|assert" $D/pytest_fft.log | head -20
timeout 600 python scripts/fft_timing.py --config 0 2>&1 | tail -3
timeout 900 python scripts/fft_timing.py --config 3 2>&1 | tail -3
