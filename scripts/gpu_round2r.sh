set -u
D=gpurun_out/r02r; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "csr or golden_small or stream or bound or headline" > $D/pytest.log 2>&1; echo "pytest rc $?"; tail -2 $D/pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_scan --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep k_scan | tail -3
