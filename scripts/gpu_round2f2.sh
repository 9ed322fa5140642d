set -u
D=gpurun_out/r02h; mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc $?"; tail -1 $D/smoke.log
timeout 3000 python -m pytest tests -q -m gpu --durations=5 > $D/pytest.log 2>&1; echo "pytest rc $?"; tail -9 $D/pytest.log
bash scripts/run_final.sh r02h
