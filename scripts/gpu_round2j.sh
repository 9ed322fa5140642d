set -u
D=gpurun_out/r02j; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc $?"; tail -2 $D/smoke.log
for c in 8 16; do timeout 300 python scripts/stream_trace.py --config 3 --chunks $c > $D/trace_$c.log 2>&1; echo "trace $c rc $?"; done
cat $D/trace_8.log | tail -45
timeout 300 python scripts/stream_trace.py --config 3 --chunks 16 2>&1 | head -1
timeout 900 compute-sanitizer --tool memcheck --leak-check no python scripts/sanitize_case.py 0 > $D/memcheck.log 2>&1; echo "memcheck rc $?"; tail -8 $D/memcheck.log
