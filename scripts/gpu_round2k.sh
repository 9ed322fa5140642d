set -u
D=gpurun_out/r02k; mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc $?"; tail -1 $D/smoke.log
for c in 8 12 16; do timeout 300 python scripts/stream_trace.py --config 3 --chunks $c > $D/trace_$c.log 2>&1; echo "trace $c rc $?"; head -1 $D/trace_$c.log; done
cat $D/trace_8.log | tail -45
timeout 1500 python -m pytest tests -x -q -m gpu > $D/pytest.log 2>&1; echo "pytest rc $?"; tail -3 $D/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $D/bench.json 2> $D/bench.err; echo "bench rc $?"; python - $D/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "fixed", d["e2e_fixed_positions"]["value"]); print({k:round(v,4) for k,v in d["phases_ms"].items()})
PY
