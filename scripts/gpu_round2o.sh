set -u
D=gpurun_out/r02o; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "stream or bound" > $D/pytest.log 2>&1; echo "pytest rc $?"; tail -1 $D/pytest.log
for c in 12 16 24; do timeout 300 python scripts/stream_trace.py --config 3 --chunks $c 2>&1 | head -1 | sed "s/^/chunks $c: /"; done
timeout 600 python bench.py --no-cpu-baseline > $D/bench.json 2> $D/bench.err; echo "bench rc $?"; python - $D/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "fixed", d["e2e_fixed_positions"]["value"], "cold", d["e2e_including_precompute"]["value"])
print({k:round(v,4) for k,v in d["phases_ms"].items()})
PY
