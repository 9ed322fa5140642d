# pytest -m gpu + a bench line without the CPU baseline (outputs in gpurun_out/$1)
set -u
D=gpurun_out/${1:-quick}; mkdir -p $D
timeout 1500 python -m pytest tests -x -q -m gpu > $D/pytest.log 2>&1; tail -3 $D/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $D/bench.json 2> $D/bench.err; python - $D/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "fixed", d["e2e_fixed_positions"]["value"])
print({k:(round(v["ms"],4), round(v.get("frac") or 0,3)) for k,v in d["phase_rooflines"].items()})
print("clocks", d["clocks"])
PY
ANKH_STREAM_TRACE=1 timeout 300 python scripts/stream_trace.py > $D/stream_trace.txt 2>&1; grep -E "untraced|copy positions|sorted|chunk 7|far chain|finalize" $D/stream_trace.txt
