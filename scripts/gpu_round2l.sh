set -u
D=gpurun_out/r02l; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "higher or golden_high or golden_small or stream" > $D/pytest_hi.log 2>&1; echo "pytest rc $?"; tail -5 $D/pytest_hi.log
timeout 300 python scripts/stream_trace.py --config 3 --chunks 8 > $D/trace_g8.log 2>&1; head -1 $D/trace_g8.log
ANKH_STREAM_NO_GRAPH=1 timeout 300 python scripts/stream_trace.py --config 3 --chunks 8 > $D/trace_ng8.log 2>&1; head -1 $D/trace_ng8.log
ANKH_STREAM_NO_GRAPH=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/stream_launches.csv python scripts/stream_ncu.py > $D/ncu_stream.log 2>&1; echo "ncu rc $?"
python - $D/stream_launches.csv <<'PY'
import csv,sys,re
rows=[r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]:
    m=re.search(r"(k_\w+(<[^>]*>)?)",r[ki]); k=m.group(1) if m else r[ki][:40]
    print(f"{k:32s} {float(r[vi].replace(',',''))/1e3:9.1f} us")
PY
timeout 600 python bench.py --no-cpu-baseline > $D/bench.json 2> $D/bench.err; echo "bench rc $?"; python - $D/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "fixed", d["e2e_fixed_positions"]["value"])
PY
