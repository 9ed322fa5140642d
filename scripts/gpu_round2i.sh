set -u
D=gpurun_out/r02i; mkdir -p $D
timeout 1800 python -m pytest tests -q -m gpu -x > $D/pytest.log 2>&1; tail -3 $D/pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $D/bench.json 2> $D/bench.err; python - $D/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"]); print({k:round(v,4) for k,v in d["phases_ms"].items()})
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_forces.csv python scripts/forces_step.py --config 3 --reps 1 > $D/ncu_forces.log 2>&1; echo "ncu $?"
python - $D/launches_forces.csv <<'PY'
import csv,sys,collections,re
rows=[r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[1:]:
    m=re.search(r"(k_\w+)",r[ki]); k=m.group(1) if m else r[ki][:40]
    agg[k][0]+=1; agg[k][1]+=float(r[vi].replace(',',''))
for k,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:20]: print(f"{k:30s} {c:5d} {t/1e6:9.3f} ms")
PY
ANKH_B200_LIB=$PWD/paper_2212_08284_b200/variants/libankh_b200_checked.so timeout 2400 python -m pytest tests -q -m gpu > $D/pytest_checked.log 2>&1; tail -3 $D/pytest_checked.log; grep -c DASSERT $D/pytest_checked.log
