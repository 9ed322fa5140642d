set -u
D=gpurun_out/r02u; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "csr or stream" > $D/pytest.log 2>&1; echo "pytest rc $?"; tail -2 $D/pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/forces_launches.csv python scripts/forces_step.py --config 3 --reps 1 > $D/ncu_forces.log 2>&1; echo "ncu rc $?"
python - $D/forces_launches.csv <<'PY'
import csv,sys,re,collections
rows=[r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[1:]:
    m=re.search(r"(k_\w+)",r[ki]); k=m.group(1) if m else r[ki][:40]
    agg[k][0]+=1; agg[k][1]+=float(r[vi].replace(',',''))
for k,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:16]: print(f"{k:30s} {c:5d} {t/1e6:9.3f} ms")
PY
