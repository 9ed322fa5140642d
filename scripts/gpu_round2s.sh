set -u
D=gpurun_out/r02s; mkdir -p $D
for w in 1 8; do
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/shard_w$w.csv python scripts/shard_ncu.py --world $w > $D/ncu_w$w.log 2>&1; echo "ncu w$w rc $?"
python - $D/shard_w$w.csv <<'PY'
import csv,sys,re
rows=[r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
tot=0
for r in rows[1:]:
    m=re.search(r"(k_\w+(<[^>]*>)?)",r[ki]); k=m.group(1) if m else r[ki][:40]
    v=float(r[vi].replace(',',''))/1e3; tot+=v
    print(f"  {k:32s} {v:9.1f} us")
print("  total", round(tot,1))
PY
done
