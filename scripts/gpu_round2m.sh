set -u
D=gpurun_out/r02m; mkdir -p $D
for v in "" "ANKH_P2P_STATIC=1"; do
  env $v timeout 300 python scripts/stream_trace.py --config 3 --chunks 8 > $D/trace_$v.log 2>&1; echo "[$v] $(head -1 $D/trace_$v.log)"
done
for c in 6 12 16; do timeout 300 python scripts/stream_trace.py --config 3 --chunks $c 2>&1 | head -1 | sed "s/^/chunks $c: /"; done
ANKH_STREAM_FIRST=1 timeout 300 python scripts/stream_trace.py --config 3 --chunks 8 2>&1 | head -1 | sed "s/^/first=1: /"
ANKH_STREAM_FIRST=0.25 timeout 300 python scripts/stream_trace.py --config 3 --chunks 8 2>&1 | head -1 | sed "s/^/first=0.25: /"
tail -42 $D/trace_.log
ANKH_STREAM_NO_GRAPH=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/stream_launches.csv python scripts/stream_ncu.py > $D/ncu_stream.log 2>&1; echo "ncu rc $?"
python - $D/stream_launches.csv <<'PY'
import csv,sys,re
rows=[r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
tot={}
for r in rows[1:]:
    m=re.search(r"(k_\w+)",r[ki]); k=m.group(1) if m else r[ki][:40]
    tot[k]=tot.get(k,0)+float(r[vi].replace(',',''))/1e3
print({k:round(v,1) for k,v in tot.items()})
PY
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "higher or csr" > $D/pytest_hi.log 2>&1; echo "pytest rc $?"; tail -5 $D/pytest_hi.log
