set -u
D=gpurun_out/r02n; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "stream or bound" > $D/pytest.log 2>&1; echo "pytest rc $?"; tail -3 $D/pytest.log
for c in 8 12 16 24 32; do timeout 300 python scripts/stream_trace.py --config 3 --chunks $c 2>&1 | head -1 | sed "s/^/chunks $c: /"; done
ANKH_P2P_STRIDE=1 timeout 300 python scripts/stream_trace.py --config 3 --chunks 16 2>&1 | head -1 | sed "s/^/stride 16: /"
ANKH_STREAM_FIRST=1 timeout 300 python scripts/stream_trace.py --config 3 --chunks 16 2>&1 | head -1 | sed "s/^/first=1 16: /"
timeout 300 python scripts/stream_trace.py --config 3 --chunks 16 > $D/trace16.log 2>&1; tail -75 $D/trace16.log | grep -E "copy positions|binned|CSR|sorted|gather 0|p2p|far chain|finalize"
ANKH_STREAM_NO_GRAPH=1 ANKH_STREAM_CHUNKS=16 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/stream_launches.csv python scripts/stream_ncu.py --calls 1 > $D/ncu_stream.log 2>&1; echo "ncu rc $?"
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
