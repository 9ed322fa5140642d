set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "stream" 2>&1 | tail -1
for g in 1 2 4; do for c in 16 32; do ANKH_STREAM_P2P_GROUP=$g timeout 300 python scripts/stream_trace.py --config 3 --chunks $c 2>&1 | head -1 | sed "s/^/group $g chunks $c: /"; done; done
