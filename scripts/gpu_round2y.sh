set -u
for mb in 0 40 60 80; do
  if [ $mb = 0 ]; then timeout 300 python scripts/stream_trace.py --config 3 --chunks 16 2>&1 | grep -E "untraced" | head -1 | sed "s/^/persist none: /";
  else ANKH_L2_PERSIST=$mb timeout 300 python scripts/stream_trace.py --config 3 --chunks 16 2>&1 | grep -E "untraced|L2 persist" | head -2 | sed "s/^/persist $mb: /"; fi
done
