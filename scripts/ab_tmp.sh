mkdir -p gpurun_out/s2ab
for i in 1 2; do
AB_TAG=split python scripts/ab_quick.py; ANKH_M2L_SPLIT=0 AB_TAG=nosplit python scripts/ab_quick.py
WORLD=8 python scripts/shard_step.py; ANKH_M2L_SPLIT=0 WORLD=8 python scripts/shard_step.py
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2ab/stream.csv python scripts/stream_trace.py > /dev/null 2>&1; echo ncu $?
