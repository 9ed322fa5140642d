set -u
D=gpurun_out/r02b; mkdir -p $D
timeout 1500 python -m pytest tests -x -q -m gpu -k "push_group or shard or loopback or nccl or inprocess or sliced" > $D/pytest_shard.log 2>&1; tail -3 $D/pytest_shard.log
AB_CONFIG=3 timeout 600 python scripts/shard_timing.py > $D/shard_timing_halo.txt 2>&1; tail -8 $D/shard_timing_halo.txt
ANKH_SHARD_ALLGATHER=1 AB_CONFIG=3 timeout 600 python scripts/shard_timing.py > $D/shard_timing_allgather.txt 2>&1; tail -8 $D/shard_timing_allgather.txt
ANKH_STREAM_TRACE=1 timeout 300 python scripts/stream_trace.py > $D/stream_trace.txt 2>&1; tail -40 $D/stream_trace.txt
