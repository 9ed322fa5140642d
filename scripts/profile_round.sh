# ncu evidence for profiles/<round>/ (one GPU; run each capture only after the
# plain bench has exited 0).  Usage: bash scripts/profile_round.sh <outdir-name>
# then, here: python scripts/profile_summary.py gpurun_out/<outdir-name> profiles/<round>
set -u
D=gpurun_out/${1:-prof}
mkdir -p $D
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > $D/bench_plain.json 2> $D/bench_plain.err || { echo "bench failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $D/launches_c3.csv $B > $D/ncu_launch.log 2>&1; echo "launch list $?"
F="ncu --set full --clock-control none --import-source on -f"
# steps per evaluation: k_p2p x1, k_m2l x7 rank classes, 9 small launches
# (init, bin, scan, scatter, leaf gather, P2M, the one-launch M2M chain, periodic, finalize)
timeout 900 $F -k regex:k_p2p -s 3 -c 1 -o $D/p2p_full $B > $D/ncu_p2p.log 2>&1; echo "p2p $?"
timeout 900 $F -k regex:k_m2l -s 21 -c 7 -o $D/m2l_full $B > $D/ncu_m2l.log 2>&1; echo "m2l $?"
timeout 900 $F -k "regex:k_init_result|k_bin|k_scan|k_scatter|k_leaf_gather|k_p2m|k_m2m|k_periodic_eval|k_finalize" \
  -s 27 -c 9 -o $D/small_full $B > $D/ncu_small.log 2>&1; echo "small $?"
AB_CONFIG=3 timeout 600 python scripts/shard_timing.py > $D/shard_timing.txt 2>&1; tail -4 $D/shard_timing.txt
