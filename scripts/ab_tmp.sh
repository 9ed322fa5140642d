mkdir -p gpurun_out/s2ab2
for r in 1 2; do for v in t32 t64 t128; do ANKH_B200_LIB=$PWD/paper_2212_08284_b200/variants/libankh_b200_bin_$v.so python scripts/p2p_ab.py; done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2ab2/stream.csv python scripts/stream_trace.py > /dev/null 2>&1; echo ncu $?
