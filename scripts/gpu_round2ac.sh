set -u
O=gpurun_out/r02ac; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_m2l_local|k_p2p_force_half" -c 2 -o $O/forces_full python scripts/forces_step.py --reps 0 > $O/forces_ncu_full.log 2>&1
tail -3 $O/forces_ncu_full.log
ls -la $O
