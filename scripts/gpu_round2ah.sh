# round-2 closing evidence: full GPU suite, bench lines, ncu captures (energy + forces kernels)
set -u
O=gpurun_out/r02ah; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -6 > $O/pytest_gpu.txt; tail -3 $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" >> $O/pytest_gpu.txt 2>&1; tail -1 $O/pytest_gpu.txt
bash scripts/run_final.sh r02ah
timeout 300 python scripts/forces_step.py --reps 3 > $O/forces_step.txt 2>&1; cat $O/forces_step.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/forces_launches.csv python scripts/forces_step.py --reps 1 > $O/forces_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -f -k regex:"k_m2l_local|k_p2p_force_half|k_l2p|k_force_out" -c 4 -o $O/forces_full python scripts/forces_step.py --reps 0 > $O/forces_ncu_full.log 2>&1
ls $O
