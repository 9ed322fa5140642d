set -u
O=gpurun_out/r02ae; mkdir -p $O
timeout 1200 python -m pytest tests/test_forces.py -q -m gpu -x 2>&1 | tail -8 > $O/pytest_forces.txt
tail -4 $O/pytest_forces.txt
timeout 300 python scripts/forces_step.py --reps 3 > $O/forces_step.txt 2>&1; cat $O/forces_step.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/forces_launches.csv python scripts/forces_step.py --reps 1 > $O/forces_ncu.log 2>&1
grep -E "k_p2p_force|k_m2l_local|k_force_out|k_l2p" $O/forces_launches.csv | awk -F'","' '{print substr($5,1,60), $(NF)}' | tail -4
