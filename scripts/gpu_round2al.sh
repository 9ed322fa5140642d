set -u
O=gpurun_out/r02al; mkdir -p $O
timeout 1500 python -m pytest tests/test_forces.py tests/test_dropin_cpp.py -q -m gpu -x 2>&1 | tail -4 | tee $O/pytest_forces.txt
timeout 300 python scripts/forces_step.py --reps 3 --field > $O/field.txt 2>&1; cat $O/field.txt
ANKH_FORCE_FULL_STENCIL=1 timeout 300 python scripts/forces_step.py --reps 3 > $O/full.txt 2>&1; cat $O/full.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_p2p_force" -c 6 --csv --log-file $O/field_launches.csv python scripts/forces_step.py --reps 0 --field > $O/field_ncu.log 2>&1
grep -E "k_p2p_force" $O/field_launches.csv | awk -F'","' '{print substr($5,1,70), $(NF)}'
