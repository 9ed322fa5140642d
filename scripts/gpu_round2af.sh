set -u
O=gpurun_out/r02ag; mkdir -p $O
V=$PWD/paper_2212_08284_b200/variants
timeout 300 python scripts/forces_step.py --reps 0 > $O/plain.txt 2>&1
for v in default r32b3 r24b4 r16b4 r16b5; do
  lib=""; [ $v != default ] && lib=$V/libankh_b200_$v.so
  ANKH_B200_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_m2l_local|k_p2p_force_half" -c 4 --csv --log-file $O/loc_$v.csv python scripts/forces_step.py --reps 0 > $O/loc_$v.log 2>&1
  echo $v; grep -E "k_m2l_local|force_half" $O/loc_$v.csv | awk -F'","' '{print substr($5,1,40), $(NF-2), $(NF)}'
done
ANKH_B200_LIB=$V/libankh_b200_r24b4.so timeout 900 python -m pytest tests/test_forces.py -q -m gpu -x -k "reference_energy or half_shell" 2>&1 | tail -3
