# k_m2l_local GEMM 1: batched 16-B partner loads (default) against one 8-B load per k-step
set -u
O=gpurun_out/r02ap; mkdir -p $O
V=$PWD/paper_2212_08284_b200/variants
timeout 300 python scripts/forces_step.py --reps 1 > $O/plain.txt 2>&1; cat $O/plain.txt
for v in default nobatch; do
  lib=""; [ $v != default ] && lib=$V/libankh_b200_$v.so
  ANKH_B200_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_m2l_local" -c 2 --csv --log-file $O/loc_$v.csv python scripts/forces_step.py --reps 0 > $O/loc_$v.log 2>&1
  echo $v; grep -E "k_m2l_local" $O/loc_$v.csv | awk -F'","' '{print substr($5,1,40), $(NF-2), $(NF)}'
done
timeout 1500 python -m pytest tests/test_forces.py tests/test_dropin_cpp.py -q -m gpu -x 2>&1 | tail -3 | tee $O/pytest_forces.txt
