# k_m2l_local staging A/B: cp.async (default) against bulk row copies on mbarriers;
# forces through the streamed host path
set -u
O=gpurun_out/r02aj; mkdir -p $O
V=$PWD/paper_2212_08284_b200/variants
timeout 900 python -m pytest tests/test_forces.py -q -m gpu -x 2>&1 | tail -3
timeout 300 python scripts/forces_step.py --reps 3 > $O/plain.txt 2>&1; cat $O/plain.txt
ANKH_B200_LIB=$V/libankh_b200_bulk.so timeout 300 python scripts/forces_step.py --reps 1 > $O/plain_bulk.txt 2>&1; tail -2 $O/plain_bulk.txt
for v in default bulk; do
  lib=""; [ $v != default ] && lib=$V/libankh_b200_$v.so
  ANKH_B200_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_m2l_local" -c 2 --csv --log-file $O/loc_$v.csv python scripts/forces_step.py --reps 0 > $O/loc_$v.log 2>&1
  echo $v; grep -E "k_m2l_local" $O/loc_$v.csv | awk -F'","' '{print substr($5,1,40), $(NF-2), $(NF)}'
done
ANKH_B200_LIB=$V/libankh_b200_bulk.so timeout 900 python -m pytest tests/test_forces.py -q -m gpu -x -k "reference_energy or at_scale" 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], 'forces', d['forces_e2e'])"
