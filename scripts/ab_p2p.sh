mkdir -p gpurun_out/ab2
V=$PWD/paper_2212_08284_b200/variants
run() { ANKH_B200_LIB=$2 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab2/$1.json 2>gpurun_out/ab2/$1.err; }
for i in 1 2; do
  run def$i ""
  run static$i $V/libankh_b200_p2p_static.so
  run p4_$i $V/libankh_b200_p2p_piece4.so
  run p16_$i $V/libankh_b200_p2p_piece16.so
done
python scripts/p2p_clocks.py > gpurun_out/ab2/clk.txt 2>&1
timeout 1000 python -m pytest tests -x -q -m gpu > gpurun_out/ab2/pytest.log 2>&1; tail -3 gpurun_out/ab2/pytest.log
