for r in 1 2 3; do for v in t32 t64 t128; do ANKH_B200_LIB=$PWD/paper_2212_08284_b200/variants/libankh_b200_bin_$v.so python scripts/p2p_ab.py; done; done
