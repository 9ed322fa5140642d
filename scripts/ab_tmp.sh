for r in 1 2; do for v in p2m_novec p2m_vec; do ANKH_B200_LIB=$PWD/paper_2212_08284_b200/variants/libankh_b200_$v.so python scripts/p2p_ab.py; done; done
for v in p2m_novec p2m_vec; do ANKH_B200_LIB=$PWD/paper_2212_08284_b200/variants/libankh_b200_$v.so AB_CONFIG=1 python scripts/p2p_ab.py; done
