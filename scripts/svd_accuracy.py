"""M2L factor accuracy of the plan (GPU Jacobi, default) and of the host
Jacobi (ANKH_HOST_SVD=1) against LAPACK's rank-k truncation of the same dense
block: max |L^T R - C_k| / max |C| per (level, offset).

    python scripts/svd_accuracy.py [--order 5]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--order", type=int, default=5)
    a = ap.parse_args()
    import paper_2212_08284_b200 as ankh
    from oracle import ankh_oracle as ora

    L, rb = a.order, 10.0
    cfg = ankh.EwaldConfig(order_cheb=L, order_equi=L, depth=3)
    gpu = ankh.Plan(1500, rb, cfg)
    os.environ["ANKH_HOST_SVD"] = "1"
    host = ankh.Plan(1500, rb, cfg)
    del os.environ["ANKH_HOST_SVD"]
    worst = [0.0, 0.0]
    for level in (1, 2, 3):
        for off in [(2, 0, 0), (-3, 1, 2), (0, -2, 3), (3, 3, -2), (2, 2, 2), (3, 0, 0), (3, 3, 0), (2, 1, 1)]:
            c = ora.m2l_dense(L, rb / (1 << level), off, 0.01)
            u, s, vt = np.linalg.svd(c)
            errs = []
            for i, p in enumerate((gpu, host)):
                lm, rm = p.m2l_factors(level, off)
                k = lm.shape[0]
                ck = (u[:, :k] * s[:k]) @ vt[:k]
                e = np.abs(lm.T @ rm - ck).max() / np.abs(c).max()
                worst[i] = max(worst[i], e)
                errs.append(e)
            print(f"level {level} off {off} rank {k}: gpu {errs[0]:.2e} host {errs[1]:.2e}  "
                  f"sigma_k/sigma_0 {s[k - 1] / s[0]:.2e} next {s[k] / s[0]:.2e}")
    print(f"worst: gpu {worst[0]:.2e} host {worst[1]:.2e}")


if __name__ == "__main__":
    main()
