"""Per-CTA phase profile of the near-field kernel (debug build, ANKH_P2P_CLOCKS).

    make -C paper_2212_08284_b200/csrc variants
    python scripts/p2p_clocks.py [--config 3]

Runs one evaluation through the `p2p_clocks` variant library and reports, in
SM clocks averaged over the CTAs (target leaves), the CTA lifetime split into:
setup (segment table), staging of the first source chunk, the fastest warp's
pair loop, the extra time until the slowest warp finishes (the idle share the
final barrier exposes), and the block reduction.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VAR = os.path.join(ROOT, "paper_2212_08284_b200", "variants", "libankh_b200_p2p_clocks.so")
os.environ.setdefault("ANKH_B200_LIB", VAR)
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    a = ap.parse_args()
    import paper_2212_08284_b200 as ankh
    from paper_2212_08284_b200 import inputs

    pos, src, rb, cfg = inputs.make_config(a.config)
    L = cfg.orders[0] if a.config != 2 else 5
    plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), threads=0)
    rep = plan.energy(pos, src)
    lib = ctypes.CDLL(os.environ["ANKH_B200_LIB"])
    nl = 8 ** rep.depth
    nl = min(nl, 1 << 17)
    buf = np.zeros(nl * 6, dtype=np.int64)
    if lib.ankh_debug_p2p_clocks_v1(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.size)):
        raise SystemExit("clock copy failed")
    c = buf.reshape(nl, 6).astype(np.float64)
    names = ["setup", "stage", "warp_min", "warp_spread", "reduce"]
    life = c[:, :5].sum(1)
    print(f"leaves {nl}  mean na {c[:, 5].mean():.2f}  mean CTA lifetime {life.mean():.0f} clk")
    for k, nm in enumerate(names):
        v = c[:, k]
        print(f"  {nm:12s} mean {v.mean():9.0f} clk  p50 {np.median(v):9.0f}  p99 {np.percentile(v, 99):9.0f}"
              f"  share {v.sum() / life.sum():6.3f}")
    # idle warp-time inside the CTA: warps finished early wait at the barrier
    print(f"  warp-spread / (warp_min + spread) = {(c[:, 3] / (c[:, 2] + c[:, 3])).mean():.3f}")
    by = {}
    for row in c:
        by.setdefault(int(row[5]), []).append(row)
    print("  na  count  lifetime  spread/compute")
    for na in sorted(by):
        r = np.array(by[na])
        if len(r) < nl // 200:
            continue
        print(f"  {na:3d} {len(r):6d} {r[:, :5].sum(1).mean():9.0f}  {(r[:, 3] / (r[:, 2] + r[:, 3])).mean():.3f}")


if __name__ == "__main__":
    main()
