"""Cold one-shot call breakdown: plan construction, first evaluation, close.

    python scripts/cold_call.py [--config 3]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    a = ap.parse_args()
    import torch

    import paper_2212_08284_b200 as ankh
    from paper_2212_08284_b200 import inputs

    pos, src, rb, cfg = inputs.make_config(a.config)
    L = cfg.orders[0] if a.config != 2 else 5
    hp, hs = torch.from_numpy(pos).pin_memory().numpy(), torch.from_numpy(src).pin_memory().numpy()
    ec = ankh.EwaldConfig(order_cheb=L, order_equi=L)
    keep = ankh.Plan(pos.shape[0], rb, ec, threads=0, phase_timing=False)  # as bench.py: a live plan
    keep.energy(hp, hs)
    if os.environ.get("COLD_BOUND"):
        keep.set_positions(hp)
        keep.energy_sources(hs)
    for mode in ("0", "1", "0", "1"):
        os.environ["ANKH_STREAM_INPUT"] = mode
        t0 = time.perf_counter()
        p = ankh.Plan(pos.shape[0], rb, ec, threads=0, phase_timing=False)
        t1 = time.perf_counter()
        p.energy(hp, hs)
        t2 = time.perf_counter()
        p.energy(hp, hs)
        t3 = time.perf_counter()
        p.close()
        t4 = time.perf_counter()
        print(f"stream={mode}: build {1e3 * (t1 - t0):.1f} ms, first eval {1e3 * (t2 - t1):.1f} ms, "
              f"second {1e3 * (t3 - t2):.1f} ms, close {1e3 * (t4 - t3):.1f} ms", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
