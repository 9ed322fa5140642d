"""Timeline of the streamed host path (ANKH_STREAM_TRACE=1) at a BASELINE config.

    python scripts/stream_trace.py [--config 3] [--chunks 8]
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
    ap.add_argument("--chunks", type=int, default=8)
    a = ap.parse_args()
    os.environ["ANKH_STREAM_CHUNKS"] = str(a.chunks)
    import torch

    import paper_2212_08284_b200 as ankh
    from paper_2212_08284_b200 import inputs

    pos, src, rb, cfg = inputs.make_config(a.config)
    L = cfg.orders[0] if a.config != 2 else 5
    hp, hs = torch.from_numpy(pos).pin_memory().numpy(), torch.from_numpy(src).pin_memory().numpy()
    plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), threads=0)
    for _ in range(3):
        plan.energy(hp, hs)
    t0 = time.perf_counter()
    for _ in range(10):
        plan.energy(hp, hs)
    print(f"untraced: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms per call", file=sys.stderr)
    os.environ["ANKH_STREAM_TRACE"] = "1"
    plan.energy(hp, hs)


if __name__ == "__main__":
    main()
