"""One streamed host-path evaluation (config 3) between cudaProfilerStart/Stop,
for an ncu launch list of the streamed path's kernels:

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \\
        python scripts/stream_ncu.py [--config 3] [--calls 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--calls", type=int, default=1)
    a = ap.parse_args()
    import torch

    import paper_2212_08284_b200 as ankh
    from paper_2212_08284_b200 import inputs

    pos, src, rb, cfg = inputs.make_config(a.config)
    L = cfg.orders[0] if a.config != 2 else 5
    hp, hs = torch.from_numpy(pos).pin_memory().numpy(), torch.from_numpy(src).pin_memory().numpy()
    plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), threads=0)
    for _ in range(3):
        plan.energy(hp, hs)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.calls):
        e = plan.energy(hp, hs).e_total
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("e_total", e)
    plan.close()


if __name__ == "__main__":
    main()
