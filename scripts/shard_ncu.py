"""One shard evaluation (world W, rank R, loopback exchange) between
cudaProfilerStart/Stop, for an ncu launch list of a shard's kernels:

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \\
        python scripts/shard_ncu.py [--world 8] [--rank 0] [--config 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--config", type=int, default=3)
    a = ap.parse_args()
    import torch

    import paper_2212_08284_b200 as ankh
    from paper_2212_08284_b200 import inputs

    pos, src, rb, cfg = inputs.make_config(a.config)
    L = cfg.orders[0] if a.config != 2 else 5
    dp, ds = torch.from_numpy(pos).cuda(), torch.from_numpy(src).cuda()
    plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), rank=a.rank, world=a.world,
                     phase_timing=False)
    if a.world > 1:
        plan.attach_loopback()
    st = torch.cuda.Stream()
    for _ in range(3):
        plan.enqueue(dp, ds, st.cuda_stream)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    plan.enqueue(dp, ds, st.cuda_stream)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    plan.close()


if __name__ == "__main__":
    main()
