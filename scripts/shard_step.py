"""One shard's evaluation (config 3 by default, rank 0 of WORLD, loopback
exchange) repeated STEPS times on one GPU -- the command to put under ncu for
a shard's kernel list:  WORLD=8 python scripts/shard_step.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2212_08284_b200 as ankh  # noqa: E402
from paper_2212_08284_b200 import inputs  # noqa: E402

ci = int(os.environ.get("AB_CONFIG", "3"))
world = int(os.environ.get("WORLD", "8"))
rank = int(os.environ.get("RANK_", "0"))
steps = int(os.environ.get("STEPS", "4"))
pos, src, rb, cfg = inputs.make_config(ci)
L = cfg.orders[0] if ci != 2 else 5
plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), rank=rank, world=world,
                 phase_timing=False)
if world > 1:
    plan.attach_loopback()
dp, ds = torch.from_numpy(pos).cuda(), torch.from_numpy(src).cuda()
st = torch.cuda.Stream()
for _ in range(steps):
    plan.enqueue(dp, ds, st.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(10):
    plan.enqueue(dp, ds, st.cuda_stream)
e1.record(st)
torch.cuda.synchronize()
print(f"world {world} rank {rank}: {e0.elapsed_time(e1) / 10:.3f} ms per evaluation", flush=True)
plan.close()
