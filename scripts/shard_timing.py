"""Per-rank device time of one shard at world = 1, 2, 4, 8 on ONE GPU (rank
0's share of the work through the phase API; the exchange itself -- an NCCL
all-gather and all-reduce -- is not included).  Estimates strong scaling of
config 3 without a multi-GPU box:  T1 / (W * T_W) is an upper bound on the
scaling efficiency."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2212_08284_b200 as ankh  # noqa: E402
from paper_2212_08284_b200 import inputs  # noqa: E402

ci = int(os.environ.get("AB_CONFIG", "3"))
pos, src, rb, cfg = inputs.make_config(ci)
L = cfg.orders[0] if ci != 2 else 5
ec = ankh.EwaldConfig(order_cheb=L, order_equi=L)
dp, ds = torch.from_numpy(pos).cuda(), torch.from_numpy(src).cuda()
base = None
for world in (1, 2, 4, 8):
    times = []
    for rank in sorted({0, world - 1}):
        plan = ankh.Plan(pos.shape[0], rb, ec, rank=rank, world=world, phase_timing=False)
        st = torch.cuda.Stream()
        for _ in range(3):
            plan.enqueue_phase(1, dp, ds, st.cuda_stream)
            plan.enqueue_phase(2, dp, ds, st.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(st)
        for _ in range(reps):
            plan.enqueue_phase(1, dp, ds, st.cuda_stream)
            plan.enqueue_phase(2, dp, ds, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / reps)
        plan.close()
    t = max(times)
    base = base or t
    print(f"world {world}: per-rank {t:.3f} ms (ranks {sorted({0, world - 1})}: "
          f"{', '.join(f'{x:.3f}' for x in times)}), efficiency bound {base / (world * t):.2f}", flush=True)
