"""Quick A/B of one build at config 3: device-resident evaluation (CUDA
graph, CUDA events) and the streamed host path (wall clock), both per call.
Environment switches (e.g. ANKH_NO_PRIORITY=1) are read at plan creation."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2212_08284_b200 as ankh  # noqa: E402
from paper_2212_08284_b200 import inputs  # noqa: E402

ci = int(os.environ.get("AB_CONFIG", "3"))
pos, src, rb, cfg = inputs.make_config(ci)
L = cfg.orders[0] if ci != 2 else 5
plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), phase_timing=False)
dp, ds = torch.from_numpy(pos).cuda(), torch.from_numpy(src).cuda()
st = torch.cuda.Stream()
for _ in range(4):
    plan.enqueue(dp, ds, st.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(20):
    plan.enqueue(dp, ds, st.cuda_stream)
e1.record(st)
torch.cuda.synchronize()
dev = e0.elapsed_time(e1) / 20
e_dev = plan.result().e_total
hp, hs = torch.from_numpy(pos).pin_memory().numpy(), torch.from_numpy(src).pin_memory().numpy()
for _ in range(3):
    plan.energy(hp, hs)
t0 = time.perf_counter()
for _ in range(20):
    e_host = plan.energy(hp, hs).e_total
host = (time.perf_counter() - t0) / 20 * 1e3
print(f"{os.environ.get('AB_TAG', '')}: device {dev:.3f} ms ({1e3 / dev:.1f}/s), host e2e {host:.3f} ms "
      f"({1e3 / host:.1f}/s), e_total {e_dev:.15g} / {e_host:.15g}", flush=True)
plan.close()
