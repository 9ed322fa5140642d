"""A/B timing of the phases on config 3 for the library selected by ANKH_B200_LIB."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2212_08284_b200 as ankh
from paper_2212_08284_b200 import inputs
ci = int(os.environ.get("AB_CONFIG", "3"))
pos, src, rb, cfg = inputs.make_config(ci)
L = cfg.orders[0] if ci != 2 else 5
plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), phase_timing=True)
dp, ds = torch.from_numpy(pos).cuda(), torch.from_numpy(src).cuda()
ph = {}
for i in range(6):
    r = plan.energy_device(dp, ds)
    if i < 2: continue
    for k, v in r.wall_times.items(): ph.setdefault(k, []).append(v * 1e3)
print(os.path.basename(ankh.LIB_PATH), "c%d" % ci, " ".join(f"{k}={statistics.median(v):.3f}" for k, v in ph.items() if k != "total"), "e=%.12g" % r.e_total, flush=True)
