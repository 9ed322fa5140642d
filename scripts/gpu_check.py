"""Ad-hoc GPU parity/timing check (developer script; tests/ hold the real gates)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch
import ref as R
import paper_2212_08284_b200 as ankh
from paper_2212_08284_b200 import inputs

def cmp(name, pos, src, rb, **kw):
    cfg = ankh.EwaldConfig(**kw)
    try:
        g = ankh.fmm_energy(ankh.ParticleSystem(pos, src, rb), cfg)
    except Exception as e:
        print(name, "GPU ERROR", type(e).__name__, e); return
    t = time.time(); r = R.fmm_energy(pos, src, rb, threads=os.cpu_count(), **kw); tr = time.time() - t
    out = [f"{name:28s} ref {tr:6.2f}s"]
    for k in ["e_total", "e_near", "e_far", "e_self", "e_periodic_far"]:
        a, b = getattr(g, k), r[k]
        out.append(f"{k}={abs(a-b)/max(abs(b),1e-300):.1e}")
    print(" ".join(out), f"e_total={g.e_total:.12g}", flush=True)

for seed, (n, rb, kw) in enumerate([
    (300, 5.0, dict(order_cheb=4, order_equi=4, depth=2, p=15)),
    (300, 5.0, dict(order_cheb=3, order_equi=3, depth=2, p=0)),
    (500, 7.0, dict(order_cheb=5, order_equi=5, depth=1, p=2)),
    (500, 7.0, dict(order_cheb=6, order_equi=6, depth=2, p=15)),
    (2000, 9.0, dict(order_cheb=4, order_equi=4, depth=3, p=15)),
    (64, 3.0, dict(order_cheb=2, order_equi=2, depth=1, p=0)),
]):
    pos, src = inputs.random_system(n, rb, seed=seed, multipoles=True)
    cmp(f"rand n={n} {kw}", pos, src, rb, **kw)
    pos, src = inputs.random_system(n, rb, seed=seed, multipoles=False)
    cmp(f"rand-q n={n}", pos, src, rb, **kw)

for ci, L in [(0, 4), (1, 4), (2, 5)]:
    pos, src, rb, c = inputs.make_config(ci)
    cmp(f"{c.name} L={L}", pos, src, rb, order_cheb=L, order_equi=L)

# timing
for ci, L in [(1, 4), (2, 5), (3, 5)]:
    pos, src, rb, c = inputs.make_config(ci)
    plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), phase_timing=True)
    dp = torch.from_numpy(pos).cuda(); ds = torch.from_numpy(src).cuda()
    rep = plan.energy_device(dp, ds)
    print(c.name, "plan info", plan.info(), "precompute", rep.wall_times["precompute"])
    for _ in range(3): rep = plan.energy_device(dp, ds)
    print(c.name, {k: round(v*1e3, 3) for k, v in rep.wall_times.items()}, "ms", "pairs", rep.near_pairs, "e", rep.e_total)
    plan2 = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), phase_timing=False)
    for _ in range(3): plan2.energy_device(dp, ds)
    torch.cuda.synchronize()
    t = time.perf_counter(); K = 10
    for _ in range(K): plan2.enqueue(dp, ds)
    plan2.result(); torch.cuda.synchronize()
    print(c.name, "ms/eval", (time.perf_counter() - t) / K * 1e3, flush=True)
