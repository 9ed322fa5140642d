"""Small evaluations for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): BASELINE configs 0 and 1 through the one-shot drop-in, the plan
device path (plain launches, graph capture, replay) and the bound-positions
path, plus a phase-timed plan.  Usage:
    compute-sanitizer --tool memcheck python scripts/sanitize_case.py [configs...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2212_08284_b200 as ankh  # noqa: E402
from paper_2212_08284_b200 import inputs  # noqa: E402


def main():
    import torch

    configs = [int(c) for c in sys.argv[1:]] or [0, 1]
    for c in configs:
        pos, src, rb, cfg = inputs.make_config(c)
        L = cfg.orders[0]
        ec = ankh.EwaldConfig(order_cheb=L, order_equi=L)
        e1 = ankh.fmm_energy(ankh.ParticleSystem(pos, src, rb), ec).e_total
        plan = ankh.Plan(pos.shape[0], rb, ec, phase_timing=False)
        dp, ds = torch.from_numpy(pos).cuda(), torch.from_numpy(src).cuda()
        e2 = [plan.energy_device(dp, ds).e_total for _ in range(3)]
        plan.set_positions(pos)
        e3 = [plan.energy_sources(src).e_total for _ in range(3)]
        plan.close()
        timed = ankh.Plan(pos.shape[0], rb, ec, phase_timing=True)
        e4 = timed.energy(pos, src).e_total
        timed.close()
        vals = [e1] + e2 + e3 + [e4]
        spread = max(abs(v - e1) for v in vals) / abs(e1)
        print(f"config {c}: e_total {e1:.17g}, spread over paths {spread:.2e}", flush=True)
        assert spread < 1e-12, vals


if __name__ == "__main__":
    main()
