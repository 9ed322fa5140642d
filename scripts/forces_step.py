"""One plan, a few energy + forces evaluations of a BASELINE config (for ncu
captures of the forces kernels and their launch list).

    python scripts/forces_step.py [--config 3] [--reps 2]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--field", action="store_true", help="also time Plan.field (moment derivatives alone)")
    a = ap.parse_args()
    import numpy as np

    import paper_2212_08284_b200 as ankh
    from paper_2212_08284_b200 import inputs

    pos, src, rb, cfg = inputs.make_config(a.config)
    L = cfg.orders[0] if a.config != 2 else 5
    plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), phase_timing=False)
    rep, f = plan.forces(pos, src)
    t0 = time.perf_counter()
    for _ in range(a.reps):
        rep, f = plan.forces(pos, src)
    dt = (time.perf_counter() - t0) / max(1, a.reps)
    print(f"config {a.config}: energy + forces {dt * 1e3:.2f} ms per call (host buffers), e_total {rep.e_total:.17g}, "
          f"|F| max {np.abs(f).max():.6g}, sum F {f.sum(axis=0)}", flush=True)
    if a.field:
        plan.field(pos, src)
        t0 = time.perf_counter()
        for _ in range(max(1, a.reps)):
            e = plan.field(pos, src)
        dt = (time.perf_counter() - t0) / max(1, a.reps)
        print(f"config {a.config}: field evaluation {dt * 1e3:.2f} ms per call (host buffers), |E| max {np.abs(e).max():.6g}",
              flush=True)
    plan.close()


if __name__ == "__main__":
    main()
