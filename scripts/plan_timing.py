"""Plan-build stage times (ANKH_PLAN_TIMING=1 prints them on stderr).

    python scripts/plan_timing.py --config 3 [--config 4]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["ANKH_PLAN_TIMING"] = "1"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, action="append")
    a = ap.parse_args()
    import paper_2212_08284_b200 as ankh
    from paper_2212_08284_b200 import inputs

    for c in a.config or [3]:
        pos, src, rb, cfg = inputs.make_config(c)
        L = cfg.orders[0] if c != 2 else 5
        for rep in range(2):
            t0 = time.perf_counter()
            plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L), threads=0)
            r = plan.energy(pos, src)
            print(f"config {c} build+first eval {time.perf_counter() - t0:.3f} s  "
                  f"precompute {r.wall_times.get('precompute', 0.0):.3f} s", file=sys.stderr, flush=True)
            del plan


if __name__ == "__main__":
    main()
