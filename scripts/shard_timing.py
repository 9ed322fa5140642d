"""Per-rank device time of one shard at world = 1, 2, 4, 8 on ONE GPU.
Estimates strong scaling of config 3 without a multi-GPU box:  T1 / (W * T_W)
is an upper bound on the scaling efficiency.

Two modes per world size:
  * serial   -- the phase API (phase 1 = binning..own P2M, phase 2 = the rest),
                back to back on one stream, no exchange;
  * overlap  -- the production schedule: the plan's CUDA graph with P2P
                concurrent with the far chain, and a loopback exchange
                (ankh_plan_attach_loopback_v1: the exchange's bytes -- the
                all-gathered exchange level and the deep-level M2L halos --
                land by device copies, the all-reduce is the identity).  The
                NVLink time of the real exchange is not included; it is
                printed beside as bytes received per rank.
"""
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


def timed(fn, st, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


base = {}
for world in (1, 2, 4, 8):
    for mode in ("serial", "overlap"):
        times = []
        for rank in sorted({0, world - 1}):
            plan = ankh.Plan(pos.shape[0], rb, ec, rank=rank, world=world, phase_timing=False)
            st = torch.cuda.Stream()
            if mode == "serial":
                def fn():
                    plan.enqueue_phase(1, dp, ds, st.cuda_stream)
                    plan.enqueue_phase(2, dp, ds, st.cuda_stream)
            else:
                if world > 1:
                    plan.attach_loopback()

                def fn():
                    plan.enqueue(dp, ds, st.cuda_stream)
            times.append(timed(fn, st))
            info = plan.info()
            plan.close()
        t = max(times)
        base.setdefault(mode, t)
        import ctypes
        rv, sd = ctypes.c_size_t(), ctypes.c_size_t()
        halo = 0 if os.environ.get("ANKH_SHARD_ALLGATHER") else 1
        ankh.lib().ankh_shard_exchange_bytes_v1(info["depth"], 1, L, 0, world, halo, ctypes.byref(rv),
                                                ctypes.byref(sd))
        leaf_bytes = rv.value
        print(f"world {world} {mode:7s}: per-rank {t:.3f} ms (ranks {sorted({0, world - 1})}: "
              f"{', '.join(f'{x:.3f}' for x in times)}), efficiency bound {base[mode] / (world * t):.2f}"
              f"{'' if mode == 'serial' else f', exchange receives {leaf_bytes / 1e6:.1f} MB per rank'}",
              flush=True)
