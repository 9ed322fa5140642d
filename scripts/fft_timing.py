"""ANKH-FFT engine vs the drop-in FMM engine at a BASELINE config: plan build,
device time per evaluation (inputs in HBM, CUDA-graph replay) and the
energies.

    python scripts/fft_timing.py [--config 3] [--order-equi L]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--order-equi", type=int, default=0)
    a = ap.parse_args()
    import torch

    import paper_2212_08284_b200 as ankh
    from paper_2212_08284_b200 import inputs

    pos, src, rb, cfg = inputs.make_config(a.config)
    L = cfg.orders[0] if a.config != 2 else 5
    Lu = a.order_equi or L
    dp, ds = torch.from_numpy(pos).cuda(), torch.from_numpy(src).cuda()
    for engine in ("fmm", "fft"):
        t0 = time.perf_counter()
        plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=Lu), engine=engine,
                         phase_timing=False)
        tb = time.perf_counter() - t0
        st = torch.cuda.Stream()
        for _ in range(3):
            rep = plan.energy_device(dp, ds, st.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10):
            plan.enqueue(dp, ds, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        rep = plan.energy_device(dp, ds, st.cuda_stream)
        print(f"{engine}: L_c={L} L_u={Lu} build {tb:.2f} s, {e0.elapsed_time(e1) / 10:.3f} ms per evaluation, "
              f"e_far {rep.e_far:.12g} e_periodic_far {rep.e_periodic_far:.12g} e_total {rep.e_total:.15g}",
              flush=True)
        plan.close()


if __name__ == "__main__":
    main()
