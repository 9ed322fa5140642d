"""Forces diagnostics: GPU forces vs central differences of the GPU's own
energy and of the reference's, per case (prints per-particle errors)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import paper_2212_08284_b200 as ankh  # noqa: E402
from paper_2212_08284_b200 import inputs  # noqa: E402
import ref as R  # noqa: E402


def run(n, rb, seed, mp, kw, h=1e-5, npart=4):
    pos, src = inputs.random_system(n, rb, seed=seed, multipoles=mp)
    cfg = ankh.EwaldConfig(**kw)
    plan = ankh.Plan(n, rb, cfg)
    rep, f = plan.forces(pos, src)
    depth = kw["depth"]
    side = 2 * rb / (1 << depth)
    u = (pos + rb) / side
    fr = u - np.floor(u)
    cand = np.where(((fr * side > 50 * h) & ((1 - fr) * side > 50 * h)).all(axis=1))[0]
    idx = cand[np.linspace(0, len(cand) - 1, npart).astype(int)]
    for i in idx:
        fg, fref = np.zeros(3), np.zeros(3)
        for d in range(3):
            p1, p2 = pos.copy(), pos.copy()
            p1[i, d] += h
            p2[i, d] -= h
            fg[d] = -(plan.energy(p1, src).e_total - plan.energy(p2, src).e_total) / (2 * h)
            if R.available():
                fref[d] = -(R.fmm_energy(p1, src, rb, threads=os.cpu_count(), **kw)["e_total"]
                            - R.fmm_energy(p2, src, rb, threads=os.cpu_count(), **kw)["e_total"]) / (2 * h)
        print(f"{kw} i={i} F={f[i]} fd_gpu={fg} fd_ref={fref} |F-fdgpu|={np.abs(f[i]-fg).max():.2e} "
              f"|fdgpu-fdref|={np.abs(fg-fref).max():.2e}", flush=True)
    plan.close()


if __name__ == "__main__":
    run(400, 5.0, 5, True, dict(order_cheb=6, order_equi=6, depth=2, p=15))
    run(400, 5.0, 5, True, dict(order_cheb=6, order_equi=6, depth=2, p=0))
    run(400, 5.0, 5, True, dict(order_cheb=5, order_equi=5, depth=2, p=15))
    run(400, 5.0, 5, True, dict(order_cheb=7, order_equi=7, depth=2, p=15))
