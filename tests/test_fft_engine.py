"""ANKH-FFT engine (Alg. 4-5): the GPU engine
(`Plan(..., engine="fft")`, csrc/k_fft.cu) against the numpy restatement
(oracle/fft_engine.py, itself pinned to a dense pair-by-pair double sum in
test_oracle.py), and its convergence to the reference's own energy as the
orders grow.  The reference has no such engine: there is no drop-in parity
for it, only these checks."""
import os

import numpy as np
import pytest

import paper_2212_08284_b200 as ankh
from paper_2212_08284_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p,Lc,Lu,depth,xi", [(15, 4, 3, 2, 0.01), (15, 5, 5, 2, 0.01), (0, 4, 4, 2, 0.1),
                                              (2, 6, 4, 3, 0.05), (15, 3, 6, 1, 0.3)])
def test_fft_far_matches_numpy_restatement(cuda, p, Lc, Lu, depth, xi):
    import fft_engine as F  # checker only

    pos, src = inputs.random_system(400, 4.0, seed=7 + depth, multipoles=True)
    cfg = ankh.EwaldConfig(order_cheb=Lc, order_equi=Lu, depth=depth, p=p, xi=xi)
    rep = ankh.fft_energy(ankh.ParticleSystem(pos, src, 4.0), cfg)
    want = F.fft_far_energy(pos, src, 4.0, depth, Lc, Lu, xi, periodic=p >= 2)
    assert abs(rep.e_far - want) <= 1e-11 * abs(want) + 1e-13, (rep.e_far, want)
    # the rest of the report is the FMM engine's own
    fmm = ankh.fmm_energy(ankh.ParticleSystem(pos, src, 4.0), cfg)
    assert (rep.e_near, rep.e_self, rep.e_periodic_far) == (fmm.e_near, fmm.e_self, fmm.e_periodic_far)
    assert rep.e_total == ((rep.e_self + rep.e_near) + rep.e_far) + rep.e_periodic_far or \
        abs(rep.e_total - (rep.e_self + rep.e_near + rep.e_far + rep.e_periodic_far)) <= 1e-12 * abs(rep.e_total)


def test_fft_engine_converges_to_the_reference(cuda, ref):
    """Config 0 (the water box, 3,000 atoms): the FFT engine's total against
    the reference's at matched orders L_c = L_u = L -- 8e-6, 1.4e-7, 1.0e-8
    relative at L = 4, 6, 8 (oracle/fft_engine.py, same numbers)."""
    pos, src, rb, _ = inputs.make_config(0)
    for L, tol in ((6, 5e-7), (8, 5e-8)):
        want = ref.fmm_energy(pos, src, rb, order_cheb=L, order_equi=L, threads=os.cpu_count())
        rep = ankh.fft_energy(ankh.ParticleSystem(pos, src, rb), ankh.EwaldConfig(order_cheb=L, order_equi=L))
        assert abs(rep.e_total - want["e_total"]) <= tol * abs(want["e_total"]), (L, rep.e_total, want["e_total"])


def test_fft_engine_plan_reuse_and_limits(cuda):
    pos, src = inputs.random_system(500, 4.0, seed=3, multipoles=True)
    cfg = ankh.EwaldConfig(order_cheb=4, order_equi=4, depth=2)
    plan = ankh.Plan(500, 4.0, cfg, engine="fft")
    try:
        a, b = plan.energy(pos, src), plan.energy(pos, src * 0.5)
        assert a.e_far != 0.0 and abs(b.e_far - 0.25 * a.e_far) <= 1e-12 * abs(a.e_far)  # quadratic
        with pytest.raises(RuntimeError, match="fft engine"):
            plan.forces(pos, src)
    finally:
        plan.close()
    with pytest.raises(ankh.InvalidArgument):
        ankh.Plan(500, 4.0, cfg, engine="bogus")
    with pytest.raises(ankh.InvalidArgument, match="order_equi"):
        ankh.Plan(500, 4.0, ankh.EwaldConfig(order_cheb=4, order_equi=17, depth=2), engine="fft")
    with pytest.raises(RuntimeError, match="depth > 6"):
        ankh.Plan(500, 4.0, ankh.EwaldConfig(order_cheb=4, order_equi=4, depth=7), engine="fft")
