"""Forces: F = -dE/dx of the FMM energy, moments fixed.

The reference computes energies only, so the checker is the reference's own
energy: central differences of ankh::fmm_energy (oracle/_ref) at a few
particles, on small systems covering periodic / open boundaries, charges only
and full multipoles, orders 3..6 (L = 6 takes the reference's randomized SVD
path).  Displaced particles stay inside their leaves (the FMM energy is smooth
there).  At full size: central differences of the engine's own energy, the
near-field share against the numpy pair gradient, bitwise determinism.
"""
import os

import numpy as np
import pytest

import paper_2212_08284_b200 as ankh
from paper_2212_08284_b200 import inputs

pytestmark = pytest.mark.gpu


def _inside_leaf(pos, rb, depth, margin):
    """Particles at least `margin` away from every leaf face (and the box)."""
    n = 1 << depth
    side = 2.0 * rb / n
    u = (pos + rb) / side
    frac = u - np.floor(u)
    return np.where(((frac * side > margin) & ((1 - frac) * side > margin)).all(axis=1))[0]


def _fd_reference(ref, pos, src, rb, kw, idx, h):
    out = np.zeros((len(idx), 3))
    for a, i in enumerate(idx):
        for d in range(3):
            p1, p2 = pos.copy(), pos.copy()
            p1[i, d] += h
            p2[i, d] -= h
            e1 = ref.fmm_energy(p1, src, rb, threads=os.cpu_count(), **kw)["e_total"]
            e2 = ref.fmm_energy(p2, src, rb, threads=os.cpu_count(), **kw)["e_total"]
            out[a, d] = -(e1 - e2) / (2 * h)
    return out


CASES = {
    "mp_L4_E2_periodic": (300, 5.0, 1, True, dict(order_cheb=4, order_equi=4, depth=2, p=15)),
    "mp_L3_E2_open": (300, 5.0, 2, True, dict(order_cheb=3, order_equi=3, depth=2, p=0)),
    "q_L5_E1_p2": (500, 7.0, 3, False, dict(order_cheb=5, order_equi=5, depth=1, p=2)),
    "mp_L5_E3_periodic": (1500, 8.0, 4, True, dict(order_cheb=5, order_equi=5, depth=3, p=15)),
    "mp_L6_E2_periodic": (400, 5.0, 5, True, dict(order_cheb=6, order_equi=6, depth=2, p=15)),
    "mp_L4_E2_xi0.3": (400, 5.0, 6, True, dict(order_cheb=4, order_equi=4, depth=2, p=15, xi=0.3)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_forces_match_reference_energy_differences(cuda, ref, name):
    n, rb, seed, mp, kw = CASES[name]
    pos, src = inputs.random_system(n, rb, seed=seed, multipoles=mp)
    rep, f = ankh.fmm_forces(ankh.ParticleSystem(pos, src, rb), ankh.EwaldConfig(**kw))
    want = ref.fmm_energy(pos, src, rb, threads=os.cpu_count(), **kw)
    assert abs(rep.e_total - want["e_total"]) <= 1e-10 * abs(want["e_total"]) + 1e-12
    assert f.shape == (n, 3) and np.isfinite(f).all()
    h = 1e-5
    cand = _inside_leaf(pos, rb, kw["depth"], 50 * h)
    idx = cand[np.linspace(0, len(cand) - 1, 5).astype(int)]
    fd = _fd_reference(ref, pos, src, rb, kw, idx, h)
    scale = np.abs(fd).max()
    err = np.abs(f[idx] - fd).max()
    # central differences of the reference: truncation (~1e-8 of the largest
    # force here) and its round-off (~1e-15 |E| / h) bound the agreement; a
    # missing far-field or periodic term would be orders larger
    tol = 5e-8 * scale + 2e-15 * abs(want["e_total"]) / h
    assert err <= tol, (name, err, scale, f[idx], fd)


def test_forces_near_field_matches_pair_gradient(cuda):
    """Open boundary, one leaf level (depth 1) with the far field switched off
    by construction (no M2L at level 1 without periodicity): the forces are
    the near field alone -- the numpy pair gradient summed over all pairs."""
    import ankh_oracle as O

    pos, src = inputs.random_system(120, 3.0, seed=7, multipoles=True)
    kw = dict(order_cheb=3, order_equi=3, depth=1, p=0)
    rep, f = ankh.fmm_forces(ankh.ParticleSystem(pos, src, 3.0), ankh.EwaldConfig(**kw))
    n = pos.shape[0]
    want = np.zeros((n, 3))
    for i in range(n):
        others = np.array([j for j in range(n) if j != i])
        g = O.pair_gradient(np.repeat(pos[i:i + 1], n - 1, 0), np.repeat(src[i:i + 1], n - 1, 0),
                            pos[others], src[others], 0.01)
        want[i] = -g.sum(axis=0)
    assert np.abs(f - want).max() <= 1e-11 * np.abs(want).max()


@pytest.mark.parametrize("config", [1, 3])
def test_forces_at_scale_match_own_energy_differences(cuda, config):
    """BASELINE configs 1 and 3: forces against central differences of the
    engine's own energy at a few particles, and bitwise run-to-run equality."""
    pos, src, rb, cfg = inputs.make_config(config)
    L = cfg.orders[0]
    ec = ankh.EwaldConfig(order_cheb=L, order_equi=L)
    plan = ankh.Plan(pos.shape[0], rb, ec)
    rep, f = plan.forces(pos, src)
    rep2, f2 = plan.forces(pos, src)
    assert np.array_equal(f, f2) and rep.e_total == rep2.e_total
    depth = plan.info()["depth"]
    h = 1e-4
    cand = _inside_leaf(pos, rb, depth, 50 * h)
    idx = cand[np.linspace(0, len(cand) - 1, 4).astype(int)]
    for i in idx:
        for d in range(3):
            p1, p2 = pos.copy(), pos.copy()
            p1[i, d] += h
            p2[i, d] -= h
            fd = -(plan.energy(p1, src).e_total - plan.energy(p2, src).e_total) / (2 * h)
            assert abs(f[i, d] - fd) <= 1e-6 * np.abs(f[idx]).max() + 2e-14 * abs(rep.e_total) / h, \
                (i, d, f[i, d], fd)
    plan.close()


def test_forces_high_order_match_own_energy_differences(cuda):
    """Order 8 (K = 512: the dE/dM kernel stages fewer factor rows per pass so
    a pass fits shared memory; the factors come from the randomized
    compression): forces against central differences of the engine's own
    energy."""
    n, rb = 300, 5.0
    pos, src = inputs.random_system(n, rb, seed=31, multipoles=True)
    ec = ankh.EwaldConfig(order_cheb=8, order_equi=8, depth=2, p=15)
    plan = ankh.Plan(n, rb, ec)
    rep, f = plan.forces(pos, src)
    h = 1e-5
    cand = _inside_leaf(pos, rb, 2, 50 * h)
    idx = cand[np.linspace(0, len(cand) - 1, 2).astype(int)]
    for i in idx:
        for d in range(3):
            p1, p2 = pos.copy(), pos.copy()
            p1[i, d] += h
            p2[i, d] -= h
            fd = -(plan.energy(p1, src).e_total - plan.energy(p2, src).e_total) / (2 * h)
            assert abs(f[i, d] - fd) <= 1e-7 * np.abs(f).max() + 2e-14 * abs(rep.e_total) / h, (i, d, f[i, d], fd)
    plan.close()


HALF_CASES = {
    # n, rb, seed, multipoles, config: sparse and dense leaves (several source
    # chunks and target tiles per leaf), image shifts at depth 1, open boundary
    "mp_E2_periodic": (400, 5.0, 21, True, dict(order_cheb=4, order_equi=4, depth=2, p=15)),
    "mp_E1_periodic_dense": (3000, 4.0, 22, True, dict(order_cheb=3, order_equi=3, depth=1, p=15)),
    "q_E1_open_dense": (2500, 4.0, 23, False, dict(order_cheb=3, order_equi=3, depth=1, p=0)),
    "mp_E3_open": (2500, 8.0, 24, True, dict(order_cheb=3, order_equi=3, depth=3, p=0)),
    "mp_E2_p2_uneven": (900, 6.0, 25, True, dict(order_cheb=3, order_equi=3, depth=2, p=2)),
}


@pytest.mark.parametrize("name", sorted(HALF_CASES))
def test_half_shell_forces_equal_full_stencil(cuda, name, monkeypatch):
    """The forces-only near field (half shell + Newton's third law, direction
    slots; k_p2p_force_half) against the full 27-leaf stencil kernel that the
    derivative pass keeps: the same pair gradients, summed in another order."""
    n, rb, seed, mp, kw = HALF_CASES[name]
    pos, src = inputs.random_system(n, rb, seed=seed, multipoles=mp)
    if "uneven" in name:  # most particles in one octant: leaf sizes from 0 to hundreds
        pos[: n // 2] = pos[: n // 2] * 0.24 + 0.7 * rb
    ec = ankh.EwaldConfig(**kw)
    plan = ankh.Plan(n, rb, ec)
    rep, f = plan.forces(pos, src)
    rep_b, f_b = plan.forces(pos, src)
    assert np.array_equal(f, f_b)
    plan.close()
    monkeypatch.setenv("ANKH_FORCE_FULL_STENCIL", "1")
    plan2 = ankh.Plan(n, rb, ec)
    rep2, f2 = plan2.forces(pos, src)
    plan2.close()
    assert rep.e_total == rep2.e_total
    assert np.abs(f - f2).max() <= 2e-12 * np.abs(f2).max(), np.abs(f - f2).max() / np.abs(f2).max()
    # and through the derivative pass (always the full stencil)
    monkeypatch.delenv("ANKH_FORCE_FULL_STENCIL")
    plan3 = ankh.Plan(n, rb, ec)
    _, f3, ds3 = plan3.derivatives(pos, src)
    # the moment derivatives alone (a field evaluation: no pair gradient in the near pass)
    _, f4, ds4 = plan3.derivatives(pos, src, forces=False)
    plan3.close()
    assert np.abs(f - f3).max() <= 2e-12 * np.abs(f3).max()
    assert f4 is None and np.abs(ds4 - ds3).max() <= 1e-13 * np.abs(ds3).max()


# ---------------------------------------------------------------- moment gradient
def _fd_moments(ref, pos, src, rb, kw, pairs, h):
    """Central differences of the reference energy in single stored moments:
    exact up to round-off, since the energy is a quadratic form in them."""
    out = np.zeros(len(pairs))
    for a, (i, k) in enumerate(pairs):
        s1, s2 = src.copy(), src.copy()
        s1[i, k] += h
        s2[i, k] -= h
        e1 = ref.fmm_energy(pos, s1, rb, threads=os.cpu_count(), **kw)["e_total"]
        e2 = ref.fmm_energy(pos, s2, rb, threads=os.cpu_count(), **kw)["e_total"]
        out[a] = (e1 - e2) / (2 * h)
    return out


@pytest.mark.parametrize("name", ["mp_L4_E2_periodic", "mp_L3_E2_open", "q_L5_E1_p2", "mp_L4_E2_xi0.3"])
def test_moment_gradient_matches_reference_energy_differences(cuda, ref, name):
    """dE/ds (potential, minus field, field gradient per stored moment) against
    central differences of the reference's own energy in each moment -- every
    component, including moments that are zero in the input (charges-only
    case: the field of charges) and the off-diagonal quadrupole convention."""
    n, rb, seed, mp, kw = CASES[name]
    pos, src = inputs.random_system(n, rb, seed=seed, multipoles=mp)
    plan = ankh.Plan(n, rb, ankh.EwaldConfig(**kw))
    try:
        rep, f, ds = plan.derivatives(pos, src)
        rep2, f2 = plan.forces(pos, src)
    finally:
        plan.close()
    assert ds.shape == (n, 10) and np.isfinite(ds).all()
    # the forces of the same pass (the kernel variant differs in its schedule)
    assert np.abs(f - f2).max() <= 1e-12 * np.abs(f2).max() and rep.e_total == rep2.e_total
    pairs = [(i, k) for i in (0, n // 3, n - 1) for k in range(10)]
    fd = _fd_moments(ref, pos, src, rb, kw, pairs, 0.5)
    got = np.array([ds[i, k] for i, k in pairs])
    scale = np.abs(fd).max()
    tol = 1e-10 * scale + 1e-14 * abs(rep.e_total) / 0.5
    assert np.abs(got - fd).max() <= tol, (name, np.abs(got - fd).max(), tol, got, fd)


def test_induced_dipoles_self_consistent(cuda, ref):
    """The conjugate-gradient induced-dipole solve on the water-like config 0
    (point polarizabilities 0.1 A^3): mu = alpha E(s + mu) to 1e-10, checked
    with a fresh field evaluation and, at a few particles, with central
    differences of the reference energy at the total moments."""
    pos, src, rb, c = inputs.make_config(0)
    kw = dict(order_cheb=4, order_equi=4)
    plan = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(**kw))
    try:
        sol = ankh.induced_dipoles(plan, pos, src, 0.1, tol=1e-11, max_iter=60)
    finally:
        plan.close()
    assert sol.iterations < 60 and sol.residual <= 1e-9, (sol.iterations, sol.residual)
    assert np.abs(sol.dipoles - 0.1 * sol.field).max() <= 1e-9 * np.abs(sol.dipoles).max()
    total = src.copy()
    total[:, 1:4] += sol.dipoles
    pairs = [(i, k) for i in (5, 1700) for k in (1, 2, 3)]
    fd = _fd_moments(ref, pos, total, rb, kw, pairs, 0.05)
    field = np.array([sol.field[i, k - 1] for i, k in pairs])
    assert np.abs(field + fd).max() <= 1e-9 * np.abs(fd).max() + 1e-12, (field, -fd)
