"""CPU tests of the oracle: the numpy restatement (oracle/ankh_oracle.py) is pinned
against the reference itself (oracle/_ref, the unmodified reference sources
compiled against oracle/shim) and against the SPEC known-answer values."""
import math

import numpy as np
import pytest

import ankh_oracle as O
from paper_2212_08284_b200 import inputs


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


# ---------------------------------------------------------------- SPEC KATs
def test_erfc_screen_kat():
    # erfc(0.01) ~= 0.98871658
    assert abs(float(O.erfc_screen(0.01)) - 0.98871658) < 5e-9
    assert float(O.erfc_screen(0.0)) == 1.0
    for z in (0.1, 0.3, 0.5, 0.7, 2.0):
        assert rel(float(O.erfc_screen(z)), math.erfc(z)) < 1e-15


def test_pair_interaction_unit_charges():
    # two unit charges at distance 1, xi=0.01 -> erfc(0.01)
    sa = np.array([1.0] + [0.0] * 9)
    e = O.pair_interaction(np.array([1.0, 0, 0]), sa, np.zeros(3), sa, 0.01)[0]
    assert rel(e, float(O.erfc_screen(0.01))) < 1e-15
    # all moments zero on one side -> 0
    z = np.zeros(10)
    assert O.pair_interaction(np.array([1.0, 0, 0]), sa, np.zeros(3), z, 0.01)[0] == 0.0


def test_pair_interaction_matches_finite_difference():
    # charge 1 at origin and a pure dipole mu=(1,0,0) at (2,0,0):
    # D_b H = mu . grad_y H(x, y)
    xi = 0.01
    h = lambda x, y: O.erfc_screen(xi * np.linalg.norm(x - y)) / np.linalg.norm(x - y)
    sa = np.array([1.0] + [0.0] * 9)
    sb = np.array([0.0, 1.0, 0, 0] + [0.0] * 6)
    xa, xb = np.zeros(3), np.array([2.0, 0, 0])
    e = O.pair_interaction(xa, sa, xb, sb, xi)[0]
    d = 1e-5
    fd = (h(xa, xb + [d, 0, 0]) - h(xa, xb - [d, 0, 0])) / (2 * d)
    assert rel(e, fd) < 1e-6


@pytest.mark.parametrize("xi,seed", [(0.01, 1), (0.3, 2), (0.6, 3)])
def test_pair_gradient_matches_reference_finite_differences(ref, xi, seed):
    """The forces' pair gradient (oracle pair_gradient, the restatement the
    GPU's pair_grad_mp follows) against central differences of the
    reference's own pair_interaction (kernel.cpp:157-204), for full q/mu/Theta
    pairs and the charge-only / dipole-only special cases."""
    rng = np.random.default_rng(seed)
    for kind in ("full", "q", "mu"):
        xa, xb = rng.normal(size=3) * 2.0, rng.normal(size=3) * 2.0
        sa, sb = rng.normal(size=10), rng.normal(size=10)
        if kind == "q":
            sa[1:] = sb[1:] = 0.0
        if kind == "mu":
            sa[4:] = sb[4:] = 0.0
        g = O.pair_gradient(xa, sa, xb, sb, xi)[0]
        h = 1e-5
        fd = np.array([(ref.pair_interaction(xa + h * e, sa, xb, sb, xi)
                        - ref.pair_interaction(xa - h * e, sa, xb, sb, xi)) / (2 * h) for e in np.eye(3)])
        assert np.abs(g - fd).max() <= 1e-8 * np.abs(fd).max(), (kind, g, fd)


def test_pair_interaction_symmetry():
    rng = np.random.default_rng(3)
    for _ in range(20):
        xa, xb = rng.uniform(-2, 2, 3), rng.uniform(-2, 2, 3)
        sa = np.concatenate([[rng.uniform(-1, 1)], rng.normal(0, 0.3, 9)])
        sb = np.concatenate([[rng.uniform(-1, 1)], rng.normal(0, 0.3, 9)])
        assert rel(O.pair_interaction(xa, sa, xb, sb, 0.2)[0],
                   O.pair_interaction(xb, sb, xa, sa, 0.2)[0]) < 1e-12


def test_self_energy_kats():
    # SPEC.md:113-115
    assert rel(O.self_energy(np.array([[1.0] + [0.0] * 9]), 0.01), -0.01 / math.sqrt(math.pi)) < 1e-15
    assert rel(O.self_energy(np.array([[0.0, 1.0, 0, 0] + [0.0] * 6]), 1.0),
               -(2.0 / 3.0) / math.sqrt(math.pi)) < 1e-15
    assert O.self_energy(np.zeros((0, 10)), 0.01) == 0.0


def test_lagrange_cardinal_and_partition_of_unity():
    # SPEC.md:160-162
    for L in (2, 3, 5, 8):
        nodes = O.cheb_nodes(L)
        for k in range(L):
            for j in range(L):
                assert abs(O.lagrange_eval_cheb(L, k, nodes[j]) - (1.0 if j == k else 0.0)) < 1e-13
        for x in (-1.0, -0.3, 0.0, 0.77, 1.0):
            assert abs(sum(O.lagrange_eval_cheb(L, k, x) for k in range(L)) - 1.0) < 1e-13
            assert abs(sum(O.lagrange_eval_equi(L, k, x) for k in range(L)) - 1.0) < 1e-13


def test_build_tree_center_particle():
    # particle at the box centre with E=1 lands in leaf (1,1,1)
    b = O.build_tree(np.zeros((1, 3)), 1.0, 1)
    assert len(b[(1 * 2 + 1) * 2 + 1]) == 1
    # upper boundary particles go to the last cell (octree.cpp:39-40)
    b = O.build_tree(np.array([[1.0, 1.0, 1.0]]), 1.0, 2)
    assert len(b[63]) == 1
    with pytest.raises(O.InvalidArgument, match="depth must be in"):
        O.build_tree(np.zeros((1, 3)), 1.0, 9)


def test_interaction_list_sizes():
    # periodic: 189 for every cell at every level; open E=2 corner leaf: 56
    for level in (1, 2, 3):
        t, _, _ = O.lambda_list(level, True)
        assert (np.bincount(t, minlength=8 ** level) == 189).all()
    t, _, _ = O.lambda_list(1, False)
    assert t.size == 0
    t, _, _ = O.lambda_list(2, False)
    assert np.bincount(t, minlength=64)[0] == 56


def test_default_depth():
    assert [O.default_depth(n) for n in (3000, 24000, 96000, 1029000, 8232000)] == [2, 3, 4, 5, 6]
    assert O.default_depth(0) == 1 and O.default_depth(64) == 1 and O.default_depth(65) == 1


def test_mt19937_64_known_answer():
    # [rand.predef]: the 10000th draw of a default-seeded mt19937_64
    r = O.MT19937_64(5489)
    assert int(r.draw(10000)[-1]) == 9981545732273789042


def test_validate_messages():
    with pytest.raises(O.InvalidArgument, match="xi must be positive"):
        O.validate_config(0.0, 15, 8, 8, 0, 1e-7, 12)
    with pytest.raises(O.InvalidArgument, match="image half-width"):
        O.validate_config(0.01, 1, 8, 8, 0, 1e-7, 12)
    pos = np.array([[0.0, 0, 0], [0.5, 0, 0], [0.0, 0, 0], [2.0, 0, 0]])
    v = O.validate_system(pos, np.zeros((4, 10)), 1.0)
    assert v[0] == (3, "outside box")
    assert (2, "duplicate position") in v


# --------------------------------------------------- pin against the reference
def test_kats_against_reference(ref, golden):
    for z, want in golden["kats"]["erfc_screen"].items():
        assert rel(float(O.erfc_screen(float(z))), float(want)) < 2e-15
    for p in golden["kats"]["pair_interaction"]:
        got = O.pair_interaction(np.array(p["xa"]), np.array(p["sa"]), np.array(p["xb"]),
                                 np.array(p["sb"]), p["xi"])[0]
        assert rel(got, float(p["e"])) < 1e-13
    for n, d in golden["kats"]["default_depth"].items():
        assert O.default_depth(int(n)) == d


def test_list_sizes_against_reference(ref):
    lam, nb = ref.list_sizes(2, False, 2)
    t, _, _ = O.lambda_list(2, False)
    assert (np.bincount(t, minlength=64) == lam).all()
    a, _, _ = O.leaf_neighbors(2, False)
    assert (np.bincount(a, minlength=64) == nb).all()
    lam, nb = ref.list_sizes(3, True, 2)
    t, _, _ = O.lambda_list(2, True)
    assert (np.bincount(t, minlength=64) == lam).all()


@pytest.mark.parametrize("seed,n,rb,depth", [(0, 500, 4.0, 2), (1, 3000, 10.0, 3), (2, 37, 1.0, 1)])
def test_leaf_csr_against_reference(ref, seed, n, rb, depth):
    pos, _ = inputs.random_system(n, rb, seed=seed)
    pos[0] = [rb, rb, rb]      # upper boundary
    pos[1] = [-rb, 0.0, rb]
    offs, idx = ref.leaf_csr(pos, rb, depth)
    o2, i2 = O.leaf_csr(pos, rb, depth)
    assert (offs == o2).all() and (idx == i2).all()


@pytest.mark.parametrize("kw", [
    dict(order_cheb=4, order_equi=4, depth=2, p=15),
    dict(order_cheb=3, order_equi=3, depth=2, p=0),
    dict(order_cheb=5, order_equi=5, depth=1, p=2),
])
def test_restatement_matches_reference(ref, kw):
    pos, src = inputs.random_system(300, 5.0, seed=7, multipoles=True)
    a = ref.fmm_energy(pos, src, 5.0, threads=4, **kw)
    b = O.fmm_energy(pos, src, 5.0, **kw)
    assert rel(b["e_total"], a["e_total"]) < 1e-11
    for k in ("e_near", "e_far", "e_self"):
        assert rel(b[k], a[k]) < 1e-12, k
    assert rel(b["e_periodic_far"], a["e_periodic_far"]) < 1e-9


def test_restatement_randomized_svd_path(ref):
    # K = 216 > 150: seeded randomized range finder (fmm.cpp:117-132)
    lm, rm = ref.m2l_factors(6, 0.7, (2, 1, 0), seed=12345)
    c = O.m2l_dense(6, 0.7, (2, 1, 0), 0.01)
    l2, r2 = O.compress_m2l(c, 1e-7, 12345)
    assert lm.shape == l2.shape
    a, b = lm.T @ rm, l2.T @ r2
    assert np.abs(a - b).max() / np.abs(c).max() < 1e-12


def test_m2l_dense_matches_reference(ref):
    for off in ((2, 0, 0), (-3, 1, 2), (0, -2, 3)):
        c = O.m2l_dense(4, 1.3, off, 0.01)
        # same operation order; the reference build may contract to FMA
        assert np.abs(c - ref.m2l_dense(4, 1.3, off, 0.01)).max() <= 4e-16 * np.abs(c).max()


def test_expansions_match_reference(ref):
    pos, src = inputs.random_system(400, 3.0, seed=5, multipoles=True)
    ex = ref.expansions(pos, src, 3.0, 2, 4)
    b = O.build_tree(pos, 3.0, 2)
    ex2 = O.upward_pass(O.leaf_expansions(pos, src, 3.0, b, 2, 4), 2, 4)
    for l in range(3):
        scale = np.abs(ex[l]).max()
        assert np.abs(ex[l] - ex2[l]).max() <= 1e-13 * scale


def test_golden_small_systems(golden):
    """The restatement reproduces the reference's golden energies."""
    for case in golden["systems"]:
        if case["kind"] != "random" or case["n"] > 600:
            continue
        pos, src = inputs.random_system(case["n"], case["box_radius"], seed=case["seed"],
                                        multipoles=case["multipoles"])
        import hashlib

        h = hashlib.sha256(pos.tobytes() + src.tobytes()).hexdigest()
        assert h == case["sha256"], "input generator drifted"
        kw = dict(case["config"])
        got = O.fmm_energy(pos, src, case["box_radius"], **kw)
        want = {k: float(v) for k, v in case["energies"].items()}
        assert rel(got["e_total"], want["e_total"]) < 1e-10, case["name"]


def test_fft_engine_restatement_matches_dense_sum():
    """oracle/fft_engine.py: the circulant/DFT evaluation of 1/2 v^T A v equals
    the pair-by-pair dense sum on tiny trees (periodic and open), and its
    spectrum is real (Cor. 3)."""
    import fft_engine as F

    from paper_2212_08284_b200 import inputs

    for depth, Lu, xi, per in ((1, 3, 0.3, True), (2, 3, 0.1, True), (2, 2, 0.1, False)):
        pos, src = inputs.random_system(120, 3.0, seed=depth, multipoles=True)
        v = F.equi_leaf_values(pos, src, 3.0, depth, 4, Lu)
        G = F.generator(3.0, depth, Lu, xi, per)
        got = F.fft_far(v, G)
        want = F.dense_far(v, 3.0, depth, Lu, xi, per)
        assert abs(got - want) <= 1e-12 * abs(want)
        d = np.fft.fftn(G)
        assert np.abs(d.imag).max() <= 1e-10 * np.abs(d).max()
