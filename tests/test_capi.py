"""CPU tests of the drop-in boundary: libankh_b200.so loads, exports every
symbol include/ankh_b200.h declares, and rejects invalid configurations with
the reference's messages before touching a device."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2212_08284_b200 as ankh
from paper_2212_08284_b200 import _lib, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "ankh_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(ankh_[a-z0-9_]+_v1)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ankh.lib()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {ankh.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    # ankh_config_v1 / ankh_report_v1 sizes as laid out by the C compiler
    assert ctypes.sizeof(api._Config) == 56
    assert ctypes.sizeof(api._Report) == 13 * 8 + 2 * 4 + 8 + 8 + 8 + 8


def test_default_config_matches_ewaldconfig():
    c = api._Config()
    ankh.lib().ankh_config_default_v1(ctypes.byref(c))
    d = ankh.EwaldConfig()
    assert (c.xi, c.p, c.order_cheb, c.order_equi, c.depth, c.svd_tol, c.recip_cutoff) == \
        (d.xi, d.p, d.order_cheb, d.order_equi, d.depth, d.svd_tol, d.recip_cutoff)


@pytest.mark.parametrize("kw,msg", [
    (dict(xi=0.0), "xi must be positive"),
    (dict(xi=float("nan")), "xi must be positive"),
    (dict(p=1), "image half-width p must be 0 (open) or >= 2 (periodic)"),
    (dict(p=-3), "image half-width p must be 0 (open) or >= 2 (periodic)"),
    (dict(order_cheb=1), "order_cheb must be >= 2"),
    (dict(order_equi=0), "order_equi must be >= 2"),
    (dict(depth=-1), "depth must be >= 1 (or 0 for automatic)"),
    (dict(svd_tol=0.0), "svd_tol must lie in (0, 1)"),
    (dict(svd_tol=1.0), "svd_tol must lie in (0, 1)"),
    (dict(recip_cutoff=0), "recip_cutoff must be >= 1"),
])
def test_config_errors_match_reference(kw, msg):
    # validate_config runs first (fmm.cpp:384) -- no device needed
    sys_ = ankh.ParticleSystem(np.zeros((1, 3)), np.array([[1.0] + [0.0] * 9]), 1.0)
    with pytest.raises(ankh.InvalidArgument) as ei:
        ankh.fmm_energy(sys_, ankh.EwaldConfig(**kw))
    assert str(ei.value) == msg


def test_size_mismatch_message():
    with pytest.raises(ankh.InvalidArgument, match="positions and sources must have equal length"):
        ankh.fmm_energy(ankh.ParticleSystem(np.zeros((2, 3)), np.zeros((1, 10)), 1.0))


# Pairs of violations in one call: the error raised is the reference's first
# (validate_config, then validate_system's box_radius, size-mismatch and
# per-particle rules -- fmm.cpp:384-388, types.cpp:20-26).  All of these fail
# before any device work.
_NAN = float("nan")
_PRECEDENCE = {
    "config+box": (dict(xi=-1.0), -1.0, 2, 2, False),
    "config+size": (dict(p=1), 1.0, 2, 1, False),
    "config+particle": (dict(order_cheb=1), 1.0, 2, 2, True),
    "box+size": ({}, float("inf"), 3, 2, False),
    "box+particle": ({}, 0.0, 2, 2, True),
    "size+particle": ({}, 1.0, 3, 2, True),
}


@pytest.mark.parametrize("case", sorted(_PRECEDENCE))
def test_error_precedence_matches_reference(case, ref):
    kw, rb, n_pos, n_src, nan_particle = _PRECEDENCE[case]
    pos = np.full((n_pos, 3), 0.25)
    pos[:, 0] = np.linspace(-0.5, 0.5, n_pos)
    src = np.zeros((n_src, 10))
    src[:, 0] = 1.0
    if nan_particle:
        pos[0, 1] = _NAN
    code, want = ref.fmm_energy_error(pos, src, rb, **kw)
    assert code == 1 and want, (code, want)
    with pytest.raises(ankh.InvalidArgument) as ei:
        ankh.fmm_energy(ankh.ParticleSystem(pos, src, rb), ankh.EwaldConfig(**kw))
    assert str(ei.value) == want


def test_check_call_orders_rules():
    """ankh_check_call_v1 itself (the C++ header's path): config, then box
    radius, then sizes."""
    c = api._Config()
    ankh.lib().ankh_config_default_v1(ctypes.byref(c))
    err = ctypes.create_string_buffer(512)
    chk = lambda rb, a, b: (ankh.lib().ankh_check_call_v1(ctypes.byref(c), rb, a, b, err, 512),
                            err.value.decode())
    assert chk(1.0, 3, 3) == (0, "")
    assert chk(-1.0, 3, 2) == (1, "fmm_energy: invalid system: box_radius must be positive and finite")
    assert chk(1.0, 3, 2) == (1, "fmm_energy: invalid system: positions and sources must have equal length")
    c.svd_tol = 2.0
    assert chk(-1.0, 3, 2) == (1, "svd_tol must lie in (0, 1)")


def test_default_depth_matches_reference_rule():
    import ankh_oracle as O

    for n in (0, 1, 64, 65, 511, 512, 513, 3000, 24000, 96000, 1029000, 8232000, 10 ** 8):
        assert ankh.default_depth(n) == O.default_depth(n)


def test_product_does_not_import_oracle():
    """The product path must never route through the checker."""
    pkg = os.path.join(ROOT, "paper_2212_08284_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp", ".h")):
                with open(os.path.join(dirpath, fn)) as f:
                    text = f.read()
                assert "ankh_oracle" not in text and "libankh_ref" not in text, fn
                assert "import ref" not in text, fn


@pytest.mark.parametrize("s_max, want_nt", [(0.0212, 6), (0.0556, 6), (0.0718, 7), (0.167, 8),
                                            (0.25, 8), (0.4, 14)])
def test_radial_fit_is_roundoff_accurate(s_max, want_nt):
    """The near-field radial polynomials (host fit, no GPU needed) reproduce
    erf(sqrt s)/sqrt s and (2/sqrt pi) exp(-s) -- the functions behind
    erfc_screen / radial, kernel.cpp:14-51 -- to 2.5e-14 relative on the
    plan's range (the fit's target: < 1e-15 of the radial factors b0 and g,
    10^4 below the 1e-11 component gate), checked here independently in
    numpy long double."""
    import ctypes
    import math

    L = ankh.lib()
    nt, sl, err = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    p = (ctypes.c_double * 14)()
    g = (ctypes.c_double * 14)()
    assert L.ankh_radial_fit_v1(s_max, ctypes.byref(nt), ctypes.byref(sl), p, g, ctypes.byref(err)) == 0
    assert nt.value == want_nt
    ld = np.longdouble
    two_sqrtpi = ld(2) / np.sqrt(ld(math.pi))
    s = np.linspace(0, min(s_max, sl.value), 997).astype(ld)
    ps = np.zeros_like(s)
    term = np.full_like(s, two_sqrtpi)
    for k in range(40):
        ps += term / (2 * k + 1)
        term *= -s / (k + 1)
    gs = two_sqrtpi * np.exp(-s)
    for coef, ref in ((p, ps), (g, gs)):
        h = np.full_like(s, ld(coef[nt.value - 1]))
        for k in range(nt.value - 2, -1, -1):
            h = h * s + ld(coef[k])
        assert float(np.max(np.abs((h - ref) / ref))) < 2.6e-14
    assert err.value < 2.6e-14


def test_induced_dipole_solver_logic_on_a_linear_mock():
    """Host logic of api.induced_dipoles (conjugate gradients on
    (alpha^-1 - J) mu = F0, one field evaluation per product) against a dense
    solve, with a mock plan whose field is linear in the moments."""
    import paper_2212_08284_b200 as ankh

    rng = np.random.default_rng(3)
    n = 40
    B = rng.normal(0, 0.2, (3 * n, 3 * n))
    J = 0.5 * (B + B.T) / np.sqrt(3 * n)
    Gq = rng.normal(0, 1.0, (3 * n, n))

    class Mock:
        calls = 0

        def field(self, pos, s):
            Mock.calls += 1
            return (Gq @ s[:, 0] + J @ s[:, 1:4].reshape(-1)).reshape(n, 3)

    pos = np.zeros((n, 3))
    src = rng.normal(0, 1.0, (n, 10))
    alpha = rng.uniform(0.2, 0.5, n)
    sol = ankh.induced_dipoles(Mock(), pos, src, alpha, tol=1e-13, max_iter=500)
    f0 = (Gq @ src[:, 0] + J @ src[:, 1:4].reshape(-1))
    A = np.diag(np.repeat(1.0 / alpha, 3)) - J
    want = np.linalg.solve(A, f0).reshape(n, 3)
    assert np.abs(sol.dipoles - want).max() <= 1e-10 * np.abs(want).max()
    assert sol.residual <= 1e-11 and sol.iterations <= 3 * n
    assert Mock.calls == sol.iterations + 3  # F0, the first product, one per iteration, the check
    with pytest.raises(ankh.InvalidArgument):
        ankh.induced_dipoles(Mock(), pos, src, 0.0)


def test_forces_out_buffer_is_validated():
    """Plan.forces(out=...) rejects a buffer of the wrong shape, dtype or
    layout before any library call (host logic; no GPU needed)."""
    import numpy as np

    from paper_2212_08284_b200 import api

    class P(api.Plan):
        def __init__(self):  # no library handle: the checks come first
            self.n = 4
            self._h = None

        def close(self):
            pass

    p = P()
    pos, src = np.zeros((4, 3)), np.zeros((4, 10))
    for bad in (np.zeros((3, 3)), np.zeros((4, 3), dtype=np.float32), np.zeros((3, 4)).T, [[0.0] * 3] * 4):
        with pytest.raises(ValueError):
            p.forces(pos, src, out=bad)
