"""The C++ drop-in header (include/ankh_b200.hpp): a reference-style caller
compiles against it (with its own or the reference's value types), links
libankh_b200.so, and on the GPU returns the same energies as the Python API."""
import os
import subprocess

import numpy as np
import pytest

import paper_2212_08284_b200 as ankh
from paper_2212_08284_b200 import inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp")
LIBDIR = os.path.join(ROOT, "paper_2212_08284_b200")


def compile_dropin(out, ref_types=False):
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-L", LIBDIR,
           "-lankh_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    if ref_types:
        cmd[3:3] = ["-DANKH_B200_USE_REFERENCE_TYPES", "-I", "/root/reference/proj/core/include"]
    subprocess.run(cmd, check=True)


def test_dropin_compiles(tmp_path):
    compile_dropin(str(tmp_path / "dropin"))


def test_dropin_compiles_with_reference_types(tmp_path):
    if not os.path.isdir("/root/reference/proj/core/include"):
        pytest.skip("reference headers not present on this host")
    compile_dropin(str(tmp_path / "dropin_ref"), ref_types=True)


@pytest.mark.gpu
def test_dropin_runs_and_matches_python(cuda, tmp_path):
    exe = str(tmp_path / "dropin")
    compile_dropin(exe)
    pos, src = inputs.random_system(700, 5.0, seed=17, multipoles=True)
    f = str(tmp_path / "p.txt")
    inputs.write_particle_file(f, pos, src, 5.0, comment="drop-in test")
    out = subprocess.run([exe, f, "4", "2", "15"], check=True, capture_output=True, text=True).stdout
    vals = [float(v) for v in out.splitlines()[0].split()]
    assert "invalid_argument: xi must be positive" in out
    p2, s2, rb = inputs.read_particle_file(f)
    assert np.array_equal(p2, pos) and np.array_equal(s2, src)
    r = ankh.fmm_energy(ankh.ParticleSystem(pos, src, 5.0),
                        ankh.EwaldConfig(order_cheb=4, order_equi=4, depth=2, p=15))
    assert vals == [r.e_total, r.e_self, r.e_near, r.e_far, r.e_periodic_far]
    # the RAII plan with bound positions: same energy, and a quarter of it for
    # moments halved (the energy is a quadratic form in the moments)
    line = [l for l in out.splitlines() if l.startswith("plan ")][0].split()
    full, quarter = float(line[1]), float(line[2])
    assert full == r.e_total
    assert abs(quarter - 0.25 * r.e_total) <= 1e-12 * abs(r.e_total)
    line = [l for l in out.splitlines() if l.startswith("forces ")][0].split()
    rf, f = ankh.fmm_forces(ankh.ParticleSystem(pos, src, 5.0),
                            ankh.EwaldConfig(order_cheb=4, order_equi=4, depth=2, p=15))
    assert [float(v) for v in line[1:]] == [rf.e_total, f[0, 0], f[0, 1], f[-1, 2]]
    line = [l for l in out.splitlines() if l.startswith("mgrad ")][0].split()
    plan = ankh.Plan(pos.shape[0], 5.0, ankh.EwaldConfig(order_cheb=4, order_equi=4, depth=2, p=15))
    try:
        rg, _, ds = plan.derivatives(pos, src, forces=False)
    finally:
        plan.close()
    got = [float(v) for v in line[1:]]
    want = [rg.e_total, ds[0, 0], ds[0, 1], ds[-1, 5]]
    assert np.allclose(got, want, rtol=1e-13, atol=0.0), (got, want)
