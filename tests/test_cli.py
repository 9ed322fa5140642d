"""CLI (SPEC `cli` module): particle files, exit codes,
manifest/report round trip (CPU) and the energy / compare / bench commands
(GPU)."""
import json
import os

import numpy as np
import pytest

import paper_2212_08284_b200 as ankh
from paper_2212_08284_b200 import cli, inputs


def run(argv, capsys=None):
    code = cli.main(argv)
    out = capsys.readouterr() if capsys else None
    return code, out


def test_gen_single_particle_and_determinism(tmp_path):
    a, b, c = (str(tmp_path / f) for f in ("a.txt", "b.txt", "c.txt"))
    assert cli.main(["gen", "--n", "1", "--box-radius", "5", "--seed", "7", "-o", a]) == 0
    pos, src, rb = inputs.read_particle_file(a)
    assert pos.shape == (1, 3) and src.shape == (1, 10) and rb == 5.0
    assert cli.main(["gen", "--n", "200", "--box-radius", "9", "--seed", "3", "-o", b]) == 0
    assert cli.main(["gen", "--n", "200", "--box-radius", "9", "--seed", "3", "-o", c]) == 0
    assert open(b, "rb").read() == open(c, "rb").read()  # same seed -> byte-identical


def test_gen_moment_bounds_and_box(tmp_path):
    f = str(tmp_path / "g.txt")
    assert cli.main(["gen", "--n", "500", "--box-radius", "4", "--seed", "1", "--moments", "full",
                     "-o", f]) == 0
    pos, src, rb = inputs.read_particle_file(f)
    assert np.all(np.abs(pos) <= rb)
    q = np.abs(src[:, 0])
    assert np.all(np.linalg.norm(src[:, 1:4], axis=1) <= 0.1 * q + 1e-15)
    theta = np.abs(src[:, 4:10]).max(axis=1)
    assert np.all(theta <= 0.1 * q)


def test_gen_water_box_648(tmp_path):
    """SPEC's desk-scale stand-in: 648 atoms, r_B = 9.3215 (216 waters)."""
    f = str(tmp_path / "w.txt")
    assert cli.main(["gen", "--kind", "lattice-jittered", "--n", "648", "--box-radius", "9.3215",
                     "--seed", "5", "-o", f]) == 0
    pos, src, rb = inputs.read_particle_file(f)
    assert pos.shape[0] == 648 and abs(src[:, 0].sum()) < 1e-12
    assert sorted(set(np.round(src[:, 0], 3))) == [-0.834, 0.417]


def test_gen_baseline_config(tmp_path):
    f = str(tmp_path / "c0.txt")
    assert cli.main(["gen", "--config", "0", "-o", f]) == 0
    pos, src, rb = inputs.read_particle_file(f)
    want_pos, want_src, want_rb, _ = inputs.make_config(0)
    assert np.array_equal(pos, want_pos) and np.array_equal(src, want_src) and rb == want_rb


def test_gen_invalid_n_is_config_error(tmp_path, capsys):
    code, _ = run(["gen", "--n", "0", "--box-radius", "1", "-o", str(tmp_path / "x")], capsys)
    assert code == cli.EXIT_CONFIG


def test_malformed_row_names_line(tmp_path, capsys):
    f = tmp_path / "bad.txt"
    f.write_text("# comment\n2 5.0\n" + " ".join(["0.1"] * 13) + "\n" + " ".join(["0.1"] * 12) + "\n")
    code, out = run(["energy", "-i", str(f)], capsys)
    assert code == cli.EXIT_PARSE
    assert "line 4" in out.err and "13 values" in out.err


@pytest.mark.parametrize("body, msg", [
    ("2 5.0\n" + " ".join(["0.1"] * 13) + "\n", "header says 2 rows"),
    ("1 5.0\n" + " ".join(["0.1"] * 12 + ["nan"]) + "\n", "non-finite"),
    ("1 5.0\n" + " ".join(["0.1"] * 12 + ["x"]) + "\n", "not a decimal"),
    ("# only a comment\n", "missing header"),
])
def test_particle_file_invariants(tmp_path, body, msg):
    f = tmp_path / "p.txt"
    f.write_text(body)
    with pytest.raises(inputs.ParticleFileError, match=msg):
        inputs.read_particle_file(str(f))


def test_unavailable_method_is_config_error(tmp_path, capsys):
    f = str(tmp_path / "s.txt")
    assert cli.main(["gen", "--n", "10", "--box-radius", "3", "-o", f]) == 0
    code, out = run(["compare", "-i", f, "--runs", "fmm", "fft:order_cheb=8"], capsys)
    assert code == cli.EXIT_CONFIG and "fft" in out.err
    code, out = run(["energy", "-i", f, "--method", "ewald"], capsys)
    assert code == cli.EXIT_CONFIG


def test_budget_guard(tmp_path, capsys):
    f = str(tmp_path / "s.txt")
    assert cli.main(["gen", "--n", "50", "--box-radius", "3", "-o", f]) == 0
    code, out = run(["energy", "-i", f, "--max-atoms", "10"], capsys)
    assert code == cli.EXIT_BUDGET


def test_config_error_exit_code(tmp_path, capsys):
    """validate_config's invalid_argument (types.cpp:65-79) maps to exit 3; the
    check runs in the library before any device work."""
    f = str(tmp_path / "s.txt")
    assert cli.main(["gen", "--n", "10", "--box-radius", "3", "-o", f]) == 0
    code, out = run(["energy", "-i", f, "--xi", "-1"], capsys)
    assert code == cli.EXIT_CONFIG and "xi" in out.err


def test_bench_sizes_must_ascend(capsys):
    code, _ = run(["bench", "--sizes", "3000,300"], capsys)
    assert code == cli.EXIT_CONFIG


def test_document_round_trip():
    m = cli.RunManifest(method="fmm", config={"order_cheb": 5, "order_equi": 5, "xi": 0.01},
                        input="in.txt", output="out.json", seed=3, threads=4)
    r = ankh.EnergyReport(e_total=-209936.42899994756, e_self=-1.0 / 3.0, e_near=1e-300,
                          e_far=-12134.688437507937, e_periodic_far=2.373543930608787e-10,
                          wall_times={"total": 0.1, "near_field": 1.0 / 7.0}, depth=5, order_cheb=5,
                          near_pairs=439460636, far_instances=3540000, far_flops=4.76e10,
                          gpu_launches=19)
    text = json.dumps(cli.document(m, r))
    m2, r2 = cli.load_document(text)
    assert m2 == m and r2 == r


@pytest.mark.gpu
def test_energy_document_matches_api(tmp_path, cuda):
    f, o = str(tmp_path / "s.txt"), str(tmp_path / "o.json")
    assert cli.main(["gen", "--n", "400", "--box-radius", "6", "--seed", "2", "-o", f]) == 0
    assert cli.main(["energy", "-i", f, "--order-cheb", "4", "--depth", "2", "-o", o]) == 0
    m, r = cli.load_document(open(o).read())
    pos, src, rb = inputs.read_particle_file(f)
    want = ankh.fmm_energy(ankh.ParticleSystem(pos, src, rb),
                           ankh.EwaldConfig(order_cheb=4, order_equi=4, depth=2))
    assert r.e_total == want.e_total and m.config["order_cheb"] == 4
    # a manifest file drives the same run
    mf = tmp_path / "m.json"
    mf.write_text(json.dumps({"method": "fmm", "config": {"order_cheb": 4, "order_equi": 4, "depth": 2},
                              "input": f}))
    o2 = str(tmp_path / "o2.json")
    assert cli.main(["energy", "--manifest", str(mf), "-o", o2]) == 0
    assert cli.load_document(open(o2).read())[1].e_total == want.e_total


@pytest.mark.gpu
def test_compare_order_sweep_converges(tmp_path, cuda, capsys):
    """cmd_compare: r = |E_ref - E| / |E_ref| against the L = 6 run (the
    reference run first) is much smaller at L = 5 than at L = 3 (geometric
    convergence of the Chebyshev interpolation; consecutive orders need not be
    monotone -- config 2 gives 2.02e-6, 2.04e-6, 1.5e-7 at L = 3, 4, 5)."""
    f, o = str(tmp_path / "s.txt"), str(tmp_path / "cmp.json")
    assert cli.main(["gen", "--kind", "lattice-jittered", "--n", "648", "--box-radius", "9.3215",
                     "--seed", "4", "-o", f]) == 0
    runs = ["fmm:order_cheb=6,depth=2", "fmm:order_cheb=3,depth=2", "fmm:order_cheb=5,depth=2"]
    assert cli.main(["compare", "-i", f, "--runs", *runs, "-o", o]) == 0
    rows = json.load(open(o))["rows"]
    assert rows[0]["r"] == 0.0
    assert 0.0 < rows[2]["r"] < rows[1]["r"] / 4, [r["r"] for r in rows]


@pytest.mark.gpu
def test_bench_table(cuda, capsys):
    code = cli.main(["bench", "--sizes", "3000,24000", "--order-cheb", "4", "--repeat", "1",
                     "--format", "json"])
    out = capsys.readouterr().out
    assert code == 0
    rows = json.loads(out)["rows"]
    assert [r["atoms"] for r in rows] == [3000, 24000]
    assert all(r["t_near_field"] > 0 and r["plan_build_s"] > 0 for r in rows)
