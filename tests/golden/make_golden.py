"""Generate tests/golden/*.json from the REFERENCE itself.

The reference's unmodified sources, compiled against oracle/shim into
oracle/_ref/libankh_ref.so (oracle/Makefile), are run on seeded inputs from
paper_2212_08284_b200.inputs.  Inputs are not stored; their sha256 is, so a
generator drift is detected instead of silently comparing different systems.

    python tests/golden/make_golden.py [--big | --high | --config 3|4]

--big adds configs 1 and 2 (L = 3..6), which take minutes on the CPU;
--high writes the order 8-10 random systems (golden_high.json), --higher the
order 11-16 ones (golden_higher.json).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

import ref as R  # noqa: E402
from paper_2212_08284_b200 import inputs  # noqa: E402

# (name, generator, n or config, box radius, seed, multipoles, config kwargs)
SMALL_CASES = [
    ("rand_mp_L4_E2_p15", 300, 5.0, 1, True, dict(order_cheb=4, order_equi=4, depth=2, p=15)),
    ("rand_mp_L3_E2_open", 300, 5.0, 2, True, dict(order_cheb=3, order_equi=3, depth=2, p=0)),
    ("rand_q_L5_E1_p2", 500, 7.0, 3, False, dict(order_cheb=5, order_equi=5, depth=1, p=2)),
    ("rand_mp_L6_E2_p15", 400, 7.0, 4, True, dict(order_cheb=6, order_equi=6, depth=2, p=15)),
    ("rand_mp_L4_E3_p15", 2000, 9.0, 5, True, dict(order_cheb=4, order_equi=4, depth=3, p=15)),
    ("rand_q_L2_E1_open", 64, 3.0, 6, False, dict(order_cheb=2, order_equi=2, depth=1, p=0)),
    ("rand_mp_L5_E3_open", 1500, 8.0, 7, True, dict(order_cheb=5, order_equi=5, depth=3, p=0)),
    ("rand_mp_L4_E2_xi0.3", 400, 4.0, 8, True, dict(order_cheb=4, order_equi=4, depth=2, p=3, xi=0.3)),
]


# orders above 7: block-per-leaf P2M, large M2L rank classes, randomized SVD
HIGH_CASES = [
    ("rand_mp_L8_E2_p15", 600, 5.0, 21, True, dict(order_cheb=8, order_equi=8, depth=2, p=15)),
    ("rand_mp_L9_E2_p15", 500, 5.0, 22, True, dict(order_cheb=9, order_equi=9, depth=2, p=15)),
    ("rand_mp_L10_E1_p2", 300, 4.0, 23, True, dict(order_cheb=10, order_equi=10, depth=1, p=2)),
    ("rand_mp_L8_E2_open", 600, 5.0, 24, True, dict(order_cheb=8, order_equi=8, depth=2, p=0)),
]


# orders past the compiled kernels (11 .. 64: runtime-order P2M / M2M, host
# randomized SVD, the periodic term in a global scratch from L = 15)
HIGHER_CASES = [
    ("rand_mp_L11_E2_p15", 300, 5.0, 31, True, dict(order_cheb=11, order_equi=11, depth=2, p=15)),
    ("rand_mp_L12_E1_p2", 250, 4.0, 32, True, dict(order_cheb=12, order_equi=12, depth=1, p=2)),
    ("rand_q_L13_E2_open", 400, 5.0, 33, False, dict(order_cheb=13, order_equi=13, depth=2, p=0)),
    ("rand_mp_L16_E1_p15", 200, 4.0, 34, True, dict(order_cheb=16, order_equi=16, depth=1, p=15)),
]


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def energies(rep):
    return {k: repr(float(rep[k])) for k in ("e_total", "e_self", "e_near", "e_far", "e_periodic_far")}


def kats():
    out = {}
    out["erfc_screen"] = {repr(z): repr(R.erfc_screen(z)) for z in
                          (0.0, 0.01, 0.02, 0.1, 0.27, 0.5, 0.5000001, 0.75, 1.5, 4.0)}
    rng = np.random.default_rng(99)
    pairs = []
    for i in range(12):
        xa = rng.uniform(-3, 3, 3)
        xb = rng.uniform(-3, 3, 3)
        sa = np.concatenate([[rng.uniform(-1, 1)], rng.normal(0, 0.2, 3), rng.normal(0, 0.1, 6)])
        sb = np.concatenate([[rng.uniform(-1, 1)], rng.normal(0, 0.2, 3), rng.normal(0, 0.1, 6)])
        if i % 4 == 0:
            sa[1:] = 0.0
        if i % 3 == 0:
            sb[4:] = 0.0
        xi = [0.01, 0.1, 0.3][i % 3]
        e = R.pair_interaction(xa, sa, xb, sb, xi)
        pairs.append({"xa": xa.tolist(), "sa": sa.tolist(), "xb": xb.tolist(), "sb": sb.tolist(),
                      "xi": xi, "e": repr(e)})
    out["pair_interaction"] = pairs
    src = np.concatenate([[1.0], np.zeros(9)])[None, :]
    out["self_energy_q1_xi0.01"] = repr(R.self_energy(src, 0.01))
    src = np.array([[0.0, 1.0, 0, 0] + [0.0] * 6])
    out["self_energy_mu100_xi1"] = repr(R.self_energy(src, 1.0))
    out["default_depth"] = {str(n): R.default_depth(n) for n in
                            (0, 1, 64, 65, 512, 513, 3000, 24000, 96000, 1029000, 8232000)}
    lam, nb = R.list_sizes(2, False, 2)
    out["lambda_open_E2_level2"] = lam.tolist()
    out["neighbors_open_E2"] = nb.tolist()
    lam, nb = R.list_sizes(3, True, 3)
    out["lambda_periodic_E3_level3_unique"] = sorted(set(lam.tolist()))
    out["neighbors_periodic_E3_unique"] = sorted(set(nb.tolist()))
    lam, _ = R.list_sizes(2, False, 1)
    out["lambda_open_E2_level1"] = lam.tolist()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--high", action="store_true", help="orders 8-10 only -> golden_high.json")
    ap.add_argument("--higher", action="store_true", help="orders 11-16 only -> golden_higher.json")
    ap.add_argument("--series", action="store_true",
                    help="with --config 4: all evaluations of the rescale series -> golden_c4_series.json")
    ap.add_argument("--config", type=int, default=None,
                    help="only BASELINE config 3 or 4 (config 4: evaluation 0 of the rescale series)")
    args = ap.parse_args()
    threads = os.cpu_count() or 1
    if args.config == 4 and args.series:
        pos, src0, rb, c = inputs.make_config(4)
        L = c.orders[0]
        facs = inputs.rescale_factors(c.seed, c.evaluations)
        out = {"generator": "tests/golden/make_golden.py --config 4 --series",
               "reference": "oracle/_ref/libankh_ref.so", "n": pos.shape[0], "box_radius": rb,
               "seed": c.seed, "config": dict(order_cheb=L, order_equi=L),
               "sha256_positions": sha(pos), "sha256_sources": sha(src0), "evaluations": []}
        path = os.path.join(HERE, "golden_c4_series.json")
        for k, f in enumerate(facs):
            src = src0.copy()
            src[:, 1:4] *= float(f)
            rep = R.fmm_energy(pos, src, rb, order_cheb=L, order_equi=L, threads=threads)
            out["evaluations"].append({"index": k, "dipole_scale": float(f), "energies": energies(rep),
                                       "ref_wall_total": rep["wall_times"]["total"]})
            with open(path, "w") as fh:  # written as it goes (long run)
                json.dump(out, fh, indent=1)
            print(k, float(f), out["evaluations"][-1]["energies"]["e_total"], flush=True)
        return
    if args.config is not None:
        pos, src, rb, c = inputs.make_config(args.config)
        L = c.orders[0]
        scale = 1.0
        if args.config == 4:
            scale = float(inputs.rescale_factors(c.seed, c.evaluations)[0])
            src = src.copy()
            src[:, 1:4] *= scale
        rep = R.fmm_energy(pos, src, rb, order_cheb=L, order_equi=L, threads=threads)
        doc = {"generator": "tests/golden/make_golden.py --config %d" % args.config,
               "reference": "oracle/_ref/libankh_ref.so",
               "system": {"name": f"{c.name}_L{L}", "config_index": args.config, "n": pos.shape[0],
                          "box_radius": rb, "seed": c.seed, "dipole_scale": scale,
                          "config": dict(order_cheb=L, order_equi=L), "sha256": sha(pos, src),
                          "energies": energies(rep), "ref_wall_times": rep["wall_times"],
                          "ref_threads": threads}}
        with open(os.path.join(HERE, f"golden_c{args.config}.json"), "w") as f:
            json.dump(doc, f, indent=1)
        print(c.name, doc["system"]["energies"]["e_total"], rep["wall_times"], flush=True)
        return
    doc = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref/libankh_ref.so",
           "kats": kats(), "systems": []}
    if args.high or args.higher:
        doc = {"generator": "tests/golden/make_golden.py --high" + ("er" if args.higher else ""),
               "reference": "oracle/_ref/libankh_ref.so", "systems": []}
    cases = HIGHER_CASES if args.higher else (HIGH_CASES if args.high else SMALL_CASES)
    for name, n, rb, seed, mp, kw in cases:
        pos, src = inputs.random_system(n, rb, seed=seed, multipoles=mp)
        rep = R.fmm_energy(pos, src, rb, threads=threads, **kw)
        depth = kw["depth"]
        offs, idx = R.leaf_csr(pos, rb, depth)
        doc["systems"].append({
            "name": name, "kind": "random", "n": n, "box_radius": rb, "seed": seed,
            "multipoles": mp, "config": kw, "sha256": sha(pos, src), "energies": energies(rep),
            "leaf_csr_sha256": hashlib.sha256(offs.tobytes() + idx.tobytes()).hexdigest(),
        })
        print(name, doc["systems"][-1]["energies"]["e_total"], flush=True)
    cfgs = [] if (args.high or args.higher) else [(0, 4)]
    if args.big:
        cfgs += [(1, 4), (2, 3), (2, 4), (2, 5), (2, 6)]
    for ci, L in cfgs:
        pos, src, rb, c = inputs.make_config(ci)
        rep = R.fmm_energy(pos, src, rb, order_cheb=L, order_equi=L, threads=threads)
        depth = R.default_depth(pos.shape[0])
        offs, idx = R.leaf_csr(pos, rb, depth)
        doc["systems"].append({
            "name": f"{c.name}_L{L}", "kind": "config", "config_index": ci, "n": pos.shape[0],
            "box_radius": rb, "seed": c.seed, "config": dict(order_cheb=L, order_equi=L),
            "sha256": sha(pos, src), "energies": energies(rep),
            "leaf_csr_sha256": hashlib.sha256(offs.tobytes() + idx.tobytes()).hexdigest(),
            "ref_wall_times": rep["wall_times"], "ref_threads": threads,
        })
        print(c.name, L, doc["systems"][-1]["energies"]["e_total"], rep["wall_times"]["total"], flush=True)
    name = ("golden_higher.json" if args.higher else "golden_high.json" if args.high else
            ("golden_big.json" if args.big else "golden.json"))
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", name)


if __name__ == "__main__":
    main()
