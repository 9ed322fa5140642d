"""Per-component relative errors of the GPU engine against every golden case
(the reference's own energies): the margins behind the parity gates."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2212_08284_b200 as ankh  # noqa: E402
from paper_2212_08284_b200 import inputs  # noqa: E402


def main():
    rows = []
    for name in ("golden.json", "golden_big.json", "golden_high.json"):
        with open(os.path.join(ROOT, "tests", "golden", name)) as f:
            d = json.load(f)
        for case in d["systems"]:
            if case["kind"] == "random":
                pos, src = inputs.random_system(case["n"], case["box_radius"], seed=case["seed"],
                                                multipoles=case["multipoles"])
                rb = case["box_radius"]
            else:
                pos, src, rb, _ = inputs.make_config(case["config_index"])
            rep = ankh.fmm_energy(ankh.ParticleSystem(pos, src, rb), ankh.EwaldConfig(**case["config"]))
            w = {k: float(v) for k, v in case["energies"].items()}
            errs = {k: abs(getattr(rep, k) - w[k]) / max(abs(w[k]), 1e-300)
                    for k in ("e_total", "e_near", "e_far", "e_self", "e_periodic_far")}
            net_q = float(np.sum(src[:, 0]))
            rows.append((name, case["name"], net_q, w["e_periodic_far"], w["e_total"], errs))
            print(f"{name:18s} {case['name']:24s} netq {net_q:+.3e} e_per {w['e_periodic_far']:+.3e} "
                  + " ".join(f"{k[2:]}={v:.1e}" for k, v in errs.items()), flush=True)


if __name__ == "__main__":
    main()
