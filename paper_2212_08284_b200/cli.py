"""Command-line front end (SPEC.md `cli` module):

    python -m paper_2212_08284_b200 energy  --input sys.txt [--order-cheb 5 ...] [--output out.json]
    python -m paper_2212_08284_b200 compare --input sys.txt --runs fmm:order_cheb=8 fmm:order_cheb=4 ...
    python -m paper_2212_08284_b200 gen     --kind uniform|lattice-jittered --n N --box-radius R ...
    python -m paper_2212_08284_b200 gen     --config 3 --output c3.txt
    python -m paper_2212_08284_b200 bench   --sizes 3000,24000,192000 [--order-cheb 5]

`energy` runs the B200 `fmm_energy` (`--method fmm`, the reference's engine;
SPEC's fft / direct / ewald engines are absent from the reference and are
rejected with exit code 3 -- the GPU direct lattice sum used to check the FMM's
accuracy is test infrastructure, oracle/direct.py).  Documents are JSON with every float printed
round-trip exact (>= 17 significant digits where needed), holding the run
manifest and the EnergyReport, so `load_document` restores both without loss.

Exit codes (SPEC: stable contract for harnesses): 0 success, 2 parse error
(particle file / manifest), 3 configuration or invariant violation (the
reference's invalid_argument / domain_error), 4 budget guard (--max-atoms),
1 any other failure (e.g. CUDA).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time
from typing import Dict, List, Optional

import numpy as np

from . import api, inputs

EXIT_OK, EXIT_OTHER, EXIT_PARSE, EXIT_CONFIG, EXIT_BUDGET = 0, 1, 2, 3, 4
# SPEC methods fmm | fft | direct | ewald: the reference implements fmm only
METHODS = ("fmm",)
CONFIG_FIELDS = ("xi", "p", "order_cheb", "order_equi", "depth", "svd_tol", "recip_cutoff")


class CliError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


@dataclasses.dataclass
class RunManifest:
    """SPEC RunManifest: method, EwaldConfig fields, input/output paths, seed, threads."""

    method: str = "fmm"
    config: Dict[str, float] = dataclasses.field(default_factory=dict)
    input: Optional[str] = None
    output: Optional[str] = None
    seed: Optional[int] = None
    threads: int = 0

    def ewald(self) -> api.EwaldConfig:
        return api.EwaldConfig(**self.config)

    def validate(self) -> None:
        if self.method not in METHODS:
            raise CliError(EXIT_CONFIG, f"method '{self.method}' is not available (methods: "
                                        f"{', '.join(METHODS)}; SPEC's fft / ewald engines are "
                                        f"absent from the reference)")
        unknown = set(self.config) - set(CONFIG_FIELDS)
        if unknown:
            raise CliError(EXIT_PARSE, f"unknown config fields: {sorted(unknown)}")


def _config_from_args(a) -> Dict[str, float]:
    cfg = {}
    for f in CONFIG_FIELDS:
        v = getattr(a, f, None)
        if v is not None:
            cfg[f] = v
    if "order_cheb" in cfg and "order_equi" not in cfg:
        cfg["order_equi"] = cfg["order_cheb"]
    return cfg


def _parse_run(spec: str) -> RunManifest:
    """'fmm:order_cheb=8,xi=0.01' -> RunManifest."""
    method, _, rest = spec.partition(":")
    cfg: Dict[str, float] = {}
    for item in filter(None, rest.split(",")):
        k, eq, v = item.partition("=")
        if not eq or k not in CONFIG_FIELDS:
            raise CliError(EXIT_PARSE, f"bad run spec item '{item}' in '{spec}'")
        try:
            cfg[k] = float(v) if k in ("xi", "svd_tol") else int(v)
        except ValueError:
            raise CliError(EXIT_PARSE, f"bad value in '{item}'") from None
    if "order_cheb" in cfg and "order_equi" not in cfg:
        cfg["order_equi"] = cfg["order_cheb"]
    m = RunManifest(method=method, config=cfg)
    m.validate()
    return m


def _read_system(path: str, max_atoms: Optional[int]) -> api.ParticleSystem:
    try:
        pos, src, rb = inputs.read_particle_file(path)
    except (OSError, inputs.ParticleFileError) as e:
        raise CliError(EXIT_PARSE, f"{path}: {e}") from None
    if max_atoms is not None and pos.shape[0] > max_atoms:
        raise CliError(EXIT_BUDGET, f"{path}: {pos.shape[0]} atoms exceed --max-atoms {max_atoms}")
    return api.ParticleSystem(pos, src, rb)


def _run(system: api.ParticleSystem, m: RunManifest) -> api.EnergyReport:
    try:
        return api.fmm_energy(system, m.ewald(), threads=m.threads)
    except (api.InvalidArgument, api.DomainError) as e:
        raise CliError(EXIT_CONFIG, str(e)) from None


def report_dict(r: api.EnergyReport) -> dict:
    return dataclasses.asdict(r)


def document(m: RunManifest, r: api.EnergyReport, extra: Optional[dict] = None) -> dict:
    d = {"manifest": dataclasses.asdict(m), "report": report_dict(r)}
    if extra:
        d.update(extra)
    return d


def load_document(text: str):
    """Inverse of the `energy` output: (RunManifest, EnergyReport)."""
    d = json.loads(text)
    return RunManifest(**d["manifest"]), api.EnergyReport(**d["report"])


def _emit(obj, path: Optional[str]) -> None:
    text = json.dumps(obj, indent=1)  # repr floats: shortest round-trip form
    if path:
        with open(path, "w") as f:
            f.write(text + "\n")
    else:
        print(text)


# ---------------------------------------------------------------------------
def cmd_energy(a) -> int:
    m = RunManifest(method=a.method, config=_config_from_args(a), input=a.input, output=a.output,
                    seed=None, threads=a.threads)
    if a.manifest:
        try:
            with open(a.manifest) as f:
                m = RunManifest(**json.load(f))
        except (OSError, TypeError, ValueError) as e:
            raise CliError(EXIT_PARSE, f"manifest {a.manifest}: {e}") from None
        m.input = m.input or a.input
        m.output = a.output or m.output
    m.validate()
    if not m.input:
        raise CliError(EXIT_PARSE, "energy: --input is required")
    system = _read_system(m.input, a.max_atoms)
    r = _run(system, m)
    _emit(document(m, r, {"atoms": system.size()}), m.output)
    return EXIT_OK


def cmd_compare(a) -> int:
    runs = [_parse_run(s) for s in a.runs]
    if len(runs) < 2:
        raise CliError(EXIT_PARSE, "compare: at least two runs are required (reference first)")
    system = _read_system(a.input, a.max_atoms)
    rows = []
    ref = None
    for m in runs:
        m.input, m.threads = a.input, a.threads
        r = _run(system, m)
        if ref is None:
            ref = r.e_total
        rows.append({"run": m.method + ":" + ",".join(f"{k}={v}" for k, v in m.config.items()),
                     "e_total": r.e_total,
                     "r": abs(ref - r.e_total) / abs(ref) if ref != 0 else abs(r.e_total),
                     "wall_times": r.wall_times})
    _emit({"input": a.input, "reference": rows[0]["run"], "rows": rows}, a.output)
    return EXIT_OK


def gen_system(kind: str, n: int, box_radius: float, seed: int, moments: str):
    """SPEC cmd_gen: reproducible from the seed; optional moments with
    |mu|, |Theta| <= 0.1 |q| (`uniform`), or a jittered water lattice
    (`lattice-jittered`, n divisible by 3; same generator as the BASELINE
    configs) / jittered point lattice otherwise."""
    if n < 1:
        raise CliError(EXIT_CONFIG, "gen: N must be >= 1")
    if not (box_radius > 0 and np.isfinite(box_radius)):
        raise CliError(EXIT_CONFIG, "gen: box radius must be finite and > 0")
    rng = np.random.default_rng([seed, n])
    if kind == "lattice-jittered" and n % 3 == 0:
        pos, src, rb = inputs.make_water_box(n // 3, 2.0 * box_radius, seed, moments != "none")
        return pos, src, rb
    if kind == "lattice-jittered":
        m = int(np.ceil(n ** (1.0 / 3.0) - 1e-9))
        a = 2.0 * box_radius / m
        sites = rng.choice(m ** 3, size=n, replace=False)
        idx = np.stack(np.unravel_index(np.sort(sites), (m, m, m)), axis=1).astype(np.float64)
        pos = -box_radius + a * (idx + 0.5) + rng.uniform(-0.15 * a, 0.15 * a, size=(n, 3))
    elif kind == "uniform":
        pos = rng.uniform(-box_radius, box_radius, size=(n, 3))
    else:
        raise CliError(EXIT_PARSE, f"gen: unknown kind '{kind}'")
    pos = np.clip(pos, -box_radius, np.nextafter(box_radius, 0.0))
    src = np.zeros((n, 10))
    q = rng.choice([-1.0, 1.0], size=n) * rng.uniform(0.5, 1.0, size=n)
    src[:, 0] = q
    if moments in ("dipoles", "full"):
        lim = 0.1 * np.abs(q)[:, None] / np.sqrt(3.0)
        src[:, 1:4] = rng.uniform(-1.0, 1.0, size=(n, 3)) * lim
    if moments == "full":
        lim = 0.1 * np.abs(q)[:, None] / 3.0
        src[:, 4:10] = rng.uniform(-1.0, 1.0, size=(n, 6)) * lim
    return np.ascontiguousarray(pos), np.ascontiguousarray(src), box_radius


def cmd_gen(a) -> int:
    if a.config is not None:
        pos, src, rb, cfg = inputs.make_config(a.config)
        comment = f"BASELINE config {a.config}: {cfg}"
    else:
        if a.n is None or a.box_radius is None:
            raise CliError(EXIT_PARSE, "gen: --n and --box-radius (or --config) are required")
        pos, src, rb = gen_system(a.kind, a.n, a.box_radius, a.seed, a.moments)
        comment = f"gen kind={a.kind} n={a.n} box_radius={a.box_radius!r} seed={a.seed} moments={a.moments}"
    if not a.output:
        raise CliError(EXIT_PARSE, "gen: --output is required")
    inputs.write_particle_file(a.output, pos, src, rb, comment=comment)
    return EXIT_OK


def cmd_bench(a) -> int:
    """Per-phase times vs N (water boxes at liquid density); precompute (the
    plan build) reported separately from the evaluation, as SPEC asks."""
    try:
        sizes = [int(s) for s in a.sizes.split(",")]
    except ValueError:
        raise CliError(EXIT_PARSE, f"bench: bad --sizes '{a.sizes}'") from None
    if sizes != sorted(sizes):
        raise CliError(EXIT_CONFIG, "bench: sizes must be sorted ascending")
    cfg = api.EwaldConfig(**_config_from_args(a))
    rows = []
    for n in sizes:
        molecules = max(1, n // 3)
        side = (molecules / 0.033428) ** (1.0 / 3.0)  # liquid water, molecules per A^3
        pos, src, rb = inputs.make_water_box(molecules, side, a.seed, True)
        t0 = time.perf_counter()
        plan = api.Plan(pos.shape[0], rb, cfg, threads=a.threads, phase_timing=True)
        build = time.perf_counter() - t0
        reps = []
        for _ in range(max(2, a.repeat + 1)):
            reps.append(plan.energy(pos, src))
        r = reps[-1]
        wt = {k: float(np.median([x.wall_times[k] for x in reps[1:]])) for k in r.wall_times}
        plan.close()
        rows.append({"atoms": int(pos.shape[0]), "depth": r.depth, "order_cheb": r.order_cheb,
                     "plan_build_s": build, **{f"t_{k}": v for k, v in wt.items()},
                     "evals_per_s": 1.0 / wt["total"] if wt["total"] > 0 else None,
                     "e_total": r.e_total})
    if a.format == "table":
        cols = ["atoms", "depth", "plan_build_s", "t_precompute", "t_interpolation", "t_far_field",
                "t_near_field", "t_periodic_far", "t_self", "t_total", "evals_per_s"]
        print(" ".join(f"{c:>15}" for c in cols))
        for row in rows:
            print(" ".join(f"{row[c]:>15.6g}" if isinstance(row[c], float) else f"{row[c]:>15}"
                           for c in cols))
    else:
        _emit({"rows": rows}, a.output)
    return EXIT_OK


# ---------------------------------------------------------------------------
def _add_config(p) -> None:
    p.add_argument("--method", default="fmm")
    p.add_argument("--xi", type=float)
    p.add_argument("--images", "-p", dest="p", type=int)
    p.add_argument("--order-cheb", dest="order_cheb", type=int)
    p.add_argument("--order-equi", dest="order_equi", type=int)
    p.add_argument("--depth", type=int)
    p.add_argument("--svd-tol", dest="svd_tol", type=float)
    p.add_argument("--recip-cutoff", dest="recip_cutoff", type=int)
    p.add_argument("--threads", type=int, default=int(os.environ.get("ANKH_THREADS", "0")))
    p.add_argument("--max-atoms", dest="max_atoms", type=int, default=None,
                   help="budget guard: refuse larger inputs (exit 4)")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2212_08284_b200",
                                 description="ANKH-FMM periodic multipole energy on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("energy", help="energy of one particle file")
    _add_config(p)
    p.add_argument("--input", "-i")
    p.add_argument("--output", "-o")
    p.add_argument("--manifest", help="RunManifest JSON (flags fill missing input/output)")
    p.set_defaults(fn=cmd_energy)
    p = sub.add_parser("compare", help="several runs on one file; r = |E_ref - E| / |E_ref|")
    _add_config(p)
    p.add_argument("--input", "-i", required=True)
    p.add_argument("--output", "-o")
    p.add_argument("--runs", nargs="+", required=True,
                   help="method[:field=value,...]; the first run is the reference")
    p.set_defaults(fn=cmd_compare)
    p = sub.add_parser("gen", help="write a particle file")
    p.add_argument("--kind", default="uniform", choices=["uniform", "lattice-jittered"])
    p.add_argument("--n", type=int)
    p.add_argument("--box-radius", dest="box_radius", type=float)
    p.add_argument("--moments", default="full", choices=["none", "dipoles", "full"])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--config", type=int, choices=range(5), help="BASELINE config system instead")
    p.add_argument("--output", "-o")
    p.set_defaults(fn=cmd_gen)
    p = sub.add_parser("bench", help="per-phase timing table vs N")
    _add_config(p)
    p.add_argument("--sizes", required=True, help="comma-separated atom counts, ascending")
    p.add_argument("--repeat", type=int, default=3)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--format", default="table", choices=["table", "json"])
    p.add_argument("--output", "-o")
    p.set_defaults(fn=cmd_bench)
    return ap


def main(argv: Optional[List[str]] = None) -> int:
    ap = build_parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # argparse usage errors
        return EXIT_PARSE if e.code else EXIT_OK
    try:
        return a.fn(a)
    except CliError as e:
        print(f"error: {e}", file=sys.stderr)
        return e.code
    except (api.InvalidArgument, api.DomainError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except Exception as e:  # CUDA / runtime failures
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return EXIT_OTHER
