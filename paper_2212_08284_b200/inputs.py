"""Synthetic water-like particle systems and the SPEC particle-file format.

These stand in for the paper's Tinker-HP inputs, which are
not available here; the recipe follows BASELINE.json ``configs`` with the open
choices pinned in SURVEY.md §8d / Appendix C:

* O sites on an m^3 lattice (m = ceil(M^(1/3)), spacing a = side/m, site
  centres -r_B + a(i + 1/2)); when M < m^3 (config 2) a seeded uniform random
  subset of the sites is occupied;
* uniform +-0.3 A jitter of each O coordinate;
* a uniformly random rotation per molecule (normalised 4-D Gaussian quaternion);
* H = O + R (+-0.9572 sin(52.26 deg), 0, 0.9572 cos(52.26 deg));
* every atom wrapped into [-r_B, r_B);
* charges O -0.834, H +0.417; configs 1-4 add mu ~ N(0, 0.1^2) per component
  and Theta from 6 upper-triangle N(0, 0.05^2) draws, mirrored, trace removed;
* seeds 1000 + config index; config 4's per-evaluation dipole rescale factors
  are U[0.9, 1.1] from an independent stream of the same seed.

Arrays use the reference's byte layout (types.hpp:13-94): positions N x 3
(x, y, z) and sources N x 10 (q, mu_x, mu_y, mu_z, Theta_xx, xy, xz, yy, yz, zz),
both float64 C-contiguous -- exactly ``std::vector<Vec3>`` /
``std::vector<MultipoleSource>`` storage.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "WaterConfig",
    "CONFIGS",
    "make_water_box",
    "make_config",
    "rescale_factors",
    "random_system",
    "write_particle_file",
    "read_particle_file",
]


@dataclasses.dataclass(frozen=True)
class WaterConfig:
    name: str
    molecules: int
    side: float
    orders: Tuple[int, ...]
    multipoles: bool
    seed: int
    evaluations: int = 1

    @property
    def atoms(self) -> int:
        return 3 * self.molecules

    @property
    def box_radius(self) -> float:
        return self.side / 2.0


# BASELINE.json configs[0..4]
CONFIGS: List[WaterConfig] = [
    WaterConfig("c0", 1_000, 31.0, (4,), False, 1000),
    WaterConfig("c1", 8_000, 62.1, (4,), True, 1001),
    WaterConfig("c2", 32_000, 98.6, (3, 4, 5, 6), True, 1002),
    WaterConfig("c3", 343_000, 217.6, (5,), True, 1003),
    WaterConfig("c4", 2_744_000, 435.2, (5,), True, 1004, evaluations=20),
]

_OH = 0.9572
_HALF_ANGLE = math.radians(104.52 / 2.0)
_Q_O = -0.834
_Q_H = 0.417


def _rotations(quat: np.ndarray) -> np.ndarray:
    q = quat / np.linalg.norm(quat, axis=1, keepdims=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    r = np.empty((q.shape[0], 3, 3))
    r[:, 0, 0] = 1 - 2 * (y * y + z * z)
    r[:, 0, 1] = 2 * (x * y - w * z)
    r[:, 0, 2] = 2 * (x * z + w * y)
    r[:, 1, 0] = 2 * (x * y + w * z)
    r[:, 1, 1] = 1 - 2 * (x * x + z * z)
    r[:, 1, 2] = 2 * (y * z - w * x)
    r[:, 2, 0] = 2 * (x * z - w * y)
    r[:, 2, 1] = 2 * (y * z + w * x)
    r[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def _wrap(x: np.ndarray, r_b: float) -> np.ndarray:
    y = np.mod(x + r_b, 2.0 * r_b) - r_b
    # guard the half-open upper edge against round-off
    y = np.where(y >= r_b, y - 2.0 * r_b, y)
    return np.where(y < -r_b, -r_b, y)


def make_water_box(molecules: int, side: float, seed: int, multipoles: bool) -> Tuple[np.ndarray, np.ndarray, float]:
    """Return (positions N x 3, sources N x 10, box_radius) for N = 3*molecules."""
    rng = np.random.default_rng(seed)
    r_b = side / 2.0
    m = int(math.ceil(round(molecules ** (1.0 / 3.0), 9)))
    while m ** 3 < molecules:
        m += 1
    a = side / m
    sites = m ** 3
    if molecules < sites:
        chosen = np.sort(rng.choice(sites, size=molecules, replace=False))
    else:
        chosen = np.arange(sites)
    i, rem = np.divmod(chosen, m * m)
    j, k = np.divmod(rem, m)
    o = np.stack([-r_b + a * (i + 0.5), -r_b + a * (j + 0.5), -r_b + a * (k + 0.5)], axis=1)
    o = o + rng.uniform(-0.3, 0.3, size=o.shape)
    rot = _rotations(rng.standard_normal((molecules, 4)))
    sx, cz = _OH * math.sin(_HALF_ANGLE), _OH * math.cos(_HALF_ANGLE)
    h1 = o + rot @ np.array([sx, 0.0, cz])
    h2 = o + rot @ np.array([-sx, 0.0, cz])
    pos = np.empty((3 * molecules, 3))
    pos[0::3], pos[1::3], pos[2::3] = o, h1, h2
    pos = _wrap(pos, r_b)
    n = 3 * molecules
    src = np.zeros((n, 10))
    src[0::3, 0] = _Q_O
    src[1::3, 0] = _Q_H
    src[2::3, 0] = _Q_H
    if multipoles:
        src[:, 1:4] = rng.normal(0.0, 0.1, size=(n, 3))
        up = rng.normal(0.0, 0.05, size=(n, 6))  # xx, xy, xz, yy, yz, zz
        tr3 = (up[:, 0] + up[:, 3] + up[:, 5]) / 3.0
        up[:, 0] -= tr3
        up[:, 3] -= tr3
        up[:, 5] -= tr3
        src[:, 4:10] = up
    return np.ascontiguousarray(pos), np.ascontiguousarray(src), r_b


def make_config(index: int) -> Tuple[np.ndarray, np.ndarray, float, WaterConfig]:
    cfg = CONFIGS[index]
    pos, src, r_b = make_water_box(cfg.molecules, cfg.side, cfg.seed, cfg.multipoles)
    return pos, src, r_b, cfg


def rescale_factors(seed: int, count: int) -> np.ndarray:
    """Config 4's per-evaluation dipole scale factors f_e ~ U[0.9, 1.1]."""
    return np.random.default_rng([seed, 1]).uniform(0.9, 1.1, size=count)


def random_system(n: int, box_radius: float, seed: int, multipoles: bool = True,
                  charge_scale: float = 1.0, neutral: bool = True) -> Tuple[np.ndarray, np.ndarray]:
    """Uniform random particles in [-r_B, r_B)^3 (for small parity cases)."""
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-box_radius, box_radius, size=(n, 3))
    src = np.zeros((n, 10))
    q = rng.uniform(-1.0, 1.0, size=n) * charge_scale
    if neutral and n > 1:
        q -= q.mean()
    src[:, 0] = q
    if multipoles:
        src[:, 1:4] = rng.normal(0.0, 0.1, size=(n, 3))
        src[:, 4:10] = rng.normal(0.0, 0.05, size=(n, 6))
    return np.ascontiguousarray(pos), np.ascontiguousarray(src)


def write_particle_file(path: str, positions: np.ndarray, sources: np.ndarray, box_radius: float,
                        comment: Optional[str] = None) -> None:
    """SPEC particle file: '#' comments, 'N r_B', then N rows of 13
    numbers x y z q mux muy muz Txx Txy Txz Tyy Tyz Tzz, printed with %.17g."""
    n = positions.shape[0]
    with open(path, "w") as f:
        if comment:
            for line in comment.splitlines():
                f.write(f"# {line}\n")
        f.write(f"{n} {box_radius:.17g}\n")
        rows = np.concatenate([positions, sources], axis=1)
        np.savetxt(f, rows, fmt="%.17g")


class ParticleFileError(ValueError):
    """Malformed particle file (SPEC ParticleFile invariants); names the line."""


def read_particle_file(path: str) -> Tuple[np.ndarray, np.ndarray, float]:
    """Parse a SPEC particle file: '#' comment lines, 'N r_B', then exactly N
    rows of 13 finite decimals.  Errors name the 1-based file line."""
    header = None
    rows = []
    with open(path) as f:
        for lineno, ln in enumerate(f, start=1):
            s = ln.strip()
            if not s or s.startswith("#"):
                continue
            toks = s.split()
            if header is None:
                if len(toks) != 2:
                    raise ParticleFileError(f"line {lineno}: header must be 'N r_B', got {len(toks)} values")
                try:
                    header = (int(toks[0]), float(toks[1]))
                except ValueError:
                    raise ParticleFileError(f"line {lineno}: header must be 'N r_B'") from None
                if header[0] < 0 or not np.isfinite(header[1]):
                    raise ParticleFileError(f"line {lineno}: invalid header values")
                continue
            if len(toks) != 13:
                raise ParticleFileError(f"line {lineno}: expected 13 values, got {len(toks)}")
            try:
                vals = [float(t) for t in toks]
            except ValueError:
                raise ParticleFileError(f"line {lineno}: not a decimal number") from None
            if not all(np.isfinite(vals)):
                raise ParticleFileError(f"line {lineno}: non-finite value")
            rows.append(vals)
    if header is None:
        raise ParticleFileError("missing header line 'N r_B'")
    n, r_b = header
    if len(rows) != n:
        raise ParticleFileError(f"header says {n} rows, found {len(rows)}")
    arr = np.asarray(rows, dtype=np.float64).reshape(n, 13)
    return np.ascontiguousarray(arr[:, :3]), np.ascontiguousarray(arr[:, 3:]), r_b
