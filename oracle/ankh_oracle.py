"""TEST INFRASTRUCTURE ONLY -- CPU restatement (numpy) of the reference's
``ankh::fmm_energy`` path, used as the parity CHECKER.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline
leg may import this module; the product (``paper_2212_08284_b200``) never does.

Every function names the reference lines it restates (paths relative to
/root/reference/proj/core).  Parity pin: this restatement is checked against
the reference itself -- the unmodified reference sources compiled against
oracle/shim into oracle/_ref/libankh_ref.so (see oracle/Makefile) -- in
tests/test_oracle.py, and against the golden vectors in tests/golden/ produced
by tests/golden/make_golden.py from that library.  Independent pieces: the SVD
and QR here are LAPACK (numpy), the FFT is pocketfft (numpy), the Gaussian
sketch uses a numpy MT19937-64.
"""
from __future__ import annotations

import math
from typing import Dict, List, Tuple

import numpy as np

try:  # accurate erfc for the z > 0.5 branch (kernel.cpp:48-51 uses std::erfc)
    from scipy.special import erfc as _erfc_vec
except Exception:  # pragma: no cover
    _erfc_vec = np.vectorize(math.erfc)

K_TWO_OVER_SQRT_PI = 1.1283791670955125739
K_INV_SQRT_PI = 0.5641895835477562869


class InvalidArgument(ValueError):
    pass


class DomainError(ArithmeticError):
    pass


# ----------------------------------------------------------------- types.cpp
def default_depth(n: int) -> int:
    """types.cpp:9-14."""
    if n <= 64:
        return 1
    levels = math.log(n / 64.0) / math.log(8.0)
    return max(1, int(math.ceil(levels - 1e-12)))


def validate_config(xi, p, order_cheb, order_equi, depth, svd_tol, recip_cutoff) -> None:
    """types.cpp:65-79 (same messages)."""
    if not (xi > 0.0) or not math.isfinite(xi):
        raise InvalidArgument("xi must be positive")
    if p < 0 or p == 1:
        raise InvalidArgument("image half-width p must be 0 (open) or >= 2 (periodic)")
    if order_cheb < 2:
        raise InvalidArgument("order_cheb must be >= 2")
    if order_equi < 2:
        raise InvalidArgument("order_equi must be >= 2")
    if depth < 0:
        raise InvalidArgument("depth must be >= 1 (or 0 for automatic)")
    if not (svd_tol > 0.0) or not (svd_tol < 1.0):
        raise InvalidArgument("svd_tol must lie in (0, 1)")
    if recip_cutoff < 1:
        raise InvalidArgument("recip_cutoff must be >= 1")


def validate_system(pos: np.ndarray, src: np.ndarray, r_b: float) -> List[Tuple[int, str]]:
    """types.cpp:16-63: violations in the reference's order."""
    out: List[Tuple[int, str]] = []
    if not (r_b > 0.0) or not math.isfinite(r_b):
        out.append((-1, "box_radius must be positive and finite"))
    if pos.shape[0] != src.shape[0]:
        out.append((-1, "positions and sources must have equal length"))
        return out
    finite = np.isfinite(pos).all(axis=1) & np.isfinite(src).all(axis=1)
    outside = (np.abs(pos) > r_b).any(axis=1)
    for i in np.nonzero(~finite | outside)[0]:
        out.append((int(i), "non-finite coordinate or moment" if not finite[i] else "outside box"))
    if pos.shape[0] > 1:
        order = np.lexsort((pos[:, 2], pos[:, 1], pos[:, 0]))
        sp = pos[order]
        dup = (sp[1:] == sp[:-1]).all(axis=1)
        for k in np.nonzero(dup)[0]:
            out.append((int(max(order[k], order[k + 1])), "duplicate position"))
    return out


# ---------------------------------------------------------------- kernel.cpp
def erfc_screen(z):
    """kernel.cpp:14-23 (13-term Maclaurin erf for 0 <= z <= 0.5) and 48-51."""
    z = np.asarray(z, dtype=np.float64)
    z2 = z * z
    term = z.copy()
    s = np.zeros_like(z)
    for n in range(13):
        s = s + term / (2 * n + 1)
        term = term * (-z2 / (n + 1))
    series = 1.0 - K_TWO_OVER_SQRT_PI * s
    small = (z >= 0.0) & (z <= 0.5)
    if small.all():
        return series
    return np.where(small, series, _erfc_vec(z))


def radial(r, xi, order):
    """kernel.cpp:26-38: b[0..order] (vectorised over r)."""
    z = xi * r
    b = [erfc_screen(z) / r]
    if order == 0:
        return b
    inv_r2 = 1.0 / (r * r)
    a = K_TWO_OVER_SQRT_PI * xi * np.exp(-z * z)
    two_xi2 = 2.0 * xi * xi
    for n in range(1, order + 1):
        b.append(((2 * n - 1) * b[n - 1] + a) * inv_r2)
        a = a * two_xi2
    return b


def _symmul(t, v):
    """SymMat3::mul (types.hpp:59-63); t[..., 6] = xx, xy, xz, yy, yz, zz."""
    return np.stack([
        t[..., 0] * v[..., 0] + t[..., 1] * v[..., 1] + t[..., 2] * v[..., 2],
        t[..., 1] * v[..., 0] + t[..., 3] * v[..., 1] + t[..., 4] * v[..., 2],
        t[..., 2] * v[..., 0] + t[..., 4] * v[..., 1] + t[..., 5] * v[..., 2],
    ], axis=-1)


def _contract(a, b):
    """SymMat3::contract (types.hpp:66-69)."""
    return (a[..., 0] * b[..., 0] + a[..., 3] * b[..., 3] + a[..., 5] * b[..., 5]
            + 2.0 * (a[..., 1] * b[..., 1] + a[..., 2] * b[..., 2] + a[..., 4] * b[..., 4]))


def pair_interaction(xa, sa, xb, sb, xi):
    """kernel.cpp:157-204, vectorised over pairs (rows).  Terms of order above
    moment_order(a)+moment_order(b) multiply exact zeros, so evaluating the full
    formula reproduces the early returns."""
    xa = np.atleast_2d(xa)
    xb = np.atleast_2d(xb)
    sa = np.atleast_2d(sa)
    sb = np.atleast_2d(sb)
    rv = xa - xb
    r2 = (rv * rv).sum(axis=1)
    if (r2 == 0.0).any():
        raise DomainError("pair_interaction: coincident points")
    r = np.sqrt(r2)
    charges_only = not (sa[:, 1:].any() or sb[:, 1:].any())
    b = radial(r, xi, 0 if charges_only else 4)
    qa, qb = sa[:, 0], sb[:, 0]
    e = qa * qb * b[0]
    if charges_only:
        return e
    mua, mub = sa[:, 1:4], sb[:, 1:4]
    ta, tb = sa[:, 4:10], sb[:, 4:10]
    F1, F2, F3, F4 = -b[1], b[2], -b[3], b[4]
    uar = (mua * rv).sum(axis=1)
    ubr = (mub * rv).sum(axis=1)
    tra = ta[:, 0] + ta[:, 3] + ta[:, 5]
    trb = tb[:, 0] + tb[:, 3] + tb[:, 5]
    e = e + (qb * uar - qa * ubr) * F1
    e = e + (qb * tra + qa * trb) * F1
    Qar = _symmul(ta, rv)
    Qbr = _symmul(tb, rv)
    raQar = (Qar * rv).sum(axis=1)
    rbQbr = (Qbr * rv).sum(axis=1)
    e = e + -((mua * mub).sum(axis=1) * F1 + uar * ubr * F2)
    e = e + (qb * raQar + qa * rbQbr) * F2
    e = e + (2.0 * (mua * Qbr).sum(axis=1) + uar * trb) * F2 + uar * rbQbr * F3
    e = e - ((2.0 * (mub * Qar).sum(axis=1) + ubr * tra) * F2 + ubr * raQar * F3)
    e = e + (tra * trb + 2.0 * _contract(ta, tb)) * F2
    e = e + (tra * rbQbr + trb * raQar + 4.0 * (Qar * Qbr).sum(axis=1)) * F3
    e = e + raQar * rbQbr * F4
    return e


def pair_gradient(xa, sa, xb, sb, xi):
    """Gradient of pair_interaction (kernel.cpp:157-204) with respect to
    r = xa - xb, moments held fixed: the near-field force on a is -grad.
    NOT a reference function (the reference computes energies only; forces
    are SURVEY.md §8f-3): the exact derivative of the same polynomial,
    e = sum_n C_n(r) b_n(r) with grad b_n = -r b_{n+1} (radial recurrence,
    kernel.cpp:26-38), checked against central differences of
    pair_interaction (tests/test_oracle.py)."""
    xa = np.atleast_2d(xa)
    xb = np.atleast_2d(xb)
    sa = np.atleast_2d(sa)
    sb = np.atleast_2d(sb)
    rv = xa - xb
    r2 = (rv * rv).sum(axis=1)
    if (r2 == 0.0).any():
        raise DomainError("pair_interaction: coincident points")
    r = np.sqrt(r2)
    b = radial(r, xi, 5)
    qa, qb = sa[:, 0], sb[:, 0]
    mua, mub = sa[:, 1:4], sb[:, 1:4]
    ta, tb = sa[:, 4:10], sb[:, 4:10]
    uar = (mua * rv).sum(axis=1)
    ubr = (mub * rv).sum(axis=1)
    tra = ta[:, 0] + ta[:, 3] + ta[:, 5]
    trb = tb[:, 0] + tb[:, 3] + tb[:, 5]
    Qar = _symmul(ta, rv)
    Qbr = _symmul(tb, rv)
    raQar = (Qar * rv).sum(axis=1)
    rbQbr = (Qbr * rv).sum(axis=1)
    dot = lambda u, v: (u * v).sum(axis=1)
    col = lambda s: s[:, None]
    # e = C0 b0 + C1 b1 + ... + C4 b4 (the reference's terms, F_n = (-1)^n b_n)
    C = [qa * qb,
         -(qb * uar - qa * ubr) - (qb * tra + qa * trb) + dot(mua, mub),
         (-uar * ubr + qb * raQar + qa * rbQbr + 2.0 * dot(mua, Qbr) + uar * trb
          - 2.0 * dot(mub, Qar) - ubr * tra + tra * trb + 2.0 * _contract(ta, tb)),
         -uar * rbQbr + ubr * raQar - (tra * rbQbr + trb * raQar + 4.0 * dot(Qar, Qbr)),
         raQar * rbQbr]
    taub = _symmul(ta, mub)
    tbua = _symmul(tb, mua)
    gC = [None,
          -(col(qb) * mua - col(qa) * mub),
          (-(col(ubr) * mua + col(uar) * mub) + 2.0 * col(qb) * Qar + 2.0 * col(qa) * Qbr
           + 2.0 * tbua + col(trb) * mua - 2.0 * taub - col(tra) * mub),
          (-(col(rbQbr) * mua + 2.0 * col(uar) * Qbr) + (col(raQar) * mub + 2.0 * col(ubr) * Qar)
           - (2.0 * col(tra) * Qbr + 2.0 * col(trb) * Qar
              + 4.0 * (_symmul(ta, Qbr) + _symmul(tb, Qar)))),
         2.0 * col(rbQbr) * Qar + 2.0 * col(raQar) * Qbr]
    g = -rv * col(sum(C[n] * b[n + 1] for n in range(5)))
    for n in range(1, 5):
        g = g + gC[n] * col(b[n])
    return g


def self_energy(src: np.ndarray, xi: float) -> float:
    """kernel.cpp:206-213."""
    if src.shape[0] == 0:
        return 0.0
    mu2 = (src[:, 1:4] ** 2).sum(axis=1)
    th = src[:, 4:10]
    acc = src[:, 0] ** 2 + (2.0 * xi * xi / 3.0) * mu2 + (8.0 * xi ** 4 / 5.0) * _contract(th, th)
    return float(-xi * K_INV_SQRT_PI * acc.sum())


# ------------------------------------------------------------- chebyshev.cpp
def cheb_nodes(order: int) -> np.ndarray:
    """Grid1D::chebyshev, chebyshev.cpp:48-58."""
    k = np.arange(order, dtype=np.float64)
    return np.cos((2.0 * k + 1.0) * math.pi / (2.0 * order))


def equi_nodes(order: int) -> np.ndarray:
    """Grid1D::equispaced, chebyshev.cpp:60-70."""
    return np.array([-1.0 + 2.0 * k / (order - 1.0) for k in range(order)])


def cheb_values(order: int, x) -> np.ndarray:
    """chebyshev.cpp:13-17: T_0..T_{L-1}(x), stacked on the last axis."""
    x = np.asarray(x, dtype=np.float64)
    t = [np.ones_like(x)]
    if order > 1:
        t.append(x.copy())
    for m in range(2, order):
        t.append(2.0 * x * t[m - 1] - t[m - 2])
    return np.stack(t, axis=-1)


def lagrange_eval_cheb(order: int, k: int, x: float) -> float:
    """chebyshev.cpp:72-83 (Chebyshev branch)."""
    t = cheb_values(order, x)
    tr = cheb_values(order, cheb_nodes(order)[k])
    s = 1.0
    for m in range(1, order):
        s += 2.0 * tr[m] * t[m]
    return s / order


def lagrange_eval_equi(order: int, k: int, x: float) -> float:
    """chebyshev.cpp:19-44 barycentric form with exact-node shortcut."""
    w = []
    b = 1.0
    for j in range(order):
        w.append(b if j % 2 == 0 else -b)
        b = b * (order - 1 - j) / (j + 1)
    nodes = equi_nodes(order)
    denom = 0.0
    for m in range(order):
        dx = x - nodes[m]
        if dx == 0.0:
            return 1.0 if m == k else 0.0
        denom += w[m] / dx
    return (w[k] / (x - nodes[k])) / denom


def diff_operator(order: int) -> List[np.ndarray]:
    """DiffOperator, chebyshev.cpp:85-108: [H, H D, H D D]."""
    if order < 2 or order > 64:
        raise InvalidArgument("DiffOperator: order out of range")
    nodes = cheb_nodes(order)
    h = np.empty((order, order))
    for k in range(order):
        t = cheb_values(order, nodes[k])
        h[k, 0] = 1.0 / order
        h[k, 1:] = 2.0 * t[1:] / order
    d = np.zeros((order, order))
    for m in range(1, order):
        for j in range(m - 1, -1, -2):
            d[m, j] = m if j == 0 else 2.0 * m
    hd1 = h @ d
    return [h, hd1, hd1 @ d]


def transfer_1d(dst_order: int, src_local, equispaced: bool = False) -> np.ndarray:
    """chebyshev.cpp:236-244: T(k, l) = S_k^{dst}(src_local[l])."""
    f = lagrange_eval_equi if equispaced else lagrange_eval_cheb
    src_local = list(src_local)
    t = np.empty((dst_order, len(src_local)))
    for l, x in enumerate(src_local):
        for k in range(dst_order):
            t[k, l] = f(dst_order, k, float(x))
    return t


def tensor3_apply(ax, ay, az, v) -> np.ndarray:
    """chebyshev.cpp:246-272: out[i,j,k] = sum Ax(i,a) Ay(j,b) Az(k,c) v[a,b,c];
    v may carry leading batch axes (..., nx*ny*nz)."""
    nx, ny, nz = ax.shape[1], ay.shape[1], az.shape[1]
    vv = np.asarray(v).reshape(v.shape[:-1] + (nx, ny, nz))
    out = np.einsum("ia,jb,kc,...abc->...ijk", ax, ay, az, vv, optimize=True)
    return out.reshape(v.shape[:-1] + (ax.shape[0] * ay.shape[0] * az.shape[0],))


def modified_charges(pos, src, center, radius, hd) -> np.ndarray:
    """chebyshev.cpp:138-203 (P2M) for one cell; rows of pos/src are the cell's particles."""
    L = hd[0].shape[0]
    inv_rad = 1.0 / radius
    local = (pos - center) * inv_rad
    if (np.abs(local) > 1.0 + 1e-9).any():
        raise InvalidArgument("modified_charges: particle outside cell")
    # S^(n)_axis[p, :] = inv_rad^n * hd[n] @ T(local)
    t = cheb_values(L, local)  # (P, 3, L)
    S = [[(inv_rad ** n) * (t[:, ax, :] @ hd[n].T) for n in range(3)] for ax in range(3)]
    terms = [
        (src[:, 0], 0, 0, 0), (src[:, 1], 1, 0, 0), (src[:, 2], 0, 1, 0), (src[:, 3], 0, 0, 1),
        (src[:, 4], 2, 0, 0), (src[:, 7], 0, 2, 0), (src[:, 9], 0, 0, 2),
        (2.0 * src[:, 5], 1, 1, 0), (2.0 * src[:, 6], 1, 0, 1), (2.0 * src[:, 8], 0, 1, 1),
    ]
    q = np.zeros((L, L, L))
    for coef, nx, ny, nz in terms:
        if not coef.any():
            continue
        q += np.einsum("p,pi,pj,pk->ijk", coef, S[0][nx], S[1][ny], S[2][nz], optimize=True)
    return q.reshape(-1)


# ---------------------------------------------------------------- octree.cpp
def build_tree(pos: np.ndarray, r_b: float, depth: int) -> List[np.ndarray]:
    """octree.cpp:27-45: lex leaf buckets (ascending particle index)."""
    if depth < 1 or depth > 8:
        raise InvalidArgument("build_tree: depth must be in [1, 8]")
    n = 1 << depth
    inv_side = n / (2.0 * r_b)
    idx = np.clip(np.floor((pos + r_b) * inv_side).astype(np.int64), 0, n - 1)
    leaf = (idx[:, 0] * n + idx[:, 1]) * n + idx[:, 2]
    order = np.argsort(leaf, kind="stable")
    counts = np.bincount(leaf, minlength=n ** 3)
    offs = np.concatenate([[0], np.cumsum(counts)])
    return [order[offs[c]:offs[c + 1]] for c in range(n ** 3)]


def leaf_csr(pos: np.ndarray, r_b: float, depth: int) -> Tuple[np.ndarray, np.ndarray]:
    buckets = build_tree(pos, r_b, depth)
    offs = np.zeros(len(buckets) + 1, dtype=np.uint32)
    offs[1:] = np.cumsum([len(b) for b in buckets])
    idx = np.concatenate(buckets).astype(np.uint32) if pos.shape[0] else np.zeros(0, np.uint32)
    return offs, idx


def _split_extended(ext, n):
    """octree.cpp:11-14."""
    ext = np.asarray(ext)
    img = np.where(ext >= 0, ext // n, -((-ext + n - 1) // n))
    return ext - n * img, img


def lambda_list(level: int, periodic: bool):
    """octree.cpp:47-87 for one level: arrays (t, s, img[3]) in the reference's
    enumeration order."""
    n = 1 << level
    ts, ss, imgs = [], [], []
    for t in range(n ** 3):
        it = (t // (n * n), (t // n) % n, t % n)
        lo = [2 * ((c >> 1) - 1) for c in it]
        hi = [2 * ((c >> 1) + 1) + 1 for c in it]
        if not periodic:
            lo = [max(x, 0) for x in lo]
            hi = [min(x, n - 1) for x in hi]
        gx, gy, gz = np.meshgrid(np.arange(lo[0], hi[0] + 1), np.arange(lo[1], hi[1] + 1),
                                 np.arange(lo[2], hi[2] + 1), indexing="ij")
        gx, gy, gz = gx.ravel(), gy.ravel(), gz.ravel()
        cheb = np.maximum(np.maximum(np.abs(gx - it[0]), np.abs(gy - it[1])), np.abs(gz - it[2]))
        keep = cheb >= 2
        gx, gy, gz = gx[keep], gy[keep], gz[keep]
        inx, imx = _split_extended(gx, n)
        iny, imy = _split_extended(gy, n)
        inz, imz = _split_extended(gz, n)
        ts.append(np.full(gx.shape, t))
        ss.append((inx * n + iny) * n + inz)
        imgs.append(np.stack([imx, imy, imz], axis=1))
    return np.concatenate(ts), np.concatenate(ss), np.concatenate(imgs)


def leaf_neighbors(depth: int, periodic: bool):
    """octree.cpp:89-110: arrays (a, b, img[3])."""
    n = 1 << depth
    cells = np.arange(n ** 3)
    it = np.stack([cells // (n * n), (cells // n) % n, cells % n], axis=1)
    aa, bb, ii = [], [], []
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                ext = it + np.array([dx, dy, dz])
                ok = np.ones(len(cells), bool) if periodic else ((ext >= 0) & (ext < n)).all(axis=1)
                inn, img = _split_extended(ext, n)
                aa.append(cells[ok])
                bb.append(((inn[:, 0] * n + inn[:, 1]) * n + inn[:, 2])[ok])
                ii.append(img[ok])
    return np.concatenate(aa), np.concatenate(bb), np.concatenate(ii)


# ------------------------------------------------------------------- fmm.cpp
_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (C++ [rand.predef]) -- numpy-vectorised twist."""

    N, M = 312, 156
    A = np.uint64(0xB5026F5AA96619E9)
    UM = np.uint64(0xFFFFFFFF80000000)
    LM = np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [seed & _MASK64]
        for i in range(1, self.N):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK64)
        self.mt = np.array(mt, dtype=np.uint64)
        self.buf = np.zeros(0, dtype=np.uint64)

    def _twist(self):
        mt = self.mt
        N, M = self.N, self.M
        one = np.uint64(1)
        y = (mt[: N - M] & self.UM) | (mt[1: N - M + 1] & self.LM)
        mt[: N - M] = mt[M:] ^ (y >> one) ^ np.where((y & one) != 0, self.A, np.uint64(0))
        y = (mt[N - M: N - 1] & self.UM) | (mt[N - M + 1: N] & self.LM)
        mt[N - M: N - 1] = mt[: M - 1] ^ (y >> one) ^ np.where((y & one) != 0, self.A, np.uint64(0))
        y = (mt[N - 1] & self.UM) | (mt[0] & self.LM)
        mt[N - 1] = mt[M - 1] ^ (y >> one) ^ (self.A if (int(y) & 1) else np.uint64(0))
        x = mt.copy()
        x ^= (x >> np.uint64(29)) & np.uint64(0x5555555555555555)
        x ^= (x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        x ^= (x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        x ^= x >> np.uint64(43)
        return x

    def draw(self, count: int) -> np.ndarray:
        while self.buf.size < count:
            self.buf = np.concatenate([self.buf, self._twist()])
        out, self.buf = self.buf[:count], self.buf[count:]
        return out


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """fmm.cpp:25-36, column-major fill; GCC evaluates the log-argument draw
    first."""
    rng = MT19937_64((seed ^ 0x9E3779B97F4A7C15) & _MASK64)
    raw = rng.draw(2 * rows * cols)
    u = ((raw >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)
    u1, u2 = u[0::2], u[1::2]
    vals = np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586477 * u2)
    return vals.reshape(cols, rows).T.copy()


def instance_offset(level: int, t, s, img):
    """fmm.cpp:43-50."""
    n = 1 << level
    it = np.stack([t // (n * n), (t // n) % n, t % n], axis=-1)
    is_ = np.stack([s // (n * n), (s // n) % n, s % n], axis=-1)
    return is_ + n * img - it


def image_lex_positive(img) -> np.ndarray:
    """fmm.cpp:52-56, vectorised over rows."""
    img = np.asarray(img)
    return np.where(img[:, 0] != 0, img[:, 0] > 0,
                    np.where(img[:, 1] != 0, img[:, 1] > 0, img[:, 2] > 0))


def m2l_dense(order: int, cell_radius: float, offset, xi: float) -> np.ndarray:
    """fmm.cpp:60-96."""
    nodes = cheb_nodes(order)
    d2 = []
    for ax in range(3):
        shift = 2.0 * cell_radius * offset[ax]
        d = cell_radius * (nodes[:, None] - nodes[None, :]) - shift
        d2.append(d * d)
    r2 = (d2[0][:, None, None, :, None, None] + d2[1][None, :, None, None, :, None]) \
        + d2[2][None, None, :, None, None, :]
    r = np.sqrt(r2).reshape(order ** 3, order ** 3)
    return erfc_screen(xi * r) / r


def compress_m2l(c: np.ndarray, svd_tol: float, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """fmm.cpp:98-133: returns (lmat, rmat), each rank x K."""
    k_full = c.shape[0]

    def finish(u, sv, v):
        rank = 1
        while rank < sv.size and sv[rank] > sv[0] * svd_tol:
            rank += 1
        return (u[:, :rank] * sv[:rank]).T.copy(), v[:, :rank].T.copy()

    if k_full <= 150:
        u, sv, vt = np.linalg.svd(c, full_matrices=False)
        return finish(u, sv, vt.T)
    q = 48
    while True:
        q = min(q, k_full)
        omega = gaussian_matrix(k_full, q, seed)
        qmat, _ = np.linalg.qr(c @ omega)
        b = qmat.T @ c
        u, sv, vt = np.linalg.svd(b, full_matrices=False)
        if q == k_full or sv[q - 1] <= sv[0] * svd_tol * 1e-2:
            return finish(qmat @ u, sv, vt.T)
        q *= 2


def offset_key(o) -> int:
    """M2LCache::key, fmm.hpp:42-44."""
    return (int(o[0]) * 4096 + int(o[1])) * 4096 + int(o[2])


def m2l_seed(level: int, key: int) -> int:
    """fmm.cpp:167-169."""
    return (level * 0x100000001B3 + (key & _MASK64)) & _MASK64


def build_m2l_cache(depth: int, periodic: bool, r_b: float, order: int, xi: float,
                    svd_tol: float) -> List[Dict[int, Tuple[np.ndarray, np.ndarray]]]:
    """fmm.cpp:141-179."""
    cache: List[Dict[int, Tuple[np.ndarray, np.ndarray]]] = [dict() for _ in range(depth + 1)]
    for level in range(1, depth + 1):
        t, s, img = lambda_list(level, periodic)
        offs = instance_offset(level, t, s, img)
        uniq = np.unique(offs, axis=0)
        rad = r_b / (1 << level)
        for o in uniq:
            key = offset_key(o)
            cache[level][key] = compress_m2l(m2l_dense(order, rad, o, xi), svd_tol, m2l_seed(level, key))
    return cache


def leaf_expansions(pos, src, r_b, buckets, depth, order) -> np.ndarray:
    """fmm.cpp:181-201: (n_leaves, K), zeros for empty leaves."""
    hd = diff_operator(order)
    n = 1 << depth
    rad = r_b / n
    out = np.zeros((n ** 3, order ** 3))
    for leaf, bucket in enumerate(buckets):
        if bucket.size == 0:
            continue
        i, j, k = leaf // (n * n), (leaf // n) % n, leaf % n
        center = np.array([-r_b + rad * (2 * i + 1), -r_b + rad * (2 * j + 1), -r_b + rad * (2 * k + 1)])
        out[leaf] = modified_charges(pos[bucket], src[bucket], center, rad, hd)
    return out


def m2m_matrices(order: int) -> Tuple[np.ndarray, np.ndarray]:
    """fmm.cpp:213-219."""
    nodes = cheb_nodes(order)
    return transfer_1d(order, 0.5 * (nodes - 1.0)), transfer_1d(order, 0.5 * (nodes + 1.0))


def upward_pass(leaf_values: np.ndarray, depth: int, order: int) -> List[np.ndarray]:
    """fmm.cpp:203-236: expansions[level] of shape (8^level, K)."""
    m2m = m2m_matrices(order)
    exps: List[np.ndarray] = [None] * (depth + 1)  # type: ignore
    exps[depth] = leaf_values
    for level in range(depth - 1, -1, -1):
        n = 1 << level
        nc = 2 * n
        parent = np.zeros((n ** 3, order ** 3))
        child = np.arange(nc ** 3)
        c = np.stack([child // (nc * nc), (child // nc) % nc, child % nc], axis=1)
        pidx = ((c[:, 0] >> 1) * n + (c[:, 1] >> 1)) * n + (c[:, 2] >> 1)
        for cx in (0, 1):
            for cy in (0, 1):
                for cz in (0, 1):
                    sel = (c[:, 0] & 1 == cx) & (c[:, 1] & 1 == cy) & (c[:, 2] & 1 == cz)
                    up = tensor3_apply(m2m[cx], m2m[cy], m2m[cz], exps[level + 1][sel])
                    np.add.at(parent, pidx[sel], up)
        exps[level] = parent
    return exps


def far_field_energy(exps, cache, depth: int, periodic: bool) -> float:
    """fmm.cpp:238-276 (mutual form)."""
    total = 0.0
    for level in range(1, depth + 1):
        t, s, img = lambda_list(level, periodic)
        canon = (t < s) | ((t == s) & image_lex_positive(img))
        t, s, img = t[canon], s[canon], img[canon]
        offs = instance_offset(level, t, s, img)
        keys = (offs[:, 0] * 4096 + offs[:, 1]) * 4096 + offs[:, 2]
        level_sum = 0.0
        m = exps[level]
        for key in np.unique(keys):
            sel = keys == key
            lmat, rmat = cache[level][int(key)]
            u = lmat @ m[t[sel]].T
            v = rmat @ m[s[sel]].T
            level_sum += float((u * v).sum())
        total += level_sum
    return total


def near_field_energy(pos, src, r_b, buckets, depth, periodic, xi, chunk=1 << 20) -> float:
    """fmm.cpp:278-327 (mutual form)."""
    a, b, img = leaf_neighbors(depth, periodic)
    sizes = np.array([len(x) for x in buckets])
    keep = (sizes[a] > 0) & (sizes[b] > 0)
    same = (img == 0).all(axis=1)
    keep &= (a < b) | ((a == b) & same)
    a, b, img, same = a[keep], b[keep], img[keep], same[keep]
    period = 2.0 * r_b
    ix_list, iy_list, sh_list = [], [], []
    for ia, ib, im, sm in zip(a, b, img, same):
        ba, bb = buckets[ia], buckets[ib]
        if ia == ib and sm:
            x, y = np.triu_indices(len(ba), k=1)
            ix_list.append(ba[x])
            iy_list.append(ba[y])
            sh_list.append(np.zeros((len(x), 3)))
        else:
            ix_list.append(np.repeat(ba, len(bb)))
            iy_list.append(np.tile(bb, len(ba)))
            sh_list.append(np.broadcast_to(period * im.astype(np.float64), (len(ba) * len(bb), 3)))
    if not ix_list:
        return 0.0
    ix = np.concatenate(ix_list)
    iy = np.concatenate(iy_list)
    sh = np.concatenate(sh_list)
    total = 0.0
    for lo in range(0, ix.size, chunk):
        hi = min(ix.size, lo + chunk)
        e = pair_interaction(pos[ix[lo:hi]], src[ix[lo:hi]], pos[iy[lo:hi]] + sh[lo:hi],
                             src[iy[lo:hi]], xi)
        total += float(e.sum())
    return total


def periodic_generator(r_b: float, order: int, xi: float, p: int) -> np.ndarray:
    """fmm.cpp:333-369: gen over the (2L-1)^3 embedding."""
    if p < 2:
        raise InvalidArgument("build_periodic_operator: p must be >= 2")
    rng = np.arange(-p, p + 1)
    gx, gy, gz = np.meshgrid(rng, rng, rng, indexing="ij")
    far = np.maximum(np.maximum(np.abs(gx), np.abs(gy)), np.abs(gz)) >= 2
    period = 2.0 * r_b
    shifts = np.stack([gx[far], gy[far], gz[far]], axis=1) * period
    L = order
    eb = 2 * L - 1
    h = 2.0 * r_b / (L - 1)
    idx = np.arange(eb)
    zc = h * np.where(idx < L, idx, idx - eb)
    gen = np.empty((eb, eb, eb))
    for a in range(eb):
        for b in range(eb):
            z = np.stack([np.full(eb, zc[a]), np.full(eb, zc[b]), zc], axis=1)
            d = z[:, None, :] - shifts[None, :, :]
            r = np.sqrt((d * d).sum(axis=2))
            gen[a, b] = (erfc_screen(xi * r) / r).sum(axis=1)
    return gen


def quadratic_form(gen: np.ndarray, v: np.ndarray, L: int) -> float:
    """spectral.cpp:26-39, 73-104: v^T A v with one r2c transform."""
    eb = 2 * L - 1
    spec = np.fft.rfftn(gen)
    padded = np.zeros((eb, eb, eb))
    padded[:L, :L, :L] = v.reshape(L, L, L)
    w = np.fft.rfftn(padded)
    mult = np.full(w.shape, 2.0)
    mult[..., 0] = 1.0
    return float((mult * spec.real * (w.real ** 2 + w.imag ** 2)).sum() / eb ** 3)


def periodic_cancellation_bound(pos, src, r_b: float, order: int, xi: float, p: int,
                                root_cheb: np.ndarray, safety: float = 64.0) -> float:
    """Round-off bound of e_periodic_far for a given system (test
    infrastructure, not a reference function).  The root expansion is a sum
    of per-particle contributions W_a that cancel for a neutral box, so its
    absolute error is ~u |sum_a |W_a||, not u |M_root|; e_per = 1/2 v^T C v
    (v = T x T x T M_root, fmm.cpp:421-427) moves by g . dM with
    g = (T x T x T)^T C v; and the quadratic form itself cancels (C > 0
    entrywise, v of both signs), so its own rounding is ~u |v|^T C |v|.
    Bound: safety * u * (||g|| ||sum_a |W_a| || + |v|^T C |v|)."""
    L = order
    hd = diff_operator(L)
    # per-particle root contributions W_a (modified_charges with the root
    # geometry, one row per particle), summed in absolute value
    inv = 1.0 / r_b
    t = cheb_values(L, pos * inv)
    S = [[(inv ** n) * (t[:, ax, :] @ hd[n].T) for n in range(3)] for ax in range(3)]
    terms = [(src[:, 0], 0, 0, 0), (src[:, 1], 1, 0, 0), (src[:, 2], 0, 1, 0), (src[:, 3], 0, 0, 1),
             (src[:, 4], 2, 0, 0), (src[:, 7], 0, 2, 0), (src[:, 9], 0, 0, 2),
             (2.0 * src[:, 5], 1, 1, 0), (2.0 * src[:, 6], 1, 0, 1), (2.0 * src[:, 8], 0, 1, 1)]
    A = np.zeros(L ** 3)
    for lo in range(0, pos.shape[0], 4096):
        hi = min(pos.shape[0], lo + 4096)
        w = np.zeros((hi - lo, L, L, L))
        for coef, nx, ny, nz in terms:
            w += np.einsum("p,pi,pj,pk->pijk", coef[lo:hi], S[0][nx][lo:hi], S[1][ny][lo:hi], S[2][nz][lo:hi],
                           optimize=True)
        A += np.abs(w.reshape(hi - lo, -1)).sum(axis=0)
    to_equi = transfer_1d(L, cheb_nodes(L), equispaced=True)
    v = tensor3_apply(to_equi, to_equi, to_equi, root_cheb)
    eb = 2 * L - 1
    gen = periodic_generator(r_b, L, xi, p)
    padded = np.zeros((eb, eb, eb))
    padded[:L, :L, :L] = v.reshape(L, L, L)
    cv = np.fft.irfftn(np.fft.rfftn(gen) * np.fft.rfftn(padded), s=(eb, eb, eb))[:L, :L, :L].reshape(-1)
    g = tensor3_apply(to_equi.T, to_equi.T, to_equi.T, cv)
    padded[:L, :L, :L] = np.abs(v).reshape(L, L, L)
    cav = np.fft.irfftn(np.fft.rfftn(gen) * np.fft.rfftn(padded), s=(eb, eb, eb))[:L, :L, :L].reshape(-1)
    vcv = float(np.abs(v) @ cav)
    return float(safety * np.finfo(np.float64).eps / 2 * (np.linalg.norm(g) * np.linalg.norm(A) + vcv))


def periodic_far_energy(root_cheb: np.ndarray, r_b: float, order: int, xi: float, p: int) -> float:
    """fmm.cpp:421-427: 0.5 * quadratic form of the equispaced root expansion."""
    to_equi = transfer_1d(order, cheb_nodes(order), equispaced=True)
    root_equi = tensor3_apply(to_equi, to_equi, to_equi, root_cheb)
    return 0.5 * quadratic_form(periodic_generator(r_b, order, xi, p), root_equi, order)


def fmm_energy(pos: np.ndarray, src: np.ndarray, r_b: float, xi: float = 0.01, p: int = 15,
               order_cheb: int = 8, order_equi: int = 8, depth: int = 0, svd_tol: float = 1e-7,
               recip_cutoff: int = 12) -> Dict[str, float]:
    """fmm.cpp:383-436; returns the EnergyReport components."""
    validate_config(xi, p, order_cheb, order_equi, depth, svd_tol, recip_cutoff)
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    src = np.ascontiguousarray(src, dtype=np.float64).reshape(-1, 10)
    viol = validate_system(pos, src, r_b)
    if viol:
        raise InvalidArgument("fmm_energy: invalid system: " + viol[0][1])
    periodic = p >= 2
    E = depth if depth > 0 else default_depth(pos.shape[0])
    buckets = build_tree(pos, r_b, E)
    hd = diff_operator(order_cheb)  # range check (chebyshev.cpp:86)
    del hd
    cache = build_m2l_cache(E, periodic, r_b, order_cheb, xi, svd_tol)
    exps = upward_pass(leaf_expansions(pos, src, r_b, buckets, E, order_cheb), E, order_cheb)
    e_far = far_field_energy(exps, cache, E, periodic)
    e_near = near_field_energy(pos, src, r_b, buckets, E, periodic, xi)
    e_per = periodic_far_energy(exps[0][0], r_b, order_cheb, xi, p) if periodic else 0.0
    e_self = self_energy(src, xi)
    rep = {"e_self": e_self, "e_near": e_near, "e_far": e_far, "e_periodic_far": e_per,
           "e_reciprocal": 0.0}
    rep["e_total"] = e_self + e_near + e_far + e_per + 0.0
    return rep
