"""TEST INFRASTRUCTURE ONLY (checker): a numpy restatement of the ANKH-FFT
far field (Alg. 4-5, Thm. 1, Cor. 1 and 3;
SPEC.md `fftengine`), against which the GPU engine (`engine="fft"`) is
checked.  There is no reference code for this engine: the checks are a dense
double sum on tiny trees (this module's `dense_far`) and convergence to the
reference's own far field (e_far + e_periodic_far of oracle/_ref) as the
orders grow.

Formulation (one level, the leaves):
  * v_c = (E x E x E) Q_c: each leaf's Chebyshev expansion Q_c (the
    reference's leaf_expansions, fmm.cpp:181-201) re-interpolated onto an
    equispaced L_u grid, E[k, l] = U_k(c_l) -- transfer_1d(equispaced(L_u),
    chebyshev nodes(L_c)), the matrix the reference's periodic term uses
    (fmm.cpp:421-425);
  * A[(t, a), (s, b)] = sum over images I with |I|_inf <= 1 of
    H(2 rad D + h (a - b)) for D = t - s + n I when |D|_inf >= 2 (the
    leaf pairs the reference's M2L covers at some level, octree.cpp:47-112),
    H(r) = erfc_screen(xi r) / r (the M2L kernel, fmm.cpp:60-96),
    h = 2 rad / (L_u - 1);
  * A is two-level block Toeplitz (cell offset, node offset per axis), so it
    embeds in a circulant of size (2n - 1)(2L_u - 1) per axis whose 6-D DFT
    is its (real) spectrum, and
        F = 1/2 v^T A v = 1/(2m) sum_k Re(diag_k) |DFT(pad(v))_k|^2
    (Cor. 3, Eq. 44: one forward transform, no inverse).
The far images 2 <= |I|_inf <= p stay on the reference's root operator
(e_periodic_far, fmm.cpp:421-427) -- an equispaced interpolation at the root
as well; SPEC's variant folds them into the diagonal through a far-image
table instead.
"""
from __future__ import annotations

import numpy as np

import ankh_oracle as O


def equi_leaf_values(pos, src, r_b, depth, order_cheb, order_equi) -> np.ndarray:
    """v[cx, cy, cz, a, b, c] (lex cells, equispaced nodes)."""
    buckets = O.build_tree(pos, r_b, depth)
    Q = O.leaf_expansions(pos, src, r_b, buckets, depth, order_cheb)
    E = O.transfer_1d(order_equi, O.cheb_nodes(order_cheb), equispaced=True)
    v = O.tensor3_apply(E, E, E, Q)
    n = 1 << depth
    Lu = order_equi
    return v.reshape(n, n, n, Lu, Lu, Lu)


def kernel(r, xi):
    return O.erfc_screen(xi * r) / r


def generator(r_b, depth, order_equi, xi, periodic=True) -> np.ndarray:
    """First column of the two-level circulant embedding: G[dcx, dcy, dcz,
    dnx, dny, dnz] over (2n-1)^3 x (2L_u-1)^3, offsets stored at o (o >= 0)
    and o + P (o < 0)."""
    n = 1 << depth
    Lu = order_equi
    rad = r_b / n
    h = 2.0 * rad / (Lu - 1)
    Pc, Pn = 2 * n - 1, 2 * Lu - 1
    dc = np.arange(Pc)
    dc = np.where(dc < n, dc, dc - Pc)
    dn = np.arange(Pn)
    dn = np.where(dn < Lu, dn, dn - Pn)
    G = np.zeros((Pc, Pc, Pc, Pn, Pn, Pn))
    imgs = (-1, 0, 1) if periodic else (0,)
    for ix in imgs:
        for iy in imgs:
            for iz in imgs:
                Dx, Dy, Dz = dc + n * ix, dc + n * iy, dc + n * iz
                far = np.maximum(np.maximum(np.abs(Dx)[:, None, None], np.abs(Dy)[None, :, None]),
                                 np.abs(Dz)[None, None, :]) >= 2
                zx = 2 * rad * Dx[:, None] + h * dn[None, :]
                zy = 2 * rad * Dy[:, None] + h * dn[None, :]
                zz = 2 * rad * Dz[:, None] + h * dn[None, :]
                r = np.sqrt(zx[:, None, None, :, None, None] ** 2 + zy[None, :, None, None, :, None] ** 2 +
                            zz[None, None, :, None, None, :] ** 2)
                safe = np.where(far[:, :, :, None, None, None], r, 1.0)
                G += np.where(far[:, :, :, None, None, None], kernel(safe, xi), 0.0)
    return G


def fft_far(v: np.ndarray, G: np.ndarray) -> float:
    n, Lu = v.shape[0], v.shape[3]
    Pc, Pn = 2 * n - 1, 2 * Lu - 1
    pad = np.zeros((Pc, Pc, Pc, Pn, Pn, Pn))
    pad[:n, :n, :n, :Lu, :Lu, :Lu] = v
    w = np.fft.fftn(pad)
    d = np.fft.fftn(G)
    return 0.5 * float(np.sum(d.real * np.abs(w) ** 2)) / pad.size


def dense_far(v: np.ndarray, r_b, depth, order_equi, xi, periodic=True) -> float:
    """1/2 v^T A v summed pair by pair (tiny trees only)."""
    n = 1 << depth
    Lu = order_equi
    rad = r_b / n
    h = 2.0 * rad / (Lu - 1)
    nodes = np.arange(Lu)
    nn = np.stack(np.meshgrid(nodes, nodes, nodes, indexing="ij"), -1).reshape(-1, 3)
    cells = [(a, b, c) for a in range(n) for b in range(n) for c in range(n)]
    e = 0.0
    for t in cells:
        for s in cells:
            for img in (np.ndindex(3, 3, 3) if periodic else [(1, 1, 1)]):
                D = np.array(t) - np.array(s) + n * (np.array(img) - 1)
                if np.abs(D).max() < 2:
                    continue
                z = 2 * rad * D[None, None, :] + h * (nn[:, None, :] - nn[None, :, :])
                e += 0.5 * v[t].reshape(-1) @ kernel(np.sqrt((z ** 2).sum(-1)), xi) @ v[s].reshape(-1)
    return e


def fft_far_energy(pos, src, r_b, depth, order_cheb, order_equi, xi=0.01, periodic=True) -> float:
    v = equi_leaf_values(pos, src, r_b, depth, order_cheb, order_equi)
    return fft_far(v, generator(r_b, depth, order_equi, xi, periodic))
