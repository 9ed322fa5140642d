"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/libankh_ref.so, the
unmodified reference sources compiled against oracle/shim (oracle/Makefile).

Used as the parity checker and as the CPU baseline (``kind: "reference"``).
The product never imports this.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libankh_ref.so")

_lib: Optional[ctypes.CDLL] = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)
_U32 = ctypes.POINTER(ctypes.c_uint32)


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.msg = msg


def available() -> bool:
    return os.path.exists(LIB_PATH)


def build() -> None:
    """Compile the reference (needs /root/reference, i.e. this container)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (run `make -C oracle`)")
        L = ctypes.CDLL(LIB_PATH)
        sz = ctypes.c_size_t
        L.ref_fmm_energy.argtypes = [sz, _D, _D, ctypes.c_double, _D, _I, ctypes.c_int, _D,
                                     ctypes.c_char_p, sz]
        L.ref_fmm_energy_sized.argtypes = [sz, sz, _D, _D, ctypes.c_double, _D, _I, ctypes.c_char_p, sz]
        L.ref_leaf_csr.argtypes = [sz, _D, ctypes.c_double, ctypes.c_int, _U32, _U32, ctypes.c_char_p, sz]
        L.ref_expansions.argtypes = [sz, _D, _D, ctypes.c_double, ctypes.c_int, ctypes.c_int, _D,
                                     ctypes.c_char_p, sz]
        L.ref_far_field.argtypes = [sz, _D, _D, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int, _D,
                                    ctypes.c_char_p, sz]
        L.ref_m2l_factors.argtypes = [ctypes.c_int, ctypes.c_double, _I, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_uint64, _D, _D, ctypes.c_int, _I,
                                      ctypes.c_char_p, sz]
        L.ref_m2l_dense.argtypes = [ctypes.c_int, ctypes.c_double, _I, ctypes.c_double, _D,
                                    ctypes.c_char_p, sz]
        L.ref_list_sizes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _U32, _U32,
                                     ctypes.c_char_p, sz]
        L.ref_erfc_screen.argtypes = [ctypes.c_double]
        L.ref_erfc_screen.restype = ctypes.c_double
        L.ref_pair_interaction.argtypes = [_D, _D, _D, _D, ctypes.c_double, _D, ctypes.c_char_p, sz]
        L.ref_self_energy.argtypes = [sz, _D, ctypes.c_double]
        L.ref_self_energy.restype = ctypes.c_double
        L.ref_default_depth.argtypes = [sz]
        L.ref_default_depth.restype = ctypes.c_int
        L.ref_periodic_far.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                       _D, ctypes.c_int, _D, ctypes.c_char_p, sz]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _check(code: int, err) -> None:
    if code != 0:
        raise RefError(code, err.value.decode())


def fmm_energy(pos, src, r_b, xi=0.01, p=15, order_cheb=8, order_equi=8, depth=0, svd_tol=1e-7,
               recip_cutoff=12, threads=1) -> Dict[str, float]:
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    src = np.ascontiguousarray(src, dtype=np.float64)
    d = np.array([xi, svd_tol], dtype=np.float64)
    i = np.array([p, order_cheb, order_equi, depth, recip_cutoff], dtype=np.int32)
    out = np.zeros(13)
    err = ctypes.create_string_buffer(512)
    n = pos.shape[0]
    _check(lib().ref_fmm_energy(n, _p(pos), _p(src), r_b, _p(d), i.ctypes.data_as(_I), threads,
                                _p(out), err, 512), err)
    keys = ["e_total", "e_self", "e_near", "e_far", "e_periodic_far", "e_reciprocal"]
    rep = {k: float(out[j]) for j, k in enumerate(keys)}
    tk = ["precompute", "interpolation", "far_field", "near_field", "periodic_far", "self", "total"]
    rep["wall_times"] = {k: float(out[6 + j]) for j, k in enumerate(tk)}
    return rep


def fmm_energy_error(pos, src, r_b, xi=0.01, p=15, order_cheb=8, order_equi=8, depth=0, svd_tol=1e-7,
                     recip_cutoff=12):
    """(code, message) the reference's fmm_energy raises on this input (the
    two arrays may differ in length); (0, "") when it does not raise."""
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    src = np.ascontiguousarray(src, dtype=np.float64).reshape(-1, 10)
    d = np.array([xi, svd_tol], dtype=np.float64)
    i = np.array([p, order_cheb, order_equi, depth, recip_cutoff], dtype=np.int32)
    err = ctypes.create_string_buffer(512)
    code = lib().ref_fmm_energy_sized(pos.shape[0], src.shape[0], _p(pos), _p(src), float(r_b), _p(d),
                                      i.ctypes.data_as(_I), err, 512)
    return code, err.value.decode()


def leaf_csr(pos, r_b, depth):
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    n = pos.shape[0]
    offs = np.zeros(8 ** depth + 1, dtype=np.uint32)
    idx = np.zeros(max(n, 1), dtype=np.uint32)
    err = ctypes.create_string_buffer(512)
    _check(lib().ref_leaf_csr(n, _p(pos), r_b, depth, offs.ctypes.data_as(_U32),
                              idx.ctypes.data_as(_U32), err, 512), err)
    return offs, idx[:n]


def expansions(pos, src, r_b, depth, order):
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    src = np.ascontiguousarray(src, dtype=np.float64)
    K = order ** 3
    total = sum(8 ** l for l in range(depth + 1)) * K
    out = np.zeros(total)
    err = ctypes.create_string_buffer(512)
    _check(lib().ref_expansions(pos.shape[0], _p(pos), _p(src), r_b, depth, order, _p(out), err, 512), err)
    res, o = [], 0
    for l in range(depth + 1):
        cnt = 8 ** l * K
        res.append(out[o:o + cnt].reshape(8 ** l, K))
        o += cnt
    return res


def far_field(pos, src, r_b, depth, order, xi=0.01, svd_tol=1e-7, periodic=True, threads=1):
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    src = np.ascontiguousarray(src, dtype=np.float64)
    out = np.zeros(4)
    err = ctypes.create_string_buffer(512)
    _check(lib().ref_far_field(pos.shape[0], _p(pos), _p(src), r_b, depth, order, xi, svd_tol,
                               int(periodic), threads, _p(out), err, 512), err)
    return {"e_far": out[0], "e_far_full": out[1], "rank_sum": out[2], "operators": out[3]}


def m2l_factors(order, cell_radius, offset, xi=0.01, svd_tol=1e-7, seed=0):
    K = order ** 3
    lm = np.zeros(K * K)
    rm = np.zeros(K * K)
    rank = ctypes.c_int(0)
    off = np.array(offset, dtype=np.int32)
    err = ctypes.create_string_buffer(512)
    _check(lib().ref_m2l_factors(order, cell_radius, off.ctypes.data_as(_I), xi, svd_tol, seed,
                                 _p(lm), _p(rm), K, ctypes.byref(rank), err, 512), err)
    k = rank.value
    return lm[: k * K].reshape(k, K), rm[: k * K].reshape(k, K)


def m2l_dense(order, cell_radius, offset, xi=0.01):
    K = order ** 3
    out = np.zeros(K * K)
    off = np.array(offset, dtype=np.int32)
    err = ctypes.create_string_buffer(512)
    _check(lib().ref_m2l_dense(order, cell_radius, off.ctypes.data_as(_I), xi, _p(out), err, 512), err)
    return out.reshape(K, K)


def list_sizes(depth, periodic, level):
    lam = np.zeros(8 ** level, dtype=np.uint32)
    nb = np.zeros(8 ** depth, dtype=np.uint32)
    err = ctypes.create_string_buffer(512)
    _check(lib().ref_list_sizes(depth, int(periodic), level, lam.ctypes.data_as(_U32),
                                nb.ctypes.data_as(_U32), err, 512), err)
    return lam, nb


def erfc_screen(z: float) -> float:
    return float(lib().ref_erfc_screen(z))


def pair_interaction(xa, sa, xb, sb, xi):
    xa, sa, xb, sb = (np.ascontiguousarray(v, dtype=np.float64) for v in (xa, sa, xb, sb))
    out = np.zeros(1)
    err = ctypes.create_string_buffer(512)
    _check(lib().ref_pair_interaction(_p(xa), _p(sa), _p(xb), _p(sb), xi, _p(out), err, 512), err)
    return float(out[0])


def self_energy(src, xi):
    src = np.ascontiguousarray(src, dtype=np.float64)
    return float(lib().ref_self_energy(src.shape[0], _p(src), xi))


def default_depth(n: int) -> int:
    return int(lib().ref_default_depth(n))


def periodic_far(r_b, order, xi, p, root_cheb, threads=1):
    root = np.ascontiguousarray(root_cheb, dtype=np.float64)
    out = np.zeros(1)
    err = ctypes.create_string_buffer(512)
    _check(lib().ref_periodic_far(r_b, order, xi, p, _p(root), threads, _p(out), err, 512), err)
    return float(out[0])
