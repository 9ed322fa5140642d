"""TEST INFRASTRUCTURE ONLY: the direct screened lattice sum on the GPU
(oracle/direct/libankh_direct.so), the exact quantity the FMM approximates:

    E = 1/2 sum_{|I|inf <= p} sum_{i,j: i != j or I != 0} pair_interaction(x_i, x_j + 2 r_B I)
        + self_energy                                  (kernel.cpp:157-213)

Used by tests/ to measure the FMM's physical accuracy; the
product library does not contain it.  Cost n^2 (2p+1)^3 pair evaluations."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "direct", "libankh_direct.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "direct")], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} not built (oracle.direct.build())")
        L = ctypes.CDLL(LIB)
        D = ctypes.POINTER(ctypes.c_double)
        L.ankh_direct_lattice_v1.argtypes = [ctypes.c_size_t, D, D, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_double, D, D, D,
                                             ctypes.c_char_p, ctypes.c_size_t]
        L.ankh_direct_lattice_v1.restype = ctypes.c_int
        _lib = L
    return _lib


def direct_energy(pos, src, box_radius: float, xi: float = 0.01, p: int = 15,
                  max_pair_evaluations: float = 1e12) -> dict:
    """{"e_lattice", "e_self", "e_total"} of the direct lattice sum."""
    import ankh_oracle as O
    import paper_2212_08284_b200 as ankh

    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    src = np.ascontiguousarray(src, dtype=np.float64).reshape(-1, 10)
    n = pos.shape[0]
    evals = float(n) * n * (2 * p + 1) ** 3
    if evals > max_pair_evaluations:
        raise RuntimeError(f"direct: n^2 (2p+1)^3 = {evals:g} pair evaluations exceed the budget")
    # the product's near-field radial polynomials, valid at any distance
    nt, sl = ctypes.c_int(), ctypes.c_double()
    pc, gc, me = (ctypes.c_double * 14)(), (ctypes.c_double * 14)(), ctypes.c_double()
    assert ankh.lib().ankh_radial_fit_v1(1e9, ctypes.byref(nt), ctypes.byref(sl), pc, gc,
                                         ctypes.byref(me)) == 0
    D = ctypes.POINTER(ctypes.c_double)
    out = ctypes.c_double()
    err = ctypes.create_string_buffer(512)
    code = _load().ankh_direct_lattice_v1(n, pos.ctypes.data_as(D), src.ctypes.data_as(D),
                                          float(box_radius), float(xi), int(p), nt.value, sl.value,
                                          pc, gc, ctypes.byref(out), err, 512)
    if code != 0:
        raise RuntimeError(err.value.decode())
    e_self = float(O.self_energy(src, xi))
    return {"e_lattice": out.value, "e_self": e_self, "e_total": out.value + e_self}
