"""Loader for the in-tree sm_100a library (libankh_b200.so).  Fails loudly when
the library is missing: the product has no CPU fallback."""
from __future__ import annotations

import ctypes
import os
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
# ANKH_B200_LIB selects an alternative in-tree build (kernel A/B experiments)
LIB_PATH = os.environ.get("ANKH_B200_LIB") or os.path.join(HERE, "libankh_b200.so")

_lib: Optional[ctypes.CDLL] = None

EXPORTS = [
    "ankh_config_default_v1",
    "ankh_fmm_energy_v1",
    "ankh_check_call_v1",
    "ankh_fmm_forces_v1",
    "ankh_plan_forces_v1",
    "ankh_plan_derivatives_v1",
    "ankh_plan_create_fft_v1",
    "ankh_plan_create_v1",
    "ankh_plan_destroy_v1",
    "ankh_plan_energy_v1",
    "ankh_plan_energy_device_v1",
    "ankh_plan_enqueue_v1",
    "ankh_plan_result_v1",
    "ankh_plan_info_v1",
    "ankh_plan_expansions_v1",
    "ankh_leaf_csr_v1",
    "ankh_plan_m2l_factors_v1",
    "ankh_version_v1",
    "ankh_plan_energies_device_v1",
    "ankh_probe_fp64_tflops_v1",
    "ankh_shard_leaf_range_v1",
    "ankh_shard_cell_owner_v1",
    "ankh_shard_m2l_instances_v1",
    "ankh_plan_enqueue_phase_v1",
    "ankh_plan_leaf_level_v1",
    "ankh_device_copy_v1",
    "ankh_nccl_unique_id_v1",
    "ankh_plan_attach_nccl_v1",
    "ankh_plan_attach_loopback_v1",
    "ankh_nccl_selftest_v1",
    "ankh_plan_attach_push_group_v1",
    "ankh_shard_src_slice_v1",
    "ankh_shard_exchange_level_v1",
    "ankh_shard_halo_cells_v1",
    "ankh_shard_exchange_bytes_v1",
    "ankh_probe_fp64_mix_ms_v1",
    "ankh_radial_fit_v1",
    "ankh_probe_dmma_tflops_v1",
    "ankh_plan_set_positions_v1",
    "ankh_plan_energy_sources_v1",
]


def build(verbose: bool = False) -> str:
    """Compile csrc/ into libankh_b200.so (nvcc -gencode arch=compute_100a,code=sm_100a)."""
    import subprocess

    cmd = ["make", "-j8", "-C", os.path.join(HERE, "csrc")]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        c_void_p, c_size_t, c_int, c_double = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_double
        D = ctypes.POINTER(ctypes.c_double)
        U32 = ctypes.POINTER(ctypes.c_uint32)
        I = ctypes.POINTER(ctypes.c_int)
        cp = ctypes.c_char_p
        L.ankh_config_default_v1.argtypes = [c_void_p]
        L.ankh_config_default_v1.restype = None
        L.ankh_fmm_energy_v1.argtypes = [c_size_t, D, D, c_double, c_void_p, c_void_p, cp, c_size_t]
        L.ankh_fmm_forces_v1.argtypes = [c_size_t, D, D, c_double, c_void_p, D, c_void_p, cp, c_size_t]
        L.ankh_plan_forces_v1.argtypes = [c_void_p, D, D, D, c_void_p, cp, c_size_t]
        L.ankh_plan_derivatives_v1.argtypes = [c_void_p, D, D, D, D, c_void_p, cp, c_size_t]
        L.ankh_check_call_v1.argtypes = [c_void_p, c_double, c_size_t, c_size_t, cp, c_size_t]
        L.ankh_plan_create_v1.argtypes = [c_size_t, c_double, c_void_p, c_void_p, cp, c_size_t]
        L.ankh_plan_create_fft_v1.argtypes = [c_size_t, c_double, c_void_p, c_void_p, cp, c_size_t]
        L.ankh_plan_destroy_v1.argtypes = [c_void_p]
        L.ankh_plan_destroy_v1.restype = None
        L.ankh_plan_energy_v1.argtypes = [c_void_p, D, D, c_void_p, cp, c_size_t]
        L.ankh_plan_energy_device_v1.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, cp, c_size_t]
        L.ankh_plan_enqueue_v1.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, cp, c_size_t]
        L.ankh_plan_result_v1.argtypes = [c_void_p, c_void_p, cp, c_size_t]
        L.ankh_plan_info_v1.argtypes = [c_void_p] + [c_void_p] * 7
        L.ankh_plan_expansions_v1.argtypes = [c_void_p, D, c_size_t, cp, c_size_t]
        L.ankh_leaf_csr_v1.argtypes = [c_size_t, D, c_double, c_int, U32, U32, cp, c_size_t]
        L.ankh_plan_m2l_factors_v1.argtypes = [c_void_p, c_int, I, D, D, c_int, I, cp, c_size_t]
        L.ankh_plan_energies_device_v1.argtypes = [c_void_p, c_void_p, c_void_p, cp, c_size_t]
        L.ankh_probe_fp64_tflops_v1.argtypes = [c_int]
        L.ankh_probe_fp64_tflops_v1.restype = c_double
        I64 = ctypes.POINTER(ctypes.c_int64)
        L.ankh_shard_leaf_range_v1.argtypes = [c_int, c_int, c_int, I64, I64]
        L.ankh_shard_cell_owner_v1.argtypes = [c_int, ctypes.c_uint32, c_int, c_int]
        L.ankh_shard_src_slice_v1.argtypes = [c_size_t, c_int, c_int, ctypes.POINTER(c_size_t),
                                              ctypes.POINTER(c_size_t)]
        L.ankh_shard_exchange_level_v1.argtypes = [c_int, c_int]
        L.ankh_shard_halo_cells_v1.argtypes = [c_int, c_int, c_int, c_int, c_int, c_int, U32, c_size_t,
                                               ctypes.POINTER(c_size_t)]
        L.ankh_shard_exchange_bytes_v1.argtypes = [c_int, c_int, c_int, c_int, c_int, c_int,
                                                   ctypes.POINTER(c_size_t), ctypes.POINTER(c_size_t)]
        L.ankh_shard_m2l_instances_v1.argtypes = [c_int, c_int, c_int, c_int, U32, U32, U32, I,
                                                  c_size_t, ctypes.POINTER(c_size_t)]
        L.ankh_plan_enqueue_phase_v1.argtypes = [c_void_p, c_int, c_void_p, c_void_p, c_void_p, cp,
                                                 c_size_t]
        L.ankh_plan_leaf_level_v1.argtypes = [c_void_p, ctypes.POINTER(c_void_p), I64, I64, I]
        L.ankh_device_copy_v1.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, cp, c_size_t]
        L.ankh_nccl_unique_id_v1.argtypes = [ctypes.c_char_p, cp, c_size_t]
        L.ankh_plan_attach_nccl_v1.argtypes = [c_void_p, ctypes.c_char_p, cp, c_size_t]
        L.ankh_plan_attach_loopback_v1.argtypes = [c_void_p, cp, c_size_t]
        L.ankh_nccl_selftest_v1.argtypes = [cp, c_size_t]
        L.ankh_plan_attach_push_group_v1.argtypes = [ctypes.POINTER(c_void_p), c_int, cp, c_size_t]
        L.ankh_plan_set_positions_v1.argtypes = [c_void_p, D, cp, c_size_t]
        L.ankh_plan_energy_sources_v1.argtypes = [c_void_p, D, c_void_p, cp, c_size_t]
        L.ankh_probe_dmma_tflops_v1.argtypes = [c_int, c_int]
        L.ankh_probe_dmma_tflops_v1.restype = c_double
        L.ankh_probe_fp64_mix_ms_v1.argtypes = [c_int, c_int, c_int]
        L.ankh_probe_fp64_mix_ms_v1.restype = c_double
        L.ankh_radial_fit_v1.argtypes = [c_double, I, D, D, D, D]
        L.ankh_version_v1.argtypes = []
        L.ankh_version_v1.restype = ctypes.c_char_p
        _lib = L
    return _lib
