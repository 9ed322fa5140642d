"""ankh_b200: B200-native (sm_100a) drop-in for the ANKH-FMM periodic
point-multipole energy call ``ankh::fmm_energy`` (arXiv 2212.08284).

The compute path is libankh_b200.so (CUDA kernels + C++ plan behind a C-ABI,
include/ankh_b200.h); this package is the thin Python host mirror of the
reference's operator API (see ``api``) plus the synthetic-input generator.
"""
from .api import (  # noqa: F401
    AnkhRuntimeError,
    CudaError,
    DomainError,
    EnergyReport,
    EwaldConfig,
    InvalidArgument,
    ParticleSystem,
    Plan,
    attach_push_group,
    build_tree_csr,
    default_depth,
    device_copy,
    exchange_leaf_levels,
    fmm_energy,
    fmm_forces,
    fft_energy,
    InducedDipoles,
    induced_dipoles,
    nccl_unique_id,
)
from ._lib import LIB_PATH, build, lib  # noqa: F401

__version__ = "0.1.0"
