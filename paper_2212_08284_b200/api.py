"""Python mirror of the reference's energy API over the C-ABI of libankh_b200.so.

Names, fields and error behaviour follow the reference (paths relative to
/root/reference/proj/core):

* ``EwaldConfig``      <- ``ankh::EwaldConfig``   (include/ankh/types.hpp:96-104)
* ``ParticleSystem``   <- ``ankh::ParticleSystem`` (types.hpp:88-94)
* ``EnergyReport``     <- ``ankh::EnergyReport``   (types.hpp:123-135)
* ``fmm_energy``       <- ``ankh::fmm_energy``     (include/ankh/fmm.hpp:98-99)
* ``default_depth``    <- ``ankh::default_depth``  (src/types.cpp:9-14)
* ``build_tree_csr``   <- ``ankh::build_tree``     (src/octree.cpp:27-45), as CSR

Exceptions map the reference's C++ types: ``InvalidArgument`` (a ValueError)
for std::invalid_argument, ``DomainError`` (an ArithmeticError) for
std::domain_error, ``AnkhRuntimeError`` for std::runtime_error and
``CudaError`` for device failures.  There is no CPU fallback: without the
built library or a GPU every call raises.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
from typing import Dict, Optional, Tuple

import numpy as np

from ._lib import lib

__all__ = [
    "EwaldConfig",
    "ParticleSystem",
    "EnergyReport",
    "InvalidArgument",
    "DomainError",
    "AnkhRuntimeError",
    "CudaError",
    "fmm_energy",
    "fmm_forces",
    "InducedDipoles",
    "fft_energy",
    "induced_dipoles",
    "default_depth",
    "build_tree_csr",
    "Plan",
    "nccl_unique_id",
    "device_copy",
    "exchange_leaf_levels",
    "attach_push_group",
]


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class DomainError(ArithmeticError):
    """std::domain_error."""


class AnkhRuntimeError(RuntimeError):
    """std::runtime_error."""


class CudaError(RuntimeError):
    """CUDA / NCCL failure (no reference counterpart)."""


_ERRORS = {1: InvalidArgument, 2: DomainError, 3: AnkhRuntimeError, 4: CudaError}


class _Config(ctypes.Structure):
    _fields_ = [
        ("xi", ctypes.c_double),
        ("p", ctypes.c_int),
        ("order_cheb", ctypes.c_int),
        ("order_equi", ctypes.c_int),
        ("depth", ctypes.c_int),
        ("svd_tol", ctypes.c_double),
        ("recip_cutoff", ctypes.c_int),
        ("threads", ctypes.c_int),
        ("device", ctypes.c_int),
        ("rank", ctypes.c_int),
        ("world", ctypes.c_int),
        ("phase_timing", ctypes.c_int),
    ]


class _Report(ctypes.Structure):
    _fields_ = [
        ("e_total", ctypes.c_double),
        ("e_self", ctypes.c_double),
        ("e_near", ctypes.c_double),
        ("e_far", ctypes.c_double),
        ("e_periodic_far", ctypes.c_double),
        ("e_reciprocal", ctypes.c_double),
        ("t_precompute", ctypes.c_double),
        ("t_interpolation", ctypes.c_double),
        ("t_far_field", ctypes.c_double),
        ("t_near_field", ctypes.c_double),
        ("t_periodic_far", ctypes.c_double),
        ("t_self", ctypes.c_double),
        ("t_total", ctypes.c_double),
        ("depth", ctypes.c_int),
        ("order_cheb", ctypes.c_int),
        ("near_pairs", ctypes.c_uint64),
        ("far_instances", ctypes.c_uint64),
        ("far_flops", ctypes.c_double),
        ("gpu_launches", ctypes.c_uint32),
    ]


@dataclasses.dataclass
class EwaldConfig:
    """ankh::EwaldConfig (types.hpp:96-104) with the same defaults."""

    xi: float = 0.01
    p: int = 15
    order_cheb: int = 8
    order_equi: int = 8
    depth: int = 0
    svd_tol: float = 1e-7
    recip_cutoff: int = 12

    def _c(self, threads: int = 0, device: int = -1, rank: int = 0, world: int = 1,
           phase_timing: bool = True) -> _Config:
        return _Config(float(self.xi), int(self.p), int(self.order_cheb), int(self.order_equi),
                       int(self.depth), float(self.svd_tol), int(self.recip_cutoff), int(threads),
                       int(device), int(rank), int(world), 1 if phase_timing else 0)


@dataclasses.dataclass
class ParticleSystem:
    """ankh::ParticleSystem: positions N x 3, sources N x 10 (q, mu, Theta xx xy xz yy yz zz)."""

    positions: np.ndarray
    sources: np.ndarray
    box_radius: float = 1.0

    def size(self) -> int:
        return int(np.asarray(self.positions).shape[0])


@dataclasses.dataclass
class EnergyReport:
    """ankh::EnergyReport (types.hpp:123-135) plus work counters."""

    e_total: float = 0.0
    e_self: float = 0.0
    e_near: float = 0.0
    e_far: float = 0.0
    e_periodic_far: float = 0.0
    e_reciprocal: float = 0.0
    wall_times: Dict[str, float] = dataclasses.field(default_factory=dict)
    depth: int = 0
    order_cheb: int = 0
    near_pairs: int = 0
    far_instances: int = 0
    far_flops: float = 0.0
    gpu_launches: int = 0

    def component_sum(self) -> float:
        return self.e_self + self.e_near + self.e_far + self.e_periodic_far + self.e_reciprocal

    @staticmethod
    def _from_c(r: _Report, wall: Optional[float] = None) -> "EnergyReport":
        times = {
            "precompute": r.t_precompute,
            "interpolation": r.t_interpolation,
            "far_field": r.t_far_field,
            "near_field": r.t_near_field,
            "periodic_far": r.t_periodic_far,
            "self": r.t_self,
            "total": r.t_total if wall is None else wall,
        }
        return EnergyReport(r.e_total, r.e_self, r.e_near, r.e_far, r.e_periodic_far,
                            r.e_reciprocal, times, r.depth, r.order_cheb, int(r.near_pairs),
                            int(r.far_instances), float(r.far_flops), int(r.gpu_launches))


def _check(code: int, err: ctypes.Array) -> None:
    if code != 0:
        raise _ERRORS.get(code, AnkhRuntimeError)(err.value.decode(errors="replace"))


def _as_host(a, cols: int) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if arr.size == 0:
        return arr.reshape(0, cols)
    return arr.reshape(-1, cols)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def default_depth(n: int) -> int:
    """types.cpp:9-14."""
    if n <= 64:
        return 1
    levels = math.log(n / 64.0) / math.log(8.0)
    return max(1, int(math.ceil(levels - 1e-12)))


def fmm_energy(system: ParticleSystem, config: Optional[EwaldConfig] = None,
               threads: int = 1) -> EnergyReport:
    """Drop-in for ankh::fmm_energy; host arrays in, energy out (one GPU).

    ``threads`` only sizes the host precompute pool (<= 0: all cores); the
    geometry-only plan is cached inside the library across calls.
    """
    config = config or EwaldConfig()
    pos = _as_host(system.positions, 3)
    src = _as_host(system.sources, 10)
    rep = _Report()
    err = ctypes.create_string_buffer(512)
    c = config._c(threads=threads)
    # validate_config, box radius, size mismatch: the reference's order (fmm.cpp:384-388)
    _check(lib().ankh_check_call_v1(ctypes.byref(c), float(system.box_radius), pos.shape[0],
                                    src.shape[0], err, 512), err)
    code = lib().ankh_fmm_energy_v1(pos.shape[0], _ptr(pos), _ptr(src), float(system.box_radius),
                                    ctypes.byref(c), ctypes.byref(rep), err, 512)
    _check(code, err)
    return EnergyReport._from_c(rep)


def fmm_forces(system: ParticleSystem, config: Optional[EwaldConfig] = None,
               threads: int = 1):
    """Energy and forces F = -dE/dx (n x 3 array, the input's particle order),
    moments held fixed in the lab frame (the reference
    computes energies only).  Returns (EnergyReport, forces)."""
    config = config or EwaldConfig()
    pos = _as_host(system.positions, 3)
    src = _as_host(system.sources, 10)
    rep = _Report()
    err = ctypes.create_string_buffer(512)
    c = config._c(threads=threads)
    _check(lib().ankh_check_call_v1(ctypes.byref(c), float(system.box_radius), pos.shape[0],
                                    src.shape[0], err, 512), err)
    forces = np.zeros((pos.shape[0], 3), dtype=np.float64)
    _check(lib().ankh_fmm_forces_v1(pos.shape[0], _ptr(pos), _ptr(src), float(system.box_radius),
                                    ctypes.byref(c), _ptr(forces), ctypes.byref(rep), err, 512), err)
    return EnergyReport._from_c(rep), forces


@dataclasses.dataclass
class InducedDipoles:
    dipoles: np.ndarray      # n x 3 induced dipoles (e.A)
    iterations: int          # conjugate-gradient iterations (one field evaluation each)
    residual: float          # |mu / alpha - E(s + mu)| / |F0|, from a fresh evaluation
    field: np.ndarray        # n x 3 total field at the solution (permanent + induced)


def induced_dipoles(plan: "Plan", positions, sources, polarizability, tol: float = 1e-10,
                    max_iter: int = 100) -> InducedDipoles:
    """Self-consistent induced dipoles mu = alpha E(s + mu) (point
    polarizabilities, the field of the same periodic FMM energy, Ewald self
    term included) -- the solve the paper's perspective and BASELINE config 4
    ("induced-dipole-style repeated solve") refer to.  E is affine in mu:
    E(s + mu) = F0 + J mu with F0 = the field of the permanent moments and
    J mu = the field of the dipoles mu alone, so (alpha^-1 - J) mu = F0 is
    solved by conjugate gradients (J is symmetric: minus the energy's Hessian
    in the dipoles); every product J p is one GPU field evaluation.
    polarizability: scalar or length-n array (A^3)."""
    pos = _as_host(positions, 3)
    src = _as_host(sources, 10)
    n = pos.shape[0]
    alpha = np.broadcast_to(np.asarray(polarizability, dtype=np.float64), (n,)).reshape(n, 1)
    if np.any(alpha <= 0):
        raise InvalidArgument("induced_dipoles: polarizabilities must be positive")
    inv_a = 1.0 / alpha
    f0 = plan.field(pos, src)
    probe = np.zeros_like(src)

    def jmul(v):
        probe[:, 1:4] = v
        return plan.field(pos, probe)

    x = alpha * f0  # the first (direct-field) guess
    r = f0 - (inv_a * x - jmul(x))
    p = r.copy()
    rr = float(np.vdot(r, r))
    bn = max(float(np.sqrt(np.vdot(f0, f0))), 1e-300)
    it = 0
    while np.sqrt(rr) / bn > tol and it < max_iter:
        ap = inv_a * p - jmul(p)
        it += 1
        step = rr / float(np.vdot(p, ap))
        x += step * p
        r -= step * ap
        rr_new = float(np.vdot(r, r))
        p = r + (rr_new / rr) * p
        rr = rr_new
    # the residual from a fresh evaluation at the total moments: mu = alpha E(s + mu)
    total = src.copy()
    total[:, 1:4] += x
    ftot = plan.field(pos, total)
    res = float(np.sqrt(np.vdot(inv_a * x - ftot, inv_a * x - ftot))) / bn
    return InducedDipoles(dipoles=x, iterations=it, residual=res, field=ftot)


def fft_energy(system: ParticleSystem, config: Optional[EwaldConfig] = None) -> EnergyReport:
    """The ANKH-FFT engine (Alg. 4-5): the far
    field of the leaf level as one circulant quadratic form on equispaced grids
    of order ``config.order_equi`` (6-D DFT on the GPU, ``k_fft.cu``), near
    field, self energy and far images as the reference computes them.  Not the
    reference's energy (which has no such engine): it converges to it as
    order_cheb and order_equi grow."""
    config = config or EwaldConfig()
    pos = _as_host(system.positions, 3)
    src = _as_host(system.sources, 10)
    plan = Plan(pos.shape[0], system.box_radius, config, engine="fft", phase_timing=False)
    try:
        return plan.energy(pos, src)
    finally:
        plan.close()


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; broadcast to the other shards)."""
    buf = ctypes.create_string_buffer(128)
    err = ctypes.create_string_buffer(512)
    _check(lib().ankh_nccl_unique_id_v1(buf, err, 512), err)
    return buf.raw


def device_copy(dst_ptr: int, src_ptr: int, nbytes: int, stream: int = 0) -> None:
    """cudaMemcpyAsync device-to-device (shard leaf-level exchange in one process)."""
    err = ctypes.create_string_buffer(512)
    _check(lib().ankh_device_copy_v1(ctypes.c_void_p(dst_ptr), ctypes.c_void_p(src_ptr), int(nbytes),
                                     ctypes.c_void_p(stream), err, 512), err)


def exchange_leaf_levels(plans, stream: int = 0) -> None:
    """Complete every shard's leaf level from the others' rows (in-process
    equivalent of the NCCL all-gather; all plans on the current device)."""
    info = [p.leaf_level() for p in plans]
    for j, (dst, _, _, stride) in enumerate(info):
        for i, (src, b, e, _) in enumerate(info):
            if i == j or e <= b:
                continue
            off = b * stride * 8
            device_copy(dst + off, src + off, (e - b) * stride * 8, stream)


def attach_push_group(plans) -> None:
    """Tests on one GPU: the shards of one sharding (plans[r] has rank r)
    exchange by stream-ordered pushes of their expansion slabs into each
    other's arrays; from the second evaluation of the same inputs on, each
    reports its true partial energies (their sum is the job's)."""
    arr = (ctypes.c_void_p * len(plans))(*[p._h for p in plans])
    err = ctypes.create_string_buffer(512)
    _check(lib().ankh_plan_attach_push_group_v1(arr, len(plans), err, 512), err)


def build_tree_csr(positions, box_radius: float, depth: int) -> Tuple[np.ndarray, np.ndarray]:
    """Leaf buckets of build_tree as CSR (offsets[8^depth+1], indices[N]), on the GPU."""
    pos = _as_host(positions, 3)
    n = pos.shape[0]
    if depth < 1 or depth > 8:
        raise InvalidArgument("build_tree: depth must be in [1, 8]")
    offs = np.zeros(8 ** depth + 1, dtype=np.uint32)
    idx = np.zeros(max(n, 1), dtype=np.uint32)
    err = ctypes.create_string_buffer(512)
    code = lib().ankh_leaf_csr_v1(n, _ptr(pos), float(box_radius), int(depth),
                                  offs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                  idx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), err, 512)
    _check(code, err)
    return offs, idx[:n]


class Plan:
    """Cached geometry-only precompute (M2L factors, periodic spectrum, buffers)
    for n particles in [-box_radius, box_radius]^3, evaluated many times.

    ``rank``/``world`` select a spatial shard (Morton leaf range + M2L tiles);
    the per-shard energies are partial sums for the caller to all-reduce.
    """

    def __init__(self, n: int, box_radius: float, config: Optional[EwaldConfig] = None,
                 threads: int = 0, device: int = -1, rank: int = 0, world: int = 1,
                 phase_timing: bool = True, engine: str = "fmm"):
        self.config = config or EwaldConfig()
        self.n = int(n)
        self.box_radius = float(box_radius)
        self._h = ctypes.c_void_p()
        err = ctypes.create_string_buffer(512)
        cfg = self.config._c(threads=threads, device=device, rank=rank, world=world,
                             phase_timing=phase_timing)
        if engine not in ("fmm", "fft"):
            raise InvalidArgument("engine must be 'fmm' (the reference's) or 'fft' (ANKH-FFT)")
        create = lib().ankh_plan_create_fft_v1 if engine == "fft" else lib().ankh_plan_create_v1
        _check(create(self.n, self.box_radius, ctypes.byref(cfg), ctypes.byref(self._h), err, 512), err)

    def close(self) -> None:
        if self._h:
            lib().ankh_plan_destroy_v1(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def energy(self, positions, sources) -> EnergyReport:
        """Host arrays (copied to HBM on the plan's stream)."""
        pos = _as_host(positions, 3)
        src = _as_host(sources, 10)
        self._check_n(pos, src)
        rep = _Report()
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_energy_v1(self._h, _ptr(pos), _ptr(src), ctypes.byref(rep), err, 512), err)
        return EnergyReport._from_c(rep)

    def forces(self, positions, sources, out=None):
        """Energy and forces F = -dE/dx (n x 3) of host arrays: (EnergyReport, forces).
        ``out``: a C-contiguous float64 (n, 3) array to receive the forces (a
        page-locked one is filled at the full copy rate; a fresh pageable
        array per call costs its page faults)."""
        pos = _as_host(positions, 3)
        src = _as_host(sources, 10)
        self._check_n(pos, src)
        rep = _Report()
        err = ctypes.create_string_buffer(512)
        if out is None:
            forces = np.zeros((pos.shape[0], 3), dtype=np.float64)
        else:
            forces = out
            if (not isinstance(forces, np.ndarray) or forces.dtype != np.float64 or
                    forces.shape != (pos.shape[0], 3) or not forces.flags.c_contiguous or
                    not forces.flags.writeable):
                raise ValueError("forces: out must be a writable C-contiguous float64 array of shape (n, 3)")
        _check(lib().ankh_plan_forces_v1(self._h, _ptr(pos), _ptr(src), _ptr(forces), ctypes.byref(rep), err,
                                         512), err)
        return EnergyReport._from_c(rep), forces

    def derivatives(self, positions, sources, forces: bool = True, _dsrc_out=None):
        """Energy, forces F = -dE/dx (n x 3, or None with ``forces=False``) and
        the moment gradient dE/ds (n x 10, the stored moment layout: dE/dq is
        the potential, dE/dmu minus the field, dE/dTheta per stored component)
        of host arrays: (EnergyReport, forces, dsrc)."""
        pos = _as_host(positions, 3)
        src = _as_host(sources, 10)
        self._check_n(pos, src)
        rep = _Report()
        err = ctypes.create_string_buffer(512)
        f = np.zeros((pos.shape[0], 3), dtype=np.float64) if forces else None
        dsrc = _dsrc_out if _dsrc_out is not None else np.zeros((pos.shape[0], 10), dtype=np.float64)
        _check(lib().ankh_plan_derivatives_v1(self._h, _ptr(pos), _ptr(src), _ptr(f) if f is not None else None,
                                              _ptr(dsrc), ctypes.byref(rep), err, 512), err)
        return EnergyReport._from_c(rep), f, dsrc

    def field(self, positions, sources) -> np.ndarray:
        """The electric field at every particle, -dE/dmu (n x 3): the quantity
        an induced-dipole solve iterates on (``induced_dipoles``)."""
        # the n x 10 result buffer is kept between calls (the induced-dipole
        # solve evaluates a field per iteration; a fresh 80 B / particle array
        # would be page-faulted in every time); the caller gets a copy
        buf = getattr(self, "_field_buf", None)
        if buf is None or buf.shape[0] != np.shape(positions)[0]:
            buf = self._field_buf = np.empty((np.shape(positions)[0], 10), dtype=np.float64)
        return -self.derivatives(positions, sources, forces=False, _dsrc_out=buf)[2][:, 1:4]

    def set_positions(self, positions) -> None:
        """Bind host positions (copied, validated, binned and sorted once) for
        repeated ``energy_sources`` calls with new moments."""
        pos = _as_host(positions, 3)
        if pos.shape[0] != self.n:
            raise InvalidArgument("fmm_energy: invalid system: positions and sources must have equal length")
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_set_positions_v1(self._h, _ptr(pos), err, 512), err)

    def energy_sources(self, sources) -> EnergyReport:
        """Evaluate new host moments (n x 10) at the bound positions."""
        src = _as_host(sources, 10)
        if src.shape[0] != self.n:
            raise InvalidArgument("fmm_energy: invalid system: positions and sources must have equal length")
        rep = _Report()
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_energy_sources_v1(self._h, _ptr(src), ctypes.byref(rep), err, 512), err)
        return EnergyReport._from_c(rep)

    def energy_device(self, positions, sources, stream: int = 0) -> EnergyReport:
        """Device tensors (torch CUDA float64, contiguous N x 3 / N x 10)."""
        self._check_dev(positions, sources)
        rep = _Report()
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_energy_device_v1(
            self._h, ctypes.c_void_p(positions.data_ptr()), ctypes.c_void_p(sources.data_ptr()),
            ctypes.c_void_p(stream), ctypes.byref(rep), err, 512), err)
        return EnergyReport._from_c(rep)

    def enqueue(self, positions, sources, stream: int = 0) -> None:
        """Queue an evaluation of device tensors without synchronising."""
        self._check_dev(positions, sources)
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_enqueue_v1(self._h, ctypes.c_void_p(positions.data_ptr()),
                                          ctypes.c_void_p(sources.data_ptr()),
                                          ctypes.c_void_p(stream), err, 512), err)

    def energies_to(self, out, stream: int = 0) -> None:
        """Queue a device copy of {e_self, e_near, e_far, e_periodic_far} into
        ``out`` (CUDA float64 tensor with >= 4 elements) for a device collective."""
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_energies_device_v1(self._h, ctypes.c_void_p(out.data_ptr()),
                                                  ctypes.c_void_p(stream), err, 512), err)

    # ---- multi-GPU shards -------------------------------------------------
    def attach_nccl(self, unique_id: bytes) -> None:
        """Join the NCCL communicator of all shards (``nccl_unique_id()`` from
        rank 0, broadcast by the caller); reports then carry job totals."""
        if len(unique_id) != 128:
            raise InvalidArgument("NCCL unique id must be 128 bytes")
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_attach_nccl_v1(self._h, unique_id, err, 512), err)

    def attach_loopback(self) -> None:
        """Diagnostics on one GPU: stand-in exchange (device copies for the
        leaf all-gather, identity all-reduce) so one shard's whole evaluation
        can be timed; reports then carry this shard's partial sums."""
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_attach_loopback_v1(self._h, err, 512), err)

    def enqueue_phase(self, phase: int, positions, sources, stream: int = 0) -> None:
        """Caller-driven shard exchange: phase 1 = binning..this shard's P2M,
        phase 2 = M2M..final reduction (after the leaf level is completed)."""
        self._check_dev(positions, sources)
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_enqueue_phase_v1(self._h, int(phase), ctypes.c_void_p(positions.data_ptr()),
                                                ctypes.c_void_p(sources.data_ptr()),
                                                ctypes.c_void_p(stream), err, 512), err)

    def leaf_level(self) -> Tuple[int, int, int, int]:
        """(device pointer, first row, end row, row stride in doubles) of the
        Morton-ordered leaf expansions; rows [first, end) are this shard's."""
        ptr = ctypes.c_void_p()
        b, e = ctypes.c_int64(), ctypes.c_int64()
        stride = ctypes.c_int()
        _check(lib().ankh_plan_leaf_level_v1(self._h, ctypes.byref(ptr), ctypes.byref(b),
                                             ctypes.byref(e), ctypes.byref(stride)),
               ctypes.create_string_buffer(b"invalid plan"))
        return int(ptr.value or 0), b.value, e.value, stride.value

    def result(self) -> EnergyReport:
        rep = _Report()
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_result_v1(self._h, ctypes.byref(rep), err, 512), err)
        return EnergyReport._from_c(rep)

    def info(self) -> Dict[str, float]:
        d, o = ctypes.c_int(), ctypes.c_int()
        nl, ni, no, nb = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        rm = ctypes.c_double()
        lib().ankh_plan_info_v1(self._h, ctypes.byref(d), ctypes.byref(o), ctypes.byref(nl),
                                ctypes.byref(ni), ctypes.byref(no), ctypes.byref(rm), ctypes.byref(nb))
        return {"depth": d.value, "order": o.value, "leaves": nl.value, "m2l_instances": ni.value,
                "m2l_operators": no.value, "m2l_rank_mean": rm.value, "device_bytes": nb.value}

    def expansions(self):
        """Per-level expansions of the last evaluation: list of (8^l, K) arrays."""
        inf = self.info()
        depth, L = inf["depth"], inf["order"]
        K = L ** 3
        total = sum(8 ** l for l in range(depth + 1)) * K
        out = np.zeros(total)
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_expansions_v1(self._h, _ptr(out), total, err, 512), err)
        res, o = [], 0
        for l in range(depth + 1):
            cnt = 8 ** l * K
            res.append(out[o:o + cnt].reshape(8 ** l, K))
            o += cnt
        return res

    def m2l_factors(self, level: int, offset) -> Tuple[np.ndarray, np.ndarray]:
        L = self.info()["order"]
        K = L ** 3
        lm = np.zeros(K * K)
        rm = np.zeros(K * K)
        rank = ctypes.c_int(0)
        off = np.asarray(offset, dtype=np.int32)
        err = ctypes.create_string_buffer(512)
        _check(lib().ankh_plan_m2l_factors_v1(self._h, int(level),
                                              off.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                              _ptr(lm), _ptr(rm), K, ctypes.byref(rank), err, 512), err)
        k = rank.value
        return lm[: k * K].reshape(k, K), rm[: k * K].reshape(k, K)

    def _check_n(self, pos: np.ndarray, src: np.ndarray) -> None:
        if pos.shape[0] != self.n or src.shape[0] != self.n:
            raise InvalidArgument("fmm_energy: invalid system: positions and sources must have equal length")

    def _check_dev(self, positions, sources) -> None:
        import torch

        for t, c in ((positions, 3), (sources, 10)):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
                    and t.is_contiguous() and t.numel() == self.n * c):
                raise InvalidArgument("device inputs must be contiguous CUDA float64 tensors of shape (n, 3) / (n, 10)")
