/* ankh_b200 -- B200-native (sm_100a) drop-in for the reference's energy call.
 *
 * C-ABI of libankh_b200.so.  Plain pointers and sizes only.  Each entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj/core):
 *
 *   ankh_fmm_energy_v1   <- ankh::fmm_energy(const ParticleSystem&,
 *                                            const EwaldConfig&, int threads)
 *                           include/ankh/fmm.hpp:98-99, src/fmm.cpp:383-436
 *   ankh_plan_*_v1       <- the same call split into a cached, geometry-only
 *                           plan (build_m2l_cache fmm.cpp:141-179,
 *                           build_periodic_operator fmm.cpp:333-377) and a
 *                           per-system evaluation (fmm.cpp:397-434).  The
 *                           reference rebuilds the plan on every call.
 *   ankh_leaf_csr_v1     <- ankh::build_tree, include/ankh/octree.hpp:41,
 *                           src/octree.cpp:27-45 (bucket contents, bit-exact)
 *
 * Data layout is byte-identical to the reference's storage:
 *   positions : n x 3 doubles  == std::vector<Vec3>            (types.hpp:13-38)
 *   sources   : n x 10 doubles == std::vector<MultipoleSource> (types.hpp:76-84)
 *               q, mu_x, mu_y, mu_z, Theta_xx, xy, xz, yy, yz, zz
 *
 * Return codes (the C++ wrapper include/ankh_b200.hpp re-throws them as the
 * reference's exception types; `err` receives the reference's message text):
 *   0 ANKH_OK
 *   1 ANKH_INVALID_ARGUMENT  std::invalid_argument (types.cpp:65-79,
 *                            fmm.cpp:385-388, octree.cpp:28, chebyshev.cpp:86)
 *   2 ANKH_DOMAIN_ERROR      std::domain_error "pair_interaction: coincident
 *                            points" (kernel.cpp:161)
 *   3 ANKH_RUNTIME_ERROR     std::runtime_error (unsupported size / plan misuse)
 *   4 ANKH_CUDA_ERROR        CUDA / NCCL failure (no reference counterpart)
 */
#ifndef ANKH_B200_H
#define ANKH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ANKH_OK = 0,
  ANKH_INVALID_ARGUMENT = 1,
  ANKH_DOMAIN_ERROR = 2,
  ANKH_RUNTIME_ERROR = 3,
  ANKH_CUDA_ERROR = 4
};

/* EwaldConfig (types.hpp:96-104) plus execution fields. */
typedef struct ankh_config_v1 {
  double xi;         /* Ewald splitting parameter (default 0.01) */
  int p;             /* image half-width: 0 open, >= 2 periodic (default 15) */
  int order_cheb;    /* Chebyshev order L (default 8) */
  int order_equi;    /* validated, unused by the FMM (types.cpp:73) */
  int depth;         /* octree depth E; 0 = default_depth(N) */
  double svd_tol;    /* M2L singular-value cutoff (default 1e-7) */
  int recip_cutoff;  /* validated, unused (types.cpp:78) */
  /* ---- extensions (no EwaldConfig counterpart) ---- */
  int threads;       /* host threads for plan precompute; <= 0 = all cores */
  int device;        /* CUDA device ordinal; -1 = current */
  int rank;          /* spatial shard index (multi-GPU), 0 for one GPU */
  int world;         /* number of shards; 1 for one GPU */
  int phase_timing;  /* 1 = record per-phase CUDA-event times in the report */
} ankh_config_v1;

/* EnergyReport (types.hpp:123-135).  With world > 1 the energies are this
 * shard's partial sums (e_self and e_periodic_far only on rank 0); the caller
 * all-reduces them. */
typedef struct ankh_report_v1 {
  double e_total, e_self, e_near, e_far, e_periodic_far, e_reciprocal;
  /* wall_times keys of fmm.cpp:409-434, seconds */
  double t_precompute, t_interpolation, t_far_field, t_near_field, t_periodic_far, t_self,
      t_total;
  int depth;         /* tree depth used */
  int order_cheb;
  uint64_t near_pairs;      /* unordered P2P pairs evaluated (this shard) */
  uint64_t far_instances;   /* canonical M2L instances evaluated (this shard) */
  double far_flops;         /* sum over instances of 4kK + 2k (this shard) */
  uint32_t gpu_launches;    /* kernels launched by the last evaluation */
} ankh_report_v1;

typedef struct ankh_plan_v1 ankh_plan_v1;

/* Fill `cfg` with the EwaldConfig defaults (types.hpp:96-104). */
void ankh_config_default_v1(ankh_config_v1* cfg);

/* Drop-in for ankh::fmm_energy.  Host buffers; host<->device copies inside.
 * A process-wide plan cache keyed by (n, box_radius, config, resolved device)
 * makes repeated calls skip the geometry-only precompute.  Reentrant: the
 * cache lock covers only the lookup; an evaluation locks its own plan, so
 * calls on different devices run concurrently.  Runs on cfg->device (or the
 * calling thread's current device when -1) and leaves the current device as
 * it found it. */
int ankh_fmm_energy_v1(size_t n, const double* positions, const double* sources,
                       double box_radius, const ankh_config_v1* cfg, ankh_report_v1* out,
                       char* err, size_t errlen);

/* Forces (the reference computes energies only):
 * forces[3 i + d] = -dE/dx_{i,d} of the same energy ankh_fmm_energy_v1
 * returns (moments held fixed in the lab frame) -- near field by the
 * gradient of pair_interaction (every neighbour pair of the energy's half
 * shell once, Newton's third law; deterministic, no atomics), far field
 * by the adjoint (dE/dM per cell from the M2L factors, the periodic root
 * operator, L2L = M2M^T, L2P = differentiated P2M).  The report holds the
 * energies.  One GPU (a sharded plan raises ANKH_RUNTIME_ERROR). */
int ankh_fmm_forces_v1(size_t n, const double* positions, const double* sources, double box_radius,
                       const ankh_config_v1* cfg, double* forces, ankh_report_v1* out, char* err,
                       size_t errlen);
int ankh_plan_forces_v1(ankh_plan_v1* plan, const double* positions, const double* sources, double* forces,
                        ankh_report_v1* out, char* err, size_t errlen);
/* Forces (optional, n x 3) and the derivative of the energy with respect to
 * every particle's 10 stored moments (optional, n x 10: dE/dq = the
 * potential, dE/dmu = minus the field, dE/dTheta per stored component --
 * an off-diagonal Theta_ij counts for both matrix entries), moments and
 * positions as in ankh_fmm_energy_v1.  The energy is bilinear in the
 * moments, so dsrc is exact for the reference's energy (central differences
 * of fmm_energy reproduce it).  The induced-dipole solve iterates on
 * -dE/dmu (api.induced_dipoles).  At least one output is required. */
int ankh_plan_derivatives_v1(ankh_plan_v1* plan, const double* positions, const double* sources, double* forces,
                             double* dsrc, ankh_report_v1* out, char* err, size_t errlen);

/* The call-level checks of fmm_energy in the reference's order, for wrappers
 * whose containers carry separate position / source lengths:
 * validate_config (fmm.cpp:384, types.cpp:65-79), then validate_system's
 * box_radius rule and its size-mismatch rule (types.cpp:20-26).  The
 * per-particle rules run on the device inside the evaluation. */
int ankh_check_call_v1(const ankh_config_v1* cfg, double box_radius, size_t n_positions,
                       size_t n_sources, char* err, size_t errlen);

/* Plan for n particles in the box [-box_radius, box_radius]^3 under cfg. */
int ankh_plan_create_v1(size_t n, double box_radius, const ankh_config_v1* cfg,
                        ankh_plan_v1** plan, char* err, size_t errlen);
void ankh_plan_destroy_v1(ankh_plan_v1* plan);
/* The same plan with the ANKH-FFT far field (PAPER.md
 * Alg. 4-5): leaf Chebyshev expansions re-interpolated onto equispaced
 * grids of order cfg->order_equi, the far field of every non-adjacent leaf
 * pair (images |I|_inf <= 1) as one circulant quadratic form evaluated with
 * a 6-D DFT (e_far), the far images on the root operator as before
 * (e_periodic_far).  Not the reference's energy: it converges to it as both
 * orders grow (the reference has no such engine; no drop-in parity). */
int ankh_plan_create_fft_v1(size_t n, double box_radius, const ankh_config_v1* cfg, ankh_plan_v1** plan,
                            char* err, size_t errlen);

/* Evaluate with HOST input buffers (copied in on the plan's stream). */
int ankh_plan_energy_v1(ankh_plan_v1* plan, const double* positions, const double* sources,
                        ankh_report_v1* out, char* err, size_t errlen);

/* Evaluate with DEVICE input buffers (same layouts), on `stream`
 * (cudaStream_t; NULL = the plan's own stream).  Synchronises before return. */
int ankh_plan_energy_device_v1(ankh_plan_v1* plan, const double* d_positions,
                               const double* d_sources, void* stream, ankh_report_v1* out,
                               char* err, size_t errlen);

/* Repeated evaluation with fixed positions (the config-4 pattern: moments
 * change, positions and box do not).  set_positions copies the HOST positions,
 * validates them and bins / sorts them once; energy_sources then copies only
 * the HOST moments (n x 10), validates them and runs the evaluation -- no
 * position copy, no re-binning.  Any other evaluation of the plan supersedes
 * the bound positions (ANKH_RUNTIME_ERROR until set again). */
int ankh_plan_set_positions_v1(ankh_plan_v1* plan, const double* positions, char* err,
                               size_t errlen);
int ankh_plan_energy_sources_v1(ankh_plan_v1* plan, const double* sources, ankh_report_v1* out,
                                char* err, size_t errlen);

/* Enqueue an evaluation without synchronising; results are fetched with
 * ankh_plan_result_v1.  Used for device-timed loops and CUDA-graph capture. */
int ankh_plan_enqueue_v1(ankh_plan_v1* plan, const double* d_positions, const double* d_sources,
                         void* stream, char* err, size_t errlen);
int ankh_plan_result_v1(ankh_plan_v1* plan, ankh_report_v1* out, char* err, size_t errlen);

/* Enqueue a device-to-device copy of this shard's {e_self, e_near, e_far,
 * e_periodic_far} (4 doubles) from the last enqueued evaluation into d_out on
 * `stream`, so a collective (e.g. an NCCL all-reduce across shards) can follow
 * on the device without a host round trip. */
int ankh_plan_energies_device_v1(ankh_plan_v1* plan, double* d_out, void* stream, char* err,
                                 size_t errlen);

/* Plan introspection. */
int ankh_plan_info_v1(const ankh_plan_v1* plan, int* depth, int* order, size_t* n_cells_leaf,
                      size_t* m2l_instances, size_t* m2l_operators, double* m2l_rank_mean,
                      size_t* device_bytes);

/* Per-level expansions (levels 0..depth, lex cell order, K = L^3 per cell)
 * from the last evaluation, copied to host `out` (count doubles). */
int ankh_plan_expansions_v1(ankh_plan_v1* plan, double* out, size_t count, char* err,
                            size_t errlen);

/* Leaf CSR of build_tree: offsets[8^depth + 1] and indices[n] (lex leaves,
 * ascending particle index inside a leaf), computed on the GPU. */
int ankh_leaf_csr_v1(size_t n, const double* positions, double box_radius, int depth,
                     uint32_t* leaf_offsets, uint32_t* indices, char* err, size_t errlen);

/* M2L factors the plan uses for (level, offset): k x K row-major each. */
int ankh_plan_m2l_factors_v1(ankh_plan_v1* plan, int level, const int* offset, double* lmat,
                             double* rmat, int max_rank, int* rank, char* err, size_t errlen);

/* ---- multi-GPU shards (cfg.rank / cfg.world) ----
 * A shard computes P2M for its Morton leaf rows, P2P for its Morton leaf
 * range and M2L for the instances whose target it owns.  Two exchanges finish
 * the job: an all-gather of the Morton-ordered leaf expansions (when
 * world | 8^depth) and an all-reduce of the energy/counter vector.
 *
 * (a) NCCL, inside the plan: rank 0 creates an id, every rank attaches it;
 *     afterwards ankh_plan_enqueue_v1 / ankh_plan_energy_*_v1 return JOB totals. */
int ankh_nccl_unique_id_v1(unsigned char* id128, char* err, size_t errlen);
int ankh_plan_attach_nccl_v1(ankh_plan_v1* plan, const unsigned char* id128, char* err,
                             size_t errlen);
/* (b) Caller-driven (in-process shards, other transports): phase 1 runs
 *     binning..P2M of this shard's rows; the caller fills the other rows of
 *     the leaf level (ankh_plan_leaf_level_v1: device pointer, row range,
 *     row stride in doubles); phase 2 runs the rest.  Energies are then this
 *     shard's partials (sum over shards). */
int ankh_plan_enqueue_phase_v1(ankh_plan_v1* plan, int phase, const double* d_positions,
                               const double* d_sources, void* stream, char* err, size_t errlen);
int ankh_plan_leaf_level_v1(ankh_plan_v1* plan, double** d_leaf_level, int64_t* row_begin,
                            int64_t* row_end, int* row_stride);
int ankh_device_copy_v1(void* dst, const void* src, size_t bytes, void* stream, char* err,
                        size_t errlen);
/* One-rank exercise of every NCCL call the shards issue (grouped all-gathers,
 * grouped sum + uint64 MIN all-reduce), eager and captured in a CUDA graph. */
int ankh_nccl_selftest_v1(char* err, size_t errlen);
/* (c) Diagnostics on a one-GPU box: a loopback "collective" that lands the
 *     leaf-level all-gather's bytes with device copies and makes the
 *     all-reduce the identity, so one shard's complete evaluation (with the
 *     exchange in its CUDA graph and P2P concurrent with the far chain) can be
 *     timed.  Energies are this shard's partials. */
int ankh_plan_attach_loopback_v1(ankh_plan_v1* plan, char* err, size_t errlen);
/* (d) Tests on one GPU: the `world` plans of one sharding (ranks 0..world-1,
 *     one process, one device) exchange by stream-ordered pushes -- at its
 *     exchange point each shard copies its own expansion slabs into the other
 *     plans' arrays.  From the second evaluation of the same inputs on, every
 *     shard reports its true partial energies (sum over shards = the job). */
int ankh_plan_attach_push_group_v1(ankh_plan_v1** plans, int world, char* err, size_t errlen);

/* ---- spatial sharding (host only; no device needed) ----
 * Shards own contiguous Morton ranges of leaves; a level-l cell belongs to the
 * shard owning its first descendant leaf.  P2P work is owned by the target
 * leaf; a canonical M2L instance (t, s) (fmm.cpp:246-250) by the owner of t or
 * of s, chosen by a hash of the pair (balanced load), so each unordered pair /
 * instance is counted once. */
int ankh_shard_leaf_range_v1(int depth, int rank, int world, int64_t* morton_begin,
                             int64_t* morton_end);
int ankh_shard_cell_owner_v1(int level, uint32_t lex_cell, int depth, int world);
/* The particle-index slice [i0, i1) whose moments a collective-attached shard
 * validates (whole 256-particle blocks; the slices partition [0, n)). */
int ankh_shard_src_slice_v1(size_t n, int rank, int world, size_t* i0, size_t* i1);
/* Lowest level l >= 1 with world | 8^l (<= depth): a collective-attached shard
 * runs M2M on its own subtree down to l, all-gathers level l and exchanges
 * the M2L halos of levels l+1 .. depth (point to point). */
int ankh_shard_exchange_level_v1(int depth, int world);
/* The M2L halo of one level: Morton cells (ascending) that
 * shard `src` owns and shard `dst` reads -- those that can form an M2L
 * instance with a cell of dst's region (2 cells past its even-aligned faces,
 * periodic wrap).  Needs world | 8^level.  `*count`
 * receives the size; at most `capacity` ids are written to `morton`. */
int ankh_shard_halo_cells_v1(int level, int depth, int periodic, int src, int dst, int world,
                             uint32_t* morton, size_t capacity, size_t* count);
/* Bytes shard `rank` receives / sends per evaluation in the upward exchange
 * at interpolation order `order` (expansion rows padded to 32 doubles):
 * halo != 0 the plan's schedule (all-gather of the exchange level + deep
 * halos), halo == 0 the whole-level all-gather of every level it splits. */
int ankh_shard_exchange_bytes_v1(int depth, int periodic, int order, int rank, int world, int halo,
                                 size_t* recv_bytes, size_t* send_bytes);
/* Canonical M2L instances (level, t, s, offset[3]) owned by `rank` (rank < 0:
 * all), in the plan's grouping order.  `*count` receives the total; at most
 * `capacity` entries are written (pass 0 to query the count). */
int ankh_shard_m2l_instances_v1(int depth, int periodic, int rank, int world, uint32_t* level,
                                uint32_t* t, uint32_t* s, int32_t* offset, size_t capacity,
                                size_t* count);

/* Near-field radial polynomials the plan uses for a given s_max = xi^2 d_max^2
 * (d_max = the largest near-pair distance, 2 sqrt(3) leaf sides): coefficients
 * (14 each, in s = xi^2 r^2) of P(s) = erf(sqrt s)/sqrt s and
 * G(s) = (2/sqrt(pi)) exp(-s) -- the reference's erfc_screen / radial
 * (kernel.cpp:14-51) -- valid for s <= *s_lim, and the fit's measured max
 * relative error.  Diagnostics (no reference counterpart); host only. */
int ankh_radial_fit_v1(double s_max, int* nterms, double* s_lim, double* p, double* g,
                       double* max_err);

/* Measured FP64 (DFMA) throughput of the current device in TFLOP/s: the
 * roofline denominator for the FP64-bound kernels (no reference counterpart). */
double ankh_probe_fp64_tflops_v1(int iters);

/* Measured FP64 tensor-core (DMMA) throughput in TFLOP/s for the MMA shape
 * 0 = m8n8k4 (the M2L kernel's), 1 = m16n8k8, 2 = m16n8k16: the roofline
 * denominator for k_m2l (no reference counterpart). */
double ankh_probe_dmma_tflops_v1(int shape, int iters);
/* Pipe-sharing probe: ms of a kernel whose warps run DFMA chains (mode 0),
 * m8n8k4 DMMAs (mode 1), or half and half (mode 2). */
double ankh_probe_fp64_mix_ms_v1(int mode, int iters_dfma, int iters_dmma);

/* Library version string. */
const char* ankh_version_v1(void);

#ifdef __cplusplus
}
#endif

#endif /* ANKH_B200_H */
