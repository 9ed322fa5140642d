// Device-side declarations shared by the sm_100a kernels and the host plan.
//
// HBM layout (all float64 unless noted):
//   part    : N x 14   particle records sorted by lex leaf id, ascending input
//                      index inside a leaf (== build_tree bucket order,
//                      octree.cpp:27-45): x y z q mux muy muz Txx Txy Txz Tyy
//                      Tyz Tzz tr(Theta)   (112 B, 16-B aligned; a leaf's
//                      records are one contiguous byte range for bulk copies)
//   leaf_off: 8^E + 1  uint32 leaf CSR offsets into `part`
//   exp     : sum_l 8^l x Kp  expansions, level-major, Morton cell order
//   factors : per M2L operator, L (kp x Kp) then R (kp x Kp), zero padded
//   inst    : uint2 (t, s) canonical M2L instances grouped by operator
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace ankh_b200 {

/// Device-side bounds checks of the checked build (make checked:
/// -DANKH_CHECKED, variants/libankh_b200_checked.so).  compute-sanitizer is
/// not available on the GPU pool, so the checked library is this engine's
/// own memcheck: every staged shared-memory index and scattered global index
/// on the hot path is asserted, and plan allocations carry guard zones
/// verified after each evaluation (plan.cpp).  Compiled out otherwise.
#ifdef ANKH_CHECKED
#define ANKH_DASSERT(cond)                                                                  \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("ANKH_DASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                  \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define ANKH_DASSERT(cond) \
  do {                     \
  } while (0)
#endif

/// Dynamic shared-memory opt-in above 48 KB.  CUDA keeps the attribute per
/// device and per kernel, so a launcher records, per kernel instantiation,
/// the devices it has been set on (bit d of `done`).  Lock-free: two threads
/// racing on a new device both set the same value, which is harmless.
template <class Kernel>
inline void smem_opt_in(std::atomic<unsigned long long>& done, Kernel* kernel, std::size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  done.fetch_or(bit, std::memory_order_acq_rel);
}

constexpr int kRec = 14;          // doubles per particle record (112 B: x y z q mu Theta tr)
constexpr int kM2LTile = 64;      // instances per M2L CTA
constexpr int kM2LChunk = 32;     // node columns per staged chunk
constexpr int kMaxKp8 = 16;       // ranks up to 128

/// Morton decode: every 3rd bit (x in bit 3k+2, y in 3k+1, z in 3k), as
/// shard.cpp's morton3 encodes.  Expansions at every level are stored in
/// Morton order (children of cell m are 8m..8m+7; a shard's cells are one
/// contiguous slice); particles and leaf CSR stay in the reference's lex order.
__host__ __device__ inline unsigned morton_compact3(unsigned v) {
  v &= 0x09249249u;
  v = (v ^ (v >> 2)) & 0x030c30c3u;
  v = (v ^ (v >> 4)) & 0x0300f00fu;
  v = (v ^ (v >> 8)) & 0x030000ffu;
  v = (v ^ (v >> 16)) & 0x000003ffu;
  return v;
}
__host__ __device__ inline unsigned morton_to_lex(unsigned m, int n) {
  const unsigned x = morton_compact3(m >> 2), y = morton_compact3(m >> 1), z = morton_compact3(m);
  return (x * static_cast<unsigned>(n) + y) * static_cast<unsigned>(n) + z;
}

/// Row stride (doubles) of one cell's expansion in HBM: K = L^3 rounded up to
/// 32 (zero tail), so every row starts 256-B aligned and the M2L stager moves
/// 16-B pieces without bounds checks.
__host__ __device__ constexpr int exp_stride(int k) { return (k + 31) / 32 * 32; }

// Everything a shard contributes additively sits in red[] so one all-reduce
// (sum) combines shards: energies, the pair counter (exact in a double up to
// 2^53) and the error flags (> 0 means raised somewhere).
// slots [0, kRedShared) are all-reduced across shards; the rest stay per shard
enum RedSlot {
  kESelf = 0, kENear, kEFar, kEPeriodic, kDuplicate, kCoincident, kRedShared,
  kNearPairs = kRedShared, kRedCount = 8
};

// streamed host path: at most this many moment chunks (per-chunk leaf lists)
constexpr int kMaxStreamChunks = 32;
/// Streamed host path: chunk c holds particles [start[c], start[c + 1]),
/// c < n; starts are multiples of 256 (k_bin's block layout).
struct StreamChunks {
  unsigned start[kMaxStreamChunks + 1];
  int n;
};

struct DevResult {
  double red[kRedCount];
  unsigned long long min_nonfinite;  // lowest index with a non-finite value (same on every shard)
  unsigned long long min_outside;    // lowest finite index outside the box (follows min_nonfinite:
                                     // the two are MIN-reduced together across shards)
  int any_multipole;                 // some particle has mu or Theta != 0
  unsigned spare;
};

struct M2LTile {
  int op;       // operator index
  int level;    // tree level (selects the expansion slice)
  int begin;    // first instance
  int count;    // instances in this tile (<= kM2LTile)
};

struct M2LOp {
  long long factor_off;  // offset (doubles) of L; R follows at + kp*Kp
  int kp;                // padded rank (multiple of 8)
  int rank;
};

// ---- launchers (defined in the .cu files) ----
/// Particles [i0, min(i1, n)) (i0 a multiple of 256): keys, leaf histogram
/// (counts) with arrival slots in idx, position flags; leafmax (optional,
/// zeroed): each leaf's largest particle index.
void launch_bin(const double* pos, const double* src, std::size_t n, double box_radius,
                double inv_side, int n_axis, unsigned* keys, unsigned* idx, unsigned* counts,
                DevResult* res, cudaStream_t st, const unsigned char* need = nullptr, std::size_t i0 = 0,
                std::size_t i1 = ~std::size_t{0}, unsigned* leafmax = nullptr);
/// Single-pass exclusive scan (k_bin.cu k_scan): the state -- scan_tiles(n)
/// status words and two counters -- is zeroed once and resets itself.
struct ScanWork {
  unsigned long long* status;
  unsigned* ctr;
};
std::size_t scan_tiles(std::size_t n);
void launch_scan(const unsigned* in, unsigned* out, std::size_t n, ScanWork w, cudaStream_t st);
std::size_t sort_temp_bytes(std::size_t n);
void launch_sort(void* temp, std::size_t temp_bytes, const unsigned* keys_in, unsigned* keys_out,
                 const unsigned* idx_in, unsigned* idx_out, std::size_t n, int end_bit, cudaStream_t st);
/// hd[n] = H D^n, n = 0..2 (3 x L x L, host order) into the P2M constant bank.
void upload_p2m_basis(int order, const double* hd, cudaStream_t st);
// list != nullptr (L <= 6 only): the leaves list[bounds[0] .. bounds[1]),
// list_count of them (streamed host path)
/// Also the self-energy summand sum of every visited leaf (kernel.cpp:206-213
/// without the -xi/sqrt(pi) factor) into self_leaf[Morton leaf].
void launch_p2m(const double* part, const unsigned* leaf_off, int depth, int order,
                double box_radius, const double* hd, double* exp_leaf, const DevResult* res,
                double* self_leaf, double xi, unsigned m_begin, unsigned m_end, cudaStream_t st, const unsigned* list = nullptr,
                const unsigned* bounds = nullptr, unsigned list_count = 0);
// streamed host path (k_bin.cu): one arrived chunk [i0, i1) of the moments --
// validation, self-energy partials, records scattered to their sorted slots
void launch_src_chunk(const double* pos, const double* src, const unsigned* inv, std::size_t i0,
                      std::size_t i1, DevResult* res, double* part, cudaStream_t st,
                      const unsigned* keys = nullptr, unsigned* leaf_mp = nullptr);
// per-leaf readiness chunk (P2M: own records; P2P: + the 13 half-shell
// neighbours) from each leaf's largest particle index (launch_bin leafmax),
// per-chunk leaf lists and their bounds (bounds[0..C] P2M, bounds[C+1..2C+1]
// P2P); cnt_cursor: 4 kMaxStreamChunks uints of scratch
void launch_stream_lists(const unsigned* leafmax, int depth, int periodic, const StreamChunks& ch,
                         unsigned char* ready, unsigned* cnt_cursor, unsigned* bounds, unsigned* list_p2m,
                         unsigned* list_p2p, cudaStream_t st);
/// The upward pass (M2M) in one launch: parents [p_begin, p_begin + p_count)
/// of level `first` (Morton; p_count 0: all), then every coarser level down
/// to `top`, each cell by the last of its children's CTAs to finish.
/// counters: m2m_counter_count(depth) zeroed uints (self-resetting).
std::size_t m2m_counter_count(int depth);
void launch_m2m_chain(double* exp, const long long* level_off, int first, int top, int order,
                      const double* m2m, unsigned* counters, cudaStream_t st, unsigned p_begin = 0,
                      unsigned p_count = 0);
void launch_m2l(const double* exp, const long long* level_off, const double* factors,
                const M2LOp* ops, const M2LTile* tiles, int n_tiles_class, int kp8,
                const int* tile_ids, const uint2* inst, int K, int Kp, double* far_partial,
                cudaStream_t st);
/// Radial polynomials of the near field in s = xi^2 r^2 (host_numerics.hpp
/// fit_radial): P(s) = erf(sqrt s)/sqrt s, G(s) = (2/sqrt(pi)) exp(-s).
struct P2PRadial {
  int nterms;    // 6..10, 12: fitted on [0, s_lim], no range test; 14: libm past s_lim
  double s_lim;
  double p[14], g[14];
};

/// Near field: one CTA per target leaf (near_partial[leaf]).  Returns the
/// number of near partials written.
// list != nullptr: the target leaves are list[bounds[0] .. bounds[1]) (Morton
// indices, list_grid of them -- the host knows the count), partials still
// indexed by leaf - leaf_begin (streamed host path)
/// leaf_mp[lex leaf] != 0: the leaf holds a dipole or quadrupole (written
/// with the records: launch_bucket_gather / launch_src_gather / launch_src_chunk).
int launch_p2p(const double* part, const unsigned* leaf_off, const unsigned* leaf_mp, int depth, int periodic,
               double period, double xi, const P2PRadial& rad, int cap, int leaf_begin,
               int leaf_end, double* near_partial, unsigned long long* pair_count, DevResult* res,
               cudaStream_t st, const unsigned* list = nullptr, const unsigned* bounds = nullptr,
               int list_grid = 0, int bspan = 1);
int p2p_max_cap();
void launch_periodic_gen(double* gen, int order, double box_radius, double xi, int p,
                         cudaStream_t st);
/// scratch: periodic_eval_scratch_doubles(order) doubles when nonzero (the
/// working set past the shared-memory size)
void launch_periodic_eval(const double* root, const double* to_equi, const double* spec_re,
                          int order, double* out, cudaStream_t st, double* scratch = nullptr);
std::size_t periodic_eval_scratch_doubles(int order);
// Runtime-order P2M / M2M (k_generic.cu) for orders past the compiled ones
constexpr unsigned kM2MGenGlobalCtas = 148;
void launch_p2m_generic(const double* part, const unsigned* leaf_off, int depth, int order, double box_radius,
                        const double* hd, double* exp_leaf, double* self_leaf, double xi, unsigned m_begin,
                        unsigned m_end, cudaStream_t st);
std::size_t m2m_generic_scratch_doubles(int order);
/// h_level_off: the host copy of the level offsets
void launch_m2m_generic(double* exp, const long long* h_level_off, int first, int top, int order,
                        const double* m2m, double* scratch, cudaStream_t st, unsigned p_begin = 0,
                        unsigned p_count = 0);
void launch_finalize(const double* near_partial, int n_near, const unsigned long long* pair_count,
                     int n_count, const double* far_partial, int n_far, const double* self_partial,
                     int n_self, double self_scale, const double* periodic, int use_periodic,
                     int include_self, double* scratch, DevResult* res, cudaStream_t st);
std::size_t finalize_scratch_bytes();
/// Bound-positions path: moment validation + self-energy partials (k_bin's
/// block layout) and the records gathered through an existing sorted index.
/// keys[i]: particle i's lex leaf; leaf_mp (zeroed by the caller) is OR-ed.
void launch_src_gather(const double* pos, const double* src, const unsigned* sorted,
                       std::size_t n, DevResult* res, double* part, cudaStream_t st,
                       const unsigned* keys, unsigned* leaf_mp);
/// counts != nullptr: also zero counts[0, n_counts) (the leaf histogram).
void launch_init_result(DevResult* res, cudaStream_t st, int any_multipole = 0,
                        unsigned* counts = nullptr, unsigned n_counts = 0);
/// Counting sort into leaves (after launch_bin with counts): scan -> offsets,
/// scatter, per-leaf ascending order (sorted = the leaf CSR's index array) and
/// the gather of 112-B records.  unsorted / scratch: N uints each; need
/// (optional, per lex leaf): only those leaves are sorted and gathered;
/// part == nullptr: sort only.  launch_bin with src == nullptr bins and
/// validates positions only.
/// inv (optional): inv[sorted[j]] = j, the sorted slot of every particle.
void launch_bucket_gather(ScanWork scan, const double* pos, const double* src,
                          const unsigned* keys, const unsigned* slots, const unsigned* counts,
                          unsigned* offsets, unsigned* unsorted, unsigned* scratch,
                          unsigned* sorted, std::size_t n, int n_leaves,
                          const unsigned char* need, double* part, cudaStream_t st,
                          bool check_src = false, DevResult* res = nullptr, unsigned* leaf_mp = nullptr,
                          unsigned* inv = nullptr);
double probe_fp64_tflops(int iters);
/// ms of k_mix<mode> (k_probe.cu): DFMA-only, DMMA-only, or half/half warps
double probe_fp64_mix_ms(int mode, int it_f, int it_m);
double probe_dmma_tflops(int shape, int iters);

// M2L instance lists on the GPU (k_inst.cu)
std::size_t m2l_instances_device(int depth, int periodic, int rank, int world, const int4* d_offs,
                                 int n_offs, unsigned* d_counts, unsigned* d_offsets,
                                 std::size_t n_blocks_total, void* d_temp, std::size_t temp_bytes,
                                 uint2* inst, cudaStream_t st);
std::size_t m2l_instances_temp_bytes(std::size_t n_blocks_total);
std::size_t m2l_instance_blocks(int depth, int n_offs);
int m2l_instance_block_size();

// M2L operator compression on the GPU (k_svd.cu)
struct M2LPack {
  long long factor_off;  // operator block (as M2LOp)
  int cls;               // symmetry class (row of the class factor arrays)
  int r0, rows, kp;      // rank rows [r0, r0 + rows) of the class factors
  int perm_off;          // node permutation (K ints) in the perm array
};
std::size_t jacobi_svd_smem(int K);
void launch_jacobi_svd(const double* c_all, int n_classes, int K, double skip_rel, double* w_all,
                       double* sig_all, int* sweeps, cudaStream_t st);
void launch_svd_factors(const double* c_all, const double* w_all, const double* sig_all,
                        const int* order, const int* rank, int n_classes, int K, double* lf,
                        double* rf, cudaStream_t st);
void launch_m2l_pack(const M2LPack* ops, int n_ops, int max_rows, const int* perms,
                     const double* lf, const double* rf, int K, int Kp, double* factors,
                     cudaStream_t st);
/// Halo rows (k_halo.cu): pack buf[j] = exp[row_off[j] ..+Kp] or, unpack,
/// the reverse; Kp even, row offsets 16-B aligned.
void launch_halo_rows(double* exp, const long long* row_off, long long n_rows, int Kp, double* buf,
                      bool unpack, cudaStream_t st);
// Forces (k_forces.cu): near-field gradient over the full
// 27-leaf stencil (f_near, sorted record order, F = -grad); per-cell dE/dM
// (loc, the expansion layout) from M2L instances -- tiles (level, parity
// class, first class index, count <= 32), op_of[level * 343 + offset slot] =
// (first operator block, blocks) -- the periodic root term, L2L, L2P (f_far);
// then forces[sorted[j]] = f_near[j] + f_far[j].
// With d_near and f_near == nullptr: the moment derivatives alone (no pair
// gradient).  With f_slot (13 x slot_stride doubles, zeroed by the caller; forces only):
// the half shell with Newton's third law, the neighbours' sums per direction
// slot, added by launch_force_out.
int force_max_cap();
int force_half_max_cap();
void launch_force_near(const double* part, const unsigned* leaf_off, const unsigned* leaf_mp, int depth,
                       int periodic, double period, double xi, const P2PRadial& rad, int cap, double* f_near,
                       cudaStream_t st, double* d_near = nullptr, double* f_slot = nullptr,
                       std::size_t slot_stride = 0);
std::size_t m2l_local_smem(int Kp);
void launch_m2l_local(const double* exp, double* loc, const long long* level_off, const double* factors,
                      const M2LOp* ops, const int2* op_of, const int4* tiles, int n_tiles, int Kp, int periodic,
                      cudaStream_t st);
void launch_periodic_local(const double* root, const double* to_equi, const double* gen, int order,
                           double* loc_root, cudaStream_t st);
void launch_l2l(const double* loc_parent, double* loc_child, int parent_level, int order, const double* m2m,
                cudaStream_t st);
void launch_l2p(const double* part, const unsigned* leaf_off, int depth, int order, double rb, const double* hd4,
                const double* loc_leaf, double* f_far, cudaStream_t st, double* d_far = nullptr);
/// dE/ds (n x 10, the caller's order) = near + far (sorted order) + the
/// self energy's derivative (include_self)
void launch_dsrc_out(const double* d_near, const double* d_far, const double* part, const unsigned* sorted,
                     std::size_t n, double xi, int include_self, double* out, cudaStream_t st);
void launch_force_out(const double* f_near, const double* f_far, const unsigned* sorted, std::size_t n,
                      double* out, cudaStream_t st, const double* f_slot = nullptr, std::size_t slot_stride = 0);
// ANKH-FFT far field (k_fft.cu): the leaf-level
// equispaced engine.  Arrays: X / tmp [cells][NF] double2, diag Pc^3 NF doubles.
struct FftShape {
  int n, Pc, Lu, Pn, NF;
  long long energy_blocks;  // partials written by launch_fft_far
};
FftShape fft_shape(int depth, int order_equi);
void launch_fft_precompute(const FftShape& s, int depth, double rb, double xi, int periodic, double2* tmp_a,
                           double2* tmp_b, double* diag, cudaStream_t st);
void launch_fft_far(const FftShape& s, const double* exp_leaf, int KS, int depth, int order_cheb, const double* E,
                    double2* x0, double2* x1, const double* diag, double* partial, cudaStream_t st);
void launch_dup_check(const unsigned* keys_sorted, const unsigned* idx_sorted, const double* pos,
                      std::size_t n, DevResult* res, cudaStream_t st);

}  // namespace ankh_b200
