// The B200 evaluation plan: geometry-only precompute resident in HBM plus the
// per-evaluation launch sequence.  One plan per (n, box radius, config).
#pragma once

#include <chrono>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ankh_b200.h"
#include "collective.hpp"
#include "kernels.cuh"

namespace ankh_b200 {

struct AnkhError : std::runtime_error {
  int code;
  AnkhError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define ANKH_CUDA(call)                                                                 \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::ankh_b200::AnkhError(ANKH_CUDA_ERROR, std::string(#call) + ": " +         \
                                                        cudaGetErrorString(e_));        \
  } while (0)

/// Makes `dev` current for a scope and restores the caller's device after:
/// every plan entry point runs on its plan's device, whatever the calling
/// thread has selected (one thread may drive plans on several GPUs).
struct DeviceGuard {
  explicit DeviceGuard(int dev, bool nothrow = false) {
    if (dev < 0 || cudaGetDevice(&prev_) != cudaSuccess) return;
    if (prev_ != dev) {
      const cudaError_t e = cudaSetDevice(dev);
      if (e == cudaSuccess)
        restore_ = true;
      else if (!nothrow)
        ANKH_CUDA(e);
    }
  }
  ~DeviceGuard() {
    if (restore_) cudaSetDevice(prev_);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;

 private:
  int prev_ = -1;
  bool restore_ = false;
};

/// Temporary device buffers from the stream-ordered pool (cudaMallocAsync),
/// released on the same stream at scope exit.
struct DeviceScratch {
  explicit DeviceScratch(cudaStream_t s) : st(s) {}
  template <class T>
  T* alloc(std::size_t count) {
    void* q = nullptr;
    ANKH_CUDA(cudaMallocAsync(&q, (count ? count : 1) * sizeof(T), st));
    ptrs.push_back(q);
    return static_cast<T*>(q);
  }
  DeviceScratch(const DeviceScratch&) = delete;
  DeviceScratch& operator=(const DeviceScratch&) = delete;
  ~DeviceScratch() {
    for (void* q : ptrs) cudaFreeAsync(q, st);
  }
  cudaStream_t st;
  std::vector<void*> ptrs;
};

/// types.cpp:9-14
int default_depth(std::size_t n);
/// types.cpp:65-79 (throws AnkhError(ANKH_INVALID_ARGUMENT, same message))
void validate_config(const ankh_config_v1& c);

struct OpInfo {
  int level;
  std::int64_t key;
  int rank;
  int first_op;    // device op index of the first row block
  int n_blocks;
};

class Plan {
 public:
  /// engine 0: the reference's SVD-compressed M2L (the drop-in); 1: the
  /// ANKH-FFT leaf-level far field (k_fft.cu, L_u = cfg.order_equi).
  Plan(std::size_t n, double box_radius, const ankh_config_v1& cfg, bool csr_only = false, int engine = 0);
  ~Plan();
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;

  /// Enqueue one evaluation reading device inputs (n x 3, n x 10).
  void enqueue(const double* d_pos, const double* d_src, cudaStream_t st);
  /// Enqueue including the host->device copy of host inputs.
  void enqueue_host(const double* h_pos, const double* h_src, cudaStream_t st);
  /// Repeated evaluation with fixed positions:
  /// copy, validate, bin and sort the positions once ...
  void set_positions(const double* h_pos, cudaStream_t st);
  /// ... then evaluate new moments (host n x 10) without re-copying or
  /// re-binning the positions.
  void enqueue_sources(const double* h_src, cudaStream_t st);
  /// Wait for the last evaluation and fill the report (throws on validation errors).
  void result(ankh_report_v1* out);
  /// Energy evaluation plus the forces F = -dE/dx (n x 3, the caller's particle
  /// order) into host memory (one GPU).
  void forces(const double* h_pos, const double* h_src, double* h_forces, ankh_report_v1* out);
  /// Forces (h_forces, n x 3, optional) and the derivative of the energy with
  /// respect to every particle's 10 moments (h_dsrc, n x 10, optional: the
  /// potential dE/dq, minus the field -dE/dmu, the field gradient dE/dTheta
  /// per stored component) -- the induced-dipole machinery.
  void derivatives(const double* h_pos, const double* h_src, double* h_forces, double* h_dsrc,
                   ankh_report_v1* out);

  void expansions(double* out, std::size_t count);
  void m2l_factors(int level, const int* offset, double* lmat, double* rmat, int max_rank,
                   int* rank);
  void leaf_csr(std::uint32_t* offsets, std::uint32_t* indices);
  /// Enqueue a device copy of {e_self, e_near, e_far, e_periodic} (4 doubles).
  void energies_to_device(double* d_out, cudaStream_t st);

  /// Shard exchange driven by the caller (in-process shards, tests): phase 1
  /// runs validation/binning/sort/gather and this shard's P2M; the caller then
  /// completes the Morton leaf level (rows outside [p2m_begin, p2m_end)); phase
  /// 2 runs M2M, M2L, P2P, the periodic term and the final reduction.
  void enqueue_phase(int phase, const double* d_pos, const double* d_src, cudaStream_t st);
  /// Device pointer to the Morton-ordered leaf level (rows of Kp doubles) and
  /// this shard's P2M row range.
  double* leaf_level(std::int64_t* begin, std::int64_t* end, int* row_stride);
  double* expansions_base() const { return d_exp_; }
  /// Receive buffer of this shard's halo rows from shard `src` (nullptr if none).
  double* halo_recv_from(int src) const;
  /// Attach an NCCL (or other) collective: the plan then all-gathers the leaf
  /// level and all-reduces the result itself; reports carry job totals.
  void attach_collective(Collective* c);

  cudaStream_t stream() const { return stream_; }
  int device() const { return device_; }

  // ---- geometry (public for introspection) ----
  std::size_t n = 0;
  double rb = 1.0;
  ankh_config_v1 cfg{};
  int depth = 1, L = 2, K = 8, Kp = 32, nax = 2, n_leaves = 8;
  bool periodic = false;
  std::size_t m2l_instances = 0, m2l_operators = 0;
  double m2l_rank_mean = 0.0, far_flops = 0.0;
  std::size_t device_bytes = 0;
  // upward exchange per evaluation (shards with a collective): bytes this
  // shard receives -- the all-gathered coarse level plus the deep-level halos
  std::size_t exchange_recv_bytes = 0, exchange_send_bytes = 0;
  double precompute_seconds = 0.0;
  bool precompute_reported = false;

 private:
  void build_all(std::chrono::steady_clock::time_point t0);
  void release() noexcept;
  void build_geometry();
  void build_m2l();
  void build_periodic();
  void build_fft();
  bool fft_ = false;
  FftShape fft_shape_{};
  double *d_fft_E_ = nullptr, *d_fft_diag_ = nullptr;
  double2 *d_fft_x0_ = nullptr, *d_fft_x1_ = nullptr;
  void allocate();
  void* dalloc(std::size_t bytes);
  // checked build (-DANKH_CHECKED): guard zones after the plan buffers
  void check_guards();
  static constexpr std::size_t kGuardBytes = 256;
  static constexpr unsigned char kGuardByte = 0xA5;
  std::vector<std::pair<void*, std::size_t>> guards_;
  /// mode 0: whole evaluation; 1: up to this shard's P2M; 2: from M2M on.
  // mode 0: full evaluation; 1 / 2: halves around a caller-driven shard
  // exchange; 3: moments only (positions bound by set_positions)
  void launch_all(const double* d_pos, const double* d_src, cudaStream_t st, int mode = 0);
  // Streamed host path (enqueue_host, one GPU, L <= 6): positions first, then
  // the moments in chunks on a copy stream; each chunk's records are scattered
  // to their sorted slots as it lands, and P2M / P2P run on the leaves whose
  // records (P2P: and those of their 13 half-shell neighbours) are complete,
  // so the PCIe copy overlaps the evaluation.  Bit-identical to enqueue().
  bool stream_eligible() const;
  void stream_setup();
  // positions chunks pos_ev[0..pch_.n) (nullptr: already in d_pos_) are
  // binned as they land; the leaf lists run beside the sort on side_stream_
  void stream_positions(cudaStream_t st, DevResult* res, const cudaEvent_t* pos_ev,
                        const std::function<void(const std::string&)>& mark = {},
                        cudaEvent_t after_inverse = nullptr);
  void enqueue_streamed(const double* h_pos, const double* h_src, cudaStream_t st);
  void enqueue_streamed_launch(const double* h_pos, const double* h_src, cudaStream_t st);
  // CUDA-graph replay of the streamed path for repeated page-locked host
  // buffers (h_pos == nullptr: bound positions): copies and kernels of one
  // evaluation in one graph launch, captured on the second such call
  cudaGraphExec_t sgraph_exec_ = nullptr;
  const double *sgraph_pos_ = nullptr, *sgraph_src_ = nullptr;
  const double *sgraph_warm_pos_ = nullptr, *sgraph_warm_src_ = nullptr;
  bool sgraph_warm_ = false;
  std::uint32_t sgraph_launches_ = 0;
  std::vector<long long> sgraph_grid_, last_grids_;  // P2M / P2P chunk grids (captured, last launch)
  bool stream_bound_ = false;  // set_positions built the streamed path's lists
  static constexpr int kMaxStreamChunks = ankh_b200::kMaxStreamChunks;
  int stream_chunks_ = 16;
  bool stream_init_ = false;
  // moment chunks (the first one small: compute starts early) and
  // positions chunks (binned as they land)
  StreamChunks sch_{}, pch_{};
  int stream_pos_chunks_ = 4;
  unsigned *d_inv_ = nullptr, *d_scnt_ = nullptr, *d_sbounds_ = nullptr;
  unsigned* d_leafmax_ = nullptr;  // = d_counts_ + n_leaves + 1 (zeroed with the histogram)
  // the previous evaluation's chunk-list bounds (page-locked copy): P2P chunk
  // grids of one CTA per listed leaf (striding covers a larger list)
  unsigned* h_sbounds_ = nullptr;
  bool h_sbounds_valid_ = false;
  unsigned *d_list_p2m_ = nullptr, *d_list_p2p_ = nullptr;
  int sm_count_ = 148;
  cudaStream_t p2p_stream2_ = nullptr;  // odd chunks' P2P (tails overlap the next chunk's start)
  unsigned char* d_ready_ = nullptr;
  cudaStream_t copy_stream_ = nullptr, gather_stream_ = nullptr;
  cudaEvent_t ev_s_start_ = nullptr, ev_s_binned_ = nullptr, ev_s_lists_ = nullptr, ev_s_sorted_ = nullptr,
              ev_s_inv_ = nullptr, ev_s_p2p2_ = nullptr;
  cudaEvent_t ev_s_posc_[kMaxStreamChunks] = {};
  cudaEvent_t ev_s_chunk_[kMaxStreamChunks] = {}, ev_s_gath_[kMaxStreamChunks] = {};
  // phase spans of a streamed evaluation (phases overlap: start/end per phase)
  cudaEvent_t ev_t_[9] = {};
  bool streamed_last_ = false;
  void validate_only(const double* d_pos, const double* d_src, cudaStream_t st);
  std::uint32_t exchange_upward(cudaStream_t st);
  int exch_level_ = 0;  // lowest level split evenly across shards (G | 8^l)
  // Deep levels halo_level_ .. depth are exchanged as M2L halos (the cells
  // within 3 of each peer's region, shard.cpp shard_halo_cells) instead of
  // all-gathered: rows packed peer-major, then level-major, on both sides.
  void build_halo();
  int halo_level_ = 0;
  std::vector<HaloPeer> halo_;
  long long *d_halo_send_off_ = nullptr, *d_halo_recv_off_ = nullptr;
  double *d_halo_send_ = nullptr, *d_halo_recv_ = nullptr;
  long long halo_send_rows_ = 0, halo_recv_rows_ = 0;
  int m2m_top_ = 0;     // highest parent level the far chain still computes (all cells)

  std::unique_ptr<Collective> coll_;
  bool shard_upward_ = false;               // P2M split across shards (+ all-gather)
  std::int64_t p2m_begin_ = 0, p2m_end_ = 0;  // Morton leaf rows this shard computes

  int device_ = 0;
  cudaStream_t stream_ = nullptr;
  cudaStream_t side_stream_ = nullptr;  // far-field chain, concurrent with P2P
  int hi_prio_ = 0;                     // stream priority of the far chain / gathers
  bool m2l_split_ = false;              // leaf-level M2L tiles beside M2M (ANKH_M2L_SPLIT=1)
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  // M2L rank classes run as parallel branches (their tails overlap; the
  // small latency-bound classes hide under the large ones)
  static constexpr int kM2LStreams = 3;
  cudaStream_t m2l_streams_[kM2LStreams] = {};
  cudaEvent_t ev_m2l_fork_ = nullptr, ev_m2m_done_ = nullptr, ev_m2l_join_[kM2LStreams] = {};
  std::vector<int> class_leaf_;  // leading leaf-level tiles of each class's range
  std::uint32_t launch_far_chain(cudaStream_t far, bool fork, bool with_periodic);
  std::uint32_t launch_fft(cudaStream_t s);  // the ANKH-FFT far field (fft_ plans)
  void launch_m2m(int first, int top, cudaStream_t st, unsigned p_begin = 0, unsigned p_count = 0);
  double* d_m2m_scratch_ = nullptr;  // runtime-order M2M past the shared-memory size
  double* d_per_scratch_ = nullptr;  // periodic term past the shared-memory size
  // CUDA-graph replay of launch_all for repeated inputs
  cudaGraphExec_t graph_exec_ = nullptr;
  const double *graph_pos_ = nullptr, *graph_src_ = nullptr;
  const double *graph_warm_pos_ = nullptr, *graph_warm_src_ = nullptr;
  // bound positions (set_positions): position flags + the moments-only graph
  DevResult* d_res_pos_ = nullptr;
  bool bound_ = false;
  cudaGraphExec_t graph_src_exec_ = nullptr;
  int graph_src_warm_ = 0;
  cudaStream_t last_stream_ = nullptr;
  std::vector<void*> allocs_;
  bool csr_only_ = false;
  int pending_code_ = 0;
  std::string pending_msg_;

  // partition
  int leaf_begin_ = 0, leaf_end_ = 0;
  bool include_self_ = true;
  // Shards (world | 8^E) split the moment pass (validation of q/mu/Theta and
  // the self-energy sum) by particle-index slice [src_i0_, src_i1_) -- whole
  // 256-particle blocks -- instead of every shard reading all N moments;
  // with NCCL attached the per-slice first violations are MIN-reduced (phase
  // API: each shard reports its slice, positions are checked by all)
  bool slice_src_ = false;
  // the record gather visits every leaf: it validates the moments, so
  // binning reads positions only
  bool gather_checks_src() const { return !slice_src_ && d_need_ == nullptr && !csr_only_; }
  double* d_self_leaf_ = nullptr;  // per Morton leaf: self-energy summand sums (P2M)
  std::size_t src_i0_ = 0, src_i1_ = 0;

  // inputs / sort
  double *d_pos_ = nullptr, *d_src_ = nullptr;
  unsigned *d_keys_ = nullptr, *d_keys2_ = nullptr, *d_idx_ = nullptr, *d_idx2_ = nullptr;
  unsigned *d_counts_ = nullptr, *d_off_ = nullptr;
  unsigned* d_leaf_mp_ = nullptr;
  unsigned* d_m2m_cnt_ = nullptr;  // arrival counters of the chained M2M  // per lex leaf: holds a dipole / quadrupole (P2P pair code)
  unsigned char* d_need_ = nullptr;  // shard: leaves whose records are gathered
  double* d_fin_scratch_ = nullptr;   // two-level final reduction
  void* d_temp_ = nullptr;  // radix sort of the validation path
  std::size_t temp_bytes_ = 0;
  ScanWork scan_{};  // the CSR offsets' single-pass scan
  double* d_part_ = nullptr;
  // expansions
  double* d_exp_ = nullptr;
  std::vector<long long> level_off_;
  long long* d_level_off_ = nullptr;
  double *d_hd_ = nullptr, *d_m2m_ = nullptr, *d_to_equi_ = nullptr, *d_spec_re_ = nullptr;
  // M2L
  double* d_factors_ = nullptr;
  M2LOp* d_ops_ = nullptr;
  M2LTile* d_tiles_ = nullptr;
  uint2* d_inst_ = nullptr;
  int* d_tile_ids_ = nullptr;
  std::vector<std::pair<int, int>> class_range_;  // per kp8: (begin, count) in d_tile_ids_
  int n_tiles_ = 0;
  std::map<std::pair<int, std::int64_t>, OpInfo> op_info_;
  std::size_t n_factors_ = 0;  // doubles in d_factors_ (m2l_factors reads them back)
  std::vector<M2LOp> h_ops_;
  // partials
  double *d_near_part_ = nullptr, *d_far_part_ = nullptr, *d_per_ = nullptr;
  unsigned long long* d_pair_count_ = nullptr;
  DevResult* d_res_ = nullptr;
  DevResult* h_res_ = nullptr;
  P2PRadial radial_{};  // near-field radial polynomials (fit_radial)
  int p2p_cap_ = 512;
  std::uint32_t launches_ = 0;
  // forces (allocated on the first forces() call)
  void force_setup();
  bool force_init_ = false;
  double *d_loc_ = nullptr, *d_fnear_ = nullptr, *d_ffar_ = nullptr, *d_fout_ = nullptr, *d_hd4_ = nullptr;
  double *d_dnear_ = nullptr, *d_dfar_ = nullptr, *d_dout_ = nullptr;  // moment derivatives (first use)
  double* d_gen_ = nullptr;  // periodic generator (build_periodic)
  int2* d_op_of_ = nullptr;
  int4* d_loc_tiles_ = nullptr;
  int n_loc_tiles_ = 0, force_cap_ = 960, force_half_cap_ = 576;
  bool force_half_ = true;      // forces alone: half shell + direction slots (ANKH_FORCE_FULL_STENCIL unsets)
  double* d_fslot_ = nullptr;   // 13 x n x 3 source-side sums of k_p2p_force_half
  // timing
  cudaEvent_t ev_[8] = {};
  bool evaluated_ = false;
};

}  // namespace ankh_b200
