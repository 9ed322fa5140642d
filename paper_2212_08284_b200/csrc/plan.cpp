// Host side of the B200 engine: geometry-only precompute and the launch
// sequence of one energy evaluation (fmm.cpp:383-436 re-planned for HBM).
#include <cstdio>
#include "plan.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <mutex>
#include <numeric>
#include <set>

#include "host_numerics.hpp"
#include "shard.hpp"

namespace ankh_b200 {

int default_depth(std::size_t n) {
  constexpr double target_per_leaf = 64.0;
  if (n <= target_per_leaf) return 1;
  const double levels = std::log(static_cast<double>(n) / target_per_leaf) / std::log(8.0);
  return std::max(1, static_cast<int>(std::ceil(levels - 1e-12)));
}

void validate_config(const ankh_config_v1& c) {
  auto bad = [](const char* m) { throw AnkhError(ANKH_INVALID_ARGUMENT, m); };
  if (!(c.xi > 0.0) || !std::isfinite(c.xi)) bad("xi must be positive");
  if (c.p < 0 || c.p == 1) bad("image half-width p must be 0 (open) or >= 2 (periodic)");
  if (c.order_cheb < 2) bad("order_cheb must be >= 2");
  if (c.order_equi < 2) bad("order_equi must be >= 2");
  if (c.depth < 0) bad("depth must be >= 1 (or 0 for automatic)");
  if (!(c.svd_tol > 0.0) || !(c.svd_tol < 1.0)) bad("svd_tol must lie in (0, 1)");
  if (c.recip_cutoff < 1) bad("recip_cutoff must be >= 1");
}

namespace {
constexpr double kInvSqrtPi = 0.5641895835477562869;
constexpr int kMaxOrderGpu = 64;     // L > kMaxOrderCompiled: runtime-order P2M / M2M (k_generic.cu)
constexpr int kMaxOrderCompiled = 10;

int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace

Plan::Plan(std::size_t n_, double box_radius, const ankh_config_v1& cfg_, bool csr_only, int engine)
    : n(n_), rb(box_radius), cfg(cfg_), csr_only_(csr_only), fft_(engine == 1) {
  const auto t0 = std::chrono::steady_clock::now();
  validate_config(cfg);
  if (!(rb > 0.0) || !std::isfinite(rb))
    throw AnkhError(ANKH_INVALID_ARGUMENT, "fmm_energy: invalid system: box_radius must be positive and finite");
  if (n >= (1ull << 31)) throw AnkhError(ANKH_RUNTIME_ERROR, "fmm_energy: more than 2^31-1 particles");
  if (cfg.world < 1) cfg.world = 1;
  if (fft_ && cfg.world > 1) throw AnkhError(ANKH_RUNTIME_ERROR, "fft engine: sharded plans (world > 1) are not supported");
  if (cfg.rank < 0 || cfg.rank >= cfg.world) throw AnkhError(ANKH_INVALID_ARGUMENT, "rank out of range");
  if (cfg.device >= 0) {
    int count = 0;
    ANKH_CUDA(cudaGetDeviceCount(&count));
    if (cfg.device >= count) throw AnkhError(ANKH_INVALID_ARGUMENT, "device index out of range");
    device_ = cfg.device;
  } else {
    ANKH_CUDA(cudaGetDevice(&device_));
  }
  // the plan's resources live on device_; the caller's current device is
  // restored when the constructor returns
  DeviceGuard on_device(device_);
  periodic = cfg.p >= 2;
  depth = cfg.depth > 0 ? cfg.depth : default_depth(n);
  L = cfg.order_cheb;
  // Errors the reference raises only after validate_system (octree.cpp:28,
  // chebyshev.cpp:86) are deferred so a system violation still wins.
  if (depth < 1 || depth > 8) {
    pending_code_ = ANKH_INVALID_ARGUMENT;
    pending_msg_ = "build_tree: depth must be in [1, 8]";
  } else if (L > 64) {
    pending_code_ = ANKH_INVALID_ARGUMENT;
    pending_msg_ = "DiffOperator: order out of range";
  } else if (L > kMaxOrderGpu) {
    pending_code_ = ANKH_RUNTIME_ERROR;
    pending_msg_ = "order_cheb > 64 is not supported by the B200 engine";
  }
  // the FFT engine's own limits, checked before any resource is created
  if (fft_ && pending_code_ == 0 && n > 0 && !csr_only) {
    if (cfg.order_equi < 2 || cfg.order_equi > 16)
      throw AnkhError(ANKH_INVALID_ARGUMENT, "fft engine: order_equi must be in [2, 16]");
    if (depth > 6) throw AnkhError(ANKH_RUNTIME_ERROR, "fft engine: depth > 6 is not supported");
    if (L > kMaxOrderCompiled) throw AnkhError(ANKH_RUNTIME_ERROR, "fft engine: order_cheb > 10 is not supported");
  }
  try {
    build_all(t0);
  } catch (...) {
    release();  // the destructor does not run for a constructor that throws
    throw;
  }
}

void Plan::build_all(std::chrono::steady_clock::time_point t0) {
  ANKH_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  // The far chain (P2M -> exchange -> M2M -> M2L) and the streamed path's
  // record gathers run at the highest stream priority: the block scheduler
  // hands them SMs first and P2P (caller's stream, default priority) fills
  // the rest, so the dependency chain never waits behind P2P's CTA backlog.
  int prio_least = 0, prio_greatest = 0;
  ANKH_CUDA(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
  hi_prio_ = std::getenv("ANKH_NO_PRIORITY") ? 0 : prio_greatest;
  {
    // leaf-level M2L beside M2M: measured slower (config 3: 5.272 vs 5.261 ms,
    // world-8 shard 0.889 vs 0.861 ms -- twice the class launches and tails)
    const char* e = std::getenv("ANKH_M2L_SPLIT");
    m2l_split_ = e && e[0] == '1';
  }
  ANKH_CUDA(cudaStreamCreateWithPriority(&side_stream_, cudaStreamNonBlocking, hi_prio_));
  ANKH_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  ANKH_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  ANKH_CUDA(cudaEventCreateWithFlags(&ev_m2l_fork_, cudaEventDisableTiming));
  ANKH_CUDA(cudaEventCreateWithFlags(&ev_m2m_done_, cudaEventDisableTiming));
  for (int k = 0; k < kM2LStreams; ++k) {
    ANKH_CUDA(cudaStreamCreateWithPriority(&m2l_streams_[k], cudaStreamNonBlocking, hi_prio_));
    ANKH_CUDA(cudaEventCreateWithFlags(&ev_m2l_join_[k], cudaEventDisableTiming));
  }
  for (auto& e : ev_) ANKH_CUDA(cudaEventCreate(&e));
  if (pending_code_ != 0) {
    depth = 1;  // validation-only plan
    L = 2;
  }
  K = L * L * L;
  Kp = exp_stride(K);  // expansion row stride == factor column stride
  nax = 1 << depth;
  n_leaves = 1 << (3 * depth);
  // ANKH_PLAN_TIMING=1: per-stage plan build times on stderr (diagnostics)
  const bool verbose = std::getenv("ANKH_PLAN_TIMING") != nullptr;
  auto stamp = [&](const char* what, std::chrono::steady_clock::time_point& t) {
    if (!verbose) return;
    ANKH_CUDA(cudaStreamSynchronize(stream_));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ankh plan] %-10s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  };
  auto ts = std::chrono::steady_clock::now();
  stamp("setup", ts);
  build_geometry();
  stamp("geometry", ts);
  allocate();
  stamp("allocate", ts);
  if (pending_code_ == 0 && n > 0 && !csr_only_) {
    build_halo();
    if (fft_)
      build_fft();
    else
      build_m2l();
    stamp("m2l", ts);
    if (periodic) build_periodic();
    stamp("periodic", ts);
  }
  ANKH_CUDA(cudaStreamSynchronize(stream_));
  precompute_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

Plan::~Plan() { release(); }

// Every resource the plan holds (also on a constructor that throws part way:
// members not created yet are null)
void Plan::release() noexcept {
  DeviceGuard on_device(device_, /*nothrow=*/true);
  for (cudaStream_t s : {stream_, last_stream_, side_stream_, copy_stream_, gather_stream_})
    if (s) cudaStreamSynchronize(s);
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (graph_src_exec_) cudaGraphExecDestroy(graph_src_exec_);
  if (sgraph_exec_) cudaGraphExecDestroy(sgraph_exec_);
  for (void* p : allocs_) cudaFreeAsync(p, stream_);  // back to the pool (kept for the next plan)
  if (stream_) cudaStreamSynchronize(stream_);
  if (h_res_) cudaFreeHost(h_res_);
  if (h_sbounds_) cudaFreeHost(h_sbounds_);
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  if (ev_m2l_fork_) cudaEventDestroy(ev_m2l_fork_);
  if (ev_m2m_done_) cudaEventDestroy(ev_m2m_done_);
  for (int k = 0; k < kM2LStreams; ++k) {
    if (m2l_streams_[k]) {
      cudaStreamSynchronize(m2l_streams_[k]);
      cudaStreamDestroy(m2l_streams_[k]);
    }
    if (ev_m2l_join_[k]) cudaEventDestroy(ev_m2l_join_[k]);
  }
  for (cudaStream_t s : {copy_stream_, gather_stream_})
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  for (cudaEvent_t e : {ev_s_start_, ev_s_binned_, ev_s_lists_, ev_s_sorted_, ev_s_inv_, ev_s_p2p2_})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_t_)
    if (e) cudaEventDestroy(e);
  for (int c = 0; c < kMaxStreamChunks; ++c) {
    if (ev_s_chunk_[c]) cudaEventDestroy(ev_s_chunk_[c]);
    if (ev_s_gath_[c]) cudaEventDestroy(ev_s_gath_[c]);
    if (ev_s_posc_[c]) cudaEventDestroy(ev_s_posc_[c]);
  }
  if (p2p_stream2_) {
    cudaStreamSynchronize(p2p_stream2_);
    cudaStreamDestroy(p2p_stream2_);
  }
  if (side_stream_) {
    cudaStreamSynchronize(side_stream_);
    cudaStreamDestroy(side_stream_);
  }
  if (stream_) cudaStreamDestroy(stream_);
  stream_ = nullptr;
}

// Plan buffers come from the device's stream-ordered pool, kept by the pool
// when a plan is destroyed (release threshold raised once per device): the
// next plan -- e.g. a one-shot call for another system size -- reuses that
// memory instead of mapping gigabytes anew (cudaMalloc / cudaFree of the
// plan's buffers took 0.03-0.9 s per build / close, erratically).
void* Plan::dalloc(std::size_t bytes) {
  static std::mutex mu;
  static std::vector<int> pooled;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(pooled.begin(), pooled.end(), device_) == pooled.end()) {
      cudaMemPool_t pool = nullptr;
      if (cudaDeviceGetDefaultMemPool(&pool, device_) == cudaSuccess) {
        unsigned long long keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      pooled.push_back(device_);
    }
  }
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
#ifdef ANKH_CHECKED
  // guard zone after every plan buffer, verified after each evaluation
  ANKH_CUDA(cudaMallocAsync(&p, bytes + kGuardBytes, stream_));
  ANKH_CUDA(cudaMemsetAsync(static_cast<char*>(p) + bytes, kGuardByte, kGuardBytes, stream_));
  guards_.emplace_back(p, bytes);
#else
  ANKH_CUDA(cudaMallocAsync(&p, bytes, stream_));
#endif
  allocs_.push_back(p);
  device_bytes += bytes;
  return p;
}

void Plan::check_guards() {
#ifdef ANKH_CHECKED
  std::vector<unsigned char> g(kGuardBytes);
  for (std::size_t k = 0; k < guards_.size(); ++k) {
    ANKH_CUDA(cudaMemcpy(g.data(), static_cast<char*>(guards_[k].first) + guards_[k].second, kGuardBytes,
                         cudaMemcpyDeviceToHost));
    for (unsigned char b : g)
      if (b != kGuardByte)
        throw AnkhError(ANKH_CUDA_ERROR, "checked build: guard zone after plan buffer #" + std::to_string(k) +
                                             " (" + std::to_string(guards_[k].second) + " bytes) was overwritten");
  }
#endif
}

void Plan::build_geometry() {
  // leaf ownership: contiguous Morton ranges
  std::int64_t lb = 0, le = 0;
  shard_leaf_range(depth, cfg.rank, cfg.world, &lb, &le);
  leaf_begin_ = static_cast<int>(lb);
  leaf_end_ = static_cast<int>(le);
  include_self_ = cfg.rank == 0;
  // P2M is split across shards when the Morton leaf slices are equal-sized
  // (world | 8^E) so one in-place all-gather completes the leaf level;
  // otherwise every shard computes all leaf expansions.
  shard_upward_ = cfg.world > 1 && (static_cast<long long>(n_leaves) % cfg.world) == 0;
  p2m_begin_ = shard_upward_ ? lb : 0;
  p2m_end_ = shard_upward_ ? le : n_leaves;
  exch_level_ = shard_upward_ ? shard_exchange_level(depth, cfg.world) : depth;
  slice_src_ = shard_upward_ && std::getenv("ANKH_SHARD_FULL_SRC") == nullptr;
  if (slice_src_) shard_src_slice(n, cfg.rank, cfg.world, &src_i0_, &src_i1_);
  // P2P polynomial length from the largest possible near distance
  // (2 leaf sides per axis): s_max = xi^2 (2 sqrt(3) * 2 r_B / n)^2
  const double side = 2.0 * rb / nax;
  const double dmax = 2.0 * std::sqrt(3.0) * side * 1.0001;
  {
    const RadialFit f = fit_radial(cfg.xi * cfg.xi * dmax * dmax);
    radial_.nterms = f.nterms;
    radial_.s_lim = f.s_lim;
    std::copy(f.p, f.p + 14, radial_.p);
    std::copy(f.g, f.g + 14, radial_.g);
  }
  // P2P CTA: 256 threads (3 CTAs/SM, 24 warps), staged-source capacity sized
  // so a leaf's own + 13 neighbour leaves (~14 x mean occupancy) fit in one
  // pass for almost every leaf.  ANKH_P2P_CAP overrides (tuning).
  const double per_leaf = static_cast<double>(n) / n_leaves;
  p2p_cap_ = static_cast<int>(std::ceil(14.0 * per_leaf * 1.3 / 32.0)) * 32;
  p2p_cap_ = std::max(256, std::min(p2p_cap_, 960));
  if (const char* e = std::getenv("ANKH_P2P_CAP")) {
    p2p_cap_ = std::max(64, std::atoi(e));
  }
}

void Plan::allocate() {
  const std::size_t nn = std::max<std::size_t>(n, 1);
  d_pos_ = static_cast<double*>(dalloc(nn * 3 * sizeof(double)));
  d_src_ = static_cast<double*>(dalloc(nn * 10 * sizeof(double)));
  d_keys_ = static_cast<unsigned*>(dalloc(nn * sizeof(unsigned)));
  d_keys2_ = static_cast<unsigned*>(dalloc(nn * sizeof(unsigned)));
  d_idx_ = static_cast<unsigned*>(dalloc(nn * sizeof(unsigned)));
  d_idx2_ = static_cast<unsigned*>(dalloc(nn * sizeof(unsigned)));
  // leaf histogram, then (streamed path) each leaf's largest particle index
  d_counts_ = static_cast<unsigned*>(dalloc(2 * (n_leaves + 1) * sizeof(unsigned)));
  d_leafmax_ = d_counts_ + (n_leaves + 1);
  {
    const std::size_t tiles = scan_tiles(static_cast<std::size_t>(n_leaves) + 1);
    scan_.status = static_cast<unsigned long long*>(dalloc(tiles * sizeof(unsigned long long) + 16));
    scan_.ctr = reinterpret_cast<unsigned*>(scan_.status + tiles);
    ANKH_CUDA(cudaMemsetAsync(scan_.status, 0, tiles * sizeof(unsigned long long) + 16, stream_));
  }
  d_off_ = static_cast<unsigned*>(dalloc((n_leaves + 1) * sizeof(unsigned)));
  d_leaf_mp_ = static_cast<unsigned*>(dalloc(static_cast<std::size_t>(n_leaves) * sizeof(unsigned)));
  ANKH_CUDA(cudaMemsetAsync(d_leaf_mp_, 0, static_cast<std::size_t>(n_leaves) * sizeof(unsigned), stream_));
  d_fin_scratch_ = static_cast<double*>(dalloc(finalize_scratch_bytes()));
  ANKH_CUDA(cudaMemsetAsync(d_fin_scratch_, 0, finalize_scratch_bytes(), stream_));  // completion counter
  // A shard gathers particle records only for the leaves it reads: its P2P
  // targets, their 13 half-shell neighbours (k_p2p's stencil, periodic wrap)
  // and its P2M rows.  (One shard: every leaf, no mask.)
  if (cfg.world > 1 && !csr_only_) {
    std::vector<unsigned char> need(n_leaves, 0);
    auto lex_of = [&](unsigned m) {
      return (morton_compact3(m >> 2) * nax + morton_compact3(m >> 1)) * nax + morton_compact3(m);
    };
    for (int m = p2m_begin_; m < p2m_end_; ++m) need[lex_of(static_cast<unsigned>(m))] = 1;
    for (int m = leaf_begin_; m < leaf_end_; ++m) {
      const unsigned lf = lex_of(static_cast<unsigned>(m));
      const int a[3] = {static_cast<int>(lf) / (nax * nax), (static_cast<int>(lf) / nax) % nax,
                        static_cast<int>(lf) % nax};
      need[lf] = 1;
      for (int d = 0; d < 13; ++d) {  // the 13 lex-positive directions of k_p2p
        const int dx = d < 4 ? 0 : 1;
        const int dy = d == 0 ? 0 : (d < 4 ? 1 : (d - 4) / 3 - 1);
        const int dz = d == 0 ? 1 : (d < 4 ? d - 2 : (d - 4) % 3 - 1);
        int b[3] = {a[0] + dx, a[1] + dy, a[2] + dz};
        bool ok = true;
        for (int q = 0; q < 3; ++q) {
          if (b[q] < 0 || b[q] >= nax) {
            if (!periodic) ok = false;
            b[q] = (b[q] + nax) % nax;
          }
        }
        if (ok) need[(static_cast<unsigned>(b[0]) * nax + b[1]) * nax + b[2]] = 1;
      }
    }
    d_need_ = static_cast<unsigned char*>(dalloc(need.size()));
    ANKH_CUDA(cudaMemcpyAsync(d_need_, need.data(), need.size(), cudaMemcpyHostToDevice, stream_));
    ANKH_CUDA(cudaStreamSynchronize(stream_));
  }
  temp_bytes_ = sort_temp_bytes(nn);
  d_temp_ = dalloc(temp_bytes_);
  d_part_ = static_cast<double*>(dalloc(nn * kRec * sizeof(double)));
  level_off_.assign(depth + 2, 0);
  // expansion rows padded to Kp = exp_stride(K) doubles; the zero tail is
  // written once here and never touched by the kernels
  for (int l = 0; l <= depth; ++l) level_off_[l + 1] = level_off_[l] + (1ll << (3 * l)) * Kp;
  d_exp_ = static_cast<double*>(dalloc(level_off_[depth + 1] * sizeof(double)));
  ANKH_CUDA(cudaMemsetAsync(d_exp_, 0, level_off_[depth + 1] * sizeof(double), stream_));
  d_m2m_cnt_ = static_cast<unsigned*>(dalloc(std::max<std::size_t>(m2m_counter_count(depth), 1) * sizeof(unsigned)));
  ANKH_CUDA(cudaMemsetAsync(d_m2m_cnt_, 0, std::max<std::size_t>(m2m_counter_count(depth), 1) * sizeof(unsigned),
                            stream_));
  d_level_off_ = static_cast<long long*>(dalloc(level_off_.size() * sizeof(long long)));
  ANKH_CUDA(cudaMemcpyAsync(d_level_off_, level_off_.data(), level_off_.size() * sizeof(long long),
                            cudaMemcpyHostToDevice, stream_));
  d_self_leaf_ = static_cast<double*>(dalloc(static_cast<std::size_t>(n_leaves) * sizeof(double)));
  d_near_part_ = static_cast<double*>(dalloc(std::max(leaf_end_ - leaf_begin_, 1) * sizeof(double)));
  d_pair_count_ = static_cast<unsigned long long*>(
      dalloc(std::max(leaf_end_ - leaf_begin_, 1) * sizeof(unsigned long long)));
  d_per_ = static_cast<double*>(dalloc(sizeof(double)));
  if (const std::size_t ps = periodic_eval_scratch_doubles(L)) d_per_scratch_ = static_cast<double*>(dalloc(ps * sizeof(double)));
  if (L > kMaxOrderCompiled)
    if (const std::size_t ms = m2m_generic_scratch_doubles(L)) d_m2m_scratch_ = static_cast<double*>(dalloc(ms * sizeof(double)));
  d_res_ = static_cast<DevResult*>(dalloc(sizeof(DevResult)));
  d_res_pos_ = static_cast<DevResult*>(dalloc(sizeof(DevResult)));
  ANKH_CUDA(cudaMallocHost(&h_res_, sizeof(DevResult)));
  // small operators (chebyshev.cpp:85-108, fmm.cpp:213-219, 421-424)
  const auto hd = diff_operator(L);
  std::vector<double> hd_all;
  for (const auto& m : hd) hd_all.insert(hd_all.end(), m.begin(), m.end());
  const std::vector<double> nodes = cheb_nodes(L);
  std::vector<double> lo(L), hi(L);
  for (int i = 0; i < L; ++i) {
    lo[i] = 0.5 * (nodes[i] - 1.0);
    hi[i] = 0.5 * (nodes[i] + 1.0);
  }
  std::vector<double> m2m = transfer_cheb(L, lo);
  const std::vector<double> m2m_hi = transfer_cheb(L, hi);
  m2m.insert(m2m.end(), m2m_hi.begin(), m2m_hi.end());
  const std::vector<double> to_equi = transfer_equi(L, nodes);
  d_hd_ = static_cast<double*>(dalloc(hd_all.size() * sizeof(double)));
  d_m2m_ = static_cast<double*>(dalloc(m2m.size() * sizeof(double)));
  d_to_equi_ = static_cast<double*>(dalloc(to_equi.size() * sizeof(double)));
  ANKH_CUDA(cudaMemcpyAsync(d_hd_, hd_all.data(), hd_all.size() * sizeof(double),
                            cudaMemcpyHostToDevice, stream_));
  upload_p2m_basis(L, hd_all.data(), stream_);  // constant-bank copy for the warp P2M
  ANKH_CUDA(cudaGetLastError());
  ANKH_CUDA(cudaMemcpyAsync(d_m2m_, m2m.data(), m2m.size() * sizeof(double),
                            cudaMemcpyHostToDevice, stream_));
  ANKH_CUDA(cudaMemcpyAsync(d_to_equi_, to_equi.data(), to_equi.size() * sizeof(double),
                            cudaMemcpyHostToDevice, stream_));
  ANKH_CUDA(cudaStreamSynchronize(stream_));
}

// build_m2l_cache (fmm.cpp:141-179) + the canonical instance lists of
// far_field_energy (fmm.cpp:244-253), grouped by (level, offset).
void Plan::build_m2l() {
  struct OffsetWork {
    int level;
    std::array<int, 3> o;
    std::vector<uint2> inst;  // host enumeration only
    std::size_t count = 0;    // instances of this operator
    Factors f;
  };
  const int threads = cfg.threads;
  const bool verbose = std::getenv("ANKH_PLAN_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto stamp = [&](const char* what) {
    if (!verbose) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ankh plan]   m2l %-9s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  // canonical instances owned by this shard (shard.cpp, fmm.cpp:244-253):
  // generated on the device straight into d_inst_ (k_inst.cu; same operator
  // order and per-operator target-Morton order as the host enumeration,
  // which ANKH_HOST_INST=1 selects)
  const bool gpu_inst = std::getenv("ANKH_HOST_INST") == nullptr;
  std::vector<OffsetWork> work;
  std::vector<OffsetInstances> groups;
  DeviceScratch inst_tmp(stream_);
  if (gpu_inst) {
    std::vector<int4> offs;
    for (int ox = -3; ox <= 3; ++ox)
      for (int oy = -3; oy <= 3; ++oy)
        for (int oz = -3; oz <= 3; ++oz)
          if (std::max({std::abs(ox), std::abs(oy), std::abs(oz)}) >= 2) offs.push_back(make_int4(ox, oy, oz, 0));
    const int n_offs = static_cast<int>(offs.size());
    const std::size_t nb = m2l_instance_blocks(depth, n_offs);
    int4* d_offs = inst_tmp.alloc<int4>(offs.size());
    unsigned* d_counts = inst_tmp.alloc<unsigned>(nb + 1);
    unsigned* d_offsets = inst_tmp.alloc<unsigned>(nb + 1);
    const std::size_t tb = m2l_instances_temp_bytes(nb);
    void* d_temp = inst_tmp.alloc<unsigned char>(tb);
    ANKH_CUDA(cudaMemcpyAsync(d_offs, offs.data(), offs.size() * sizeof(int4), cudaMemcpyHostToDevice, stream_));
    ANKH_CUDA(cudaMemsetAsync(d_counts, 0, (nb + 1) * sizeof(unsigned), stream_));
    const int shard = cfg.world > 1 ? cfg.rank : -1;
    m2l_instances_device(depth, periodic, shard, cfg.world, d_offs, n_offs, d_counts, d_offsets, nb, d_temp,
                         tb, nullptr, stream_);
    ANKH_CUDA(cudaGetLastError());
    std::vector<unsigned> off(nb + 1);
    ANKH_CUDA(cudaMemcpyAsync(off.data(), d_offsets, off.size() * sizeof(unsigned), cudaMemcpyDeviceToHost,
                              stream_));
    ANKH_CUDA(cudaStreamSynchronize(stream_));
    const std::size_t total = off[nb];
    d_inst_ = static_cast<uint2*>(dalloc(std::max<std::size_t>(total, 1) * sizeof(uint2)));
    m2l_instances_device(depth, periodic, shard, cfg.world, d_offs, n_offs, d_counts, d_offsets, nb, d_temp,
                         tb, d_inst_, stream_);
    ANKH_CUDA(cudaGetLastError());
    const int bs = m2l_instance_block_size();
    std::size_t blk = 0;
    for (int level = 1; level <= depth; ++level) {
      const std::size_t per_op = ((std::size_t(1) << (3 * level)) + bs - 1) / bs;
      for (int j = 0; j < n_offs; ++j, blk += per_op) {
        const std::size_t c = off[blk + per_op] - off[blk];
        if (c == 0) continue;
        OffsetWork w;
        w.level = level;
        w.o = {offs[j].x, offs[j].y, offs[j].z};
        w.count = c;
        work.push_back(std::move(w));
      }
    }
  } else {
    groups = enumerate_m2l(depth, periodic, cfg.world > 1 ? cfg.rank : -1, cfg.world, threads);
    work.resize(groups.size());
  }
  parallel_for(static_cast<int>(groups.size()), threads, [&](int i) {
    work[i].level = groups[i].level;
    work[i].o = groups[i].offset;
    work[i].inst.resize(groups[i].t.size());
    // expansions are stored in Morton order: instance cells become Morton rows,
    // and a tile's 64 instances are Morton-contiguous targets (L2 locality)
    const unsigned nl = 1u << groups[i].level;
    auto to_morton = [nl](unsigned c) { return morton3(c / (nl * nl), (c / nl) % nl, c % nl); };
    for (std::size_t k = 0; k < groups[i].t.size(); ++k)
      work[i].inst[k] = make_uint2(to_morton(groups[i].t[k]), to_morton(groups[i].s[k]));
    std::sort(work[i].inst.begin(), work[i].inst.end(),
              [](const uint2& a, const uint2& b) { return a.x < b.x; });
    work[i].count = work[i].inst.size();
    groups[i] = OffsetInstances{};  // release as we go
  });
  groups.clear();
  stamp("instances");
  // factors: exact SVD path uses the signed-permutation symmetry of the block
  // (one SVD per class, SURVEY.md Decision 3); K > 150 replicates the
  // reference's seeded randomized path per offset.
  // GPU path (default for the exact SVD): dense class blocks on the host (the
  // reference's erfc formula), batched Jacobi SVD + factor rows on the device
  // (k_svd.cu); only the sigmas come back for the rank rule.
  std::vector<int> work_cls;
  DeviceScratch svd_tmp(stream_);
  double *d_lf = nullptr, *d_rf = nullptr;
  const bool gpu_fac = K <= 150 && std::getenv("ANKH_HOST_SVD") == nullptr;
  if (gpu_fac) {
    std::map<std::pair<int, std::array<int, 3>>, int> cls_of;
    for (const auto& w : work) cls_of[{w.level, symmetry_of(w.o).rep}] = 0;
    std::vector<std::pair<int, std::array<int, 3>>> keys;
    for (auto& kv : cls_of) {
      kv.second = static_cast<int>(keys.size());
      keys.push_back(kv.first);
    }
    const int nc = static_cast<int>(keys.size());
    const std::size_t kk = static_cast<std::size_t>(K) * K;
    std::vector<double> hc(nc * kk);
    parallel_for(nc, threads, [&](int i) {
      const std::vector<double> c = m2l_dense(L, rb / (1 << keys[i].first), keys[i].second, cfg.xi);
      std::copy(c.begin(), c.end(), hc.begin() + i * kk);
    });
    stamp("dense");
    double* d_c = svd_tmp.alloc<double>(nc * kk);
    double* d_w = svd_tmp.alloc<double>(nc * kk);
    double* d_sig = svd_tmp.alloc<double>(static_cast<std::size_t>(nc) * K);
    d_lf = svd_tmp.alloc<double>(nc * kk);
    d_rf = svd_tmp.alloc<double>(nc * kk);
    int* d_order = svd_tmp.alloc<int>(static_cast<std::size_t>(nc) * K);
    int* d_rank = svd_tmp.alloc<int>(nc);
    ANKH_CUDA(cudaMemcpyAsync(d_c, hc.data(), hc.size() * sizeof(double), cudaMemcpyHostToDevice, stream_));
    int* d_sweeps = verbose ? svd_tmp.alloc<int>(nc) : nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (verbose) {
      ANKH_CUDA(cudaEventCreate(&e0));
      ANKH_CUDA(cudaEventCreate(&e1));
      ANKH_CUDA(cudaEventRecord(e0, stream_));
    }
    launch_jacobi_svd(d_c, nc, K, cfg.svd_tol * 1e-6, d_w, d_sig, d_sweeps, stream_);
    ANKH_CUDA(cudaGetLastError());
    if (verbose) {
      ANKH_CUDA(cudaEventRecord(e1, stream_));
      ANKH_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      ANKH_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      std::vector<int> sw(nc);
      ANKH_CUDA(cudaMemcpy(sw.data(), d_sweeps, nc * sizeof(int), cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "[ankh plan]   m2l jacobi kernel %.3f ms, %d classes, sweeps max %d\n", ms, nc,
                   nc ? *std::max_element(sw.begin(), sw.end()) : 0);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    std::vector<double> sig(static_cast<std::size_t>(nc) * K);
    ANKH_CUDA(cudaMemcpyAsync(sig.data(), d_sig, sig.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    ANKH_CUDA(cudaStreamSynchronize(stream_));
    // finish() (host_numerics.cpp): stable descending order, rank rule
    std::vector<int> order(static_cast<std::size_t>(nc) * K), rank(nc);
    for (int i = 0; i < nc; ++i) {
      int* o = order.data() + static_cast<std::size_t>(i) * K;
      const double* sv = sig.data() + static_cast<std::size_t>(i) * K;
      std::iota(o, o + K, 0);
      std::stable_sort(o, o + K, [&](int x, int y) { return sv[x] > sv[y]; });
      int r = 1;
      while (r < K && sv[o[r]] > sv[o[0]] * cfg.svd_tol) ++r;
      rank[i] = r;
    }
    ANKH_CUDA(cudaMemcpyAsync(d_order, order.data(), order.size() * sizeof(int), cudaMemcpyHostToDevice, stream_));
    ANKH_CUDA(cudaMemcpyAsync(d_rank, rank.data(), rank.size() * sizeof(int), cudaMemcpyHostToDevice, stream_));
    launch_svd_factors(d_c, d_w, d_sig, d_order, d_rank, nc, K, d_lf, d_rf, stream_);
    ANKH_CUDA(cudaGetLastError());
    work_cls.resize(work.size());
    for (std::size_t wi = 0; wi < work.size(); ++wi) {
      const int c = cls_of.at({work[wi].level, symmetry_of(work[wi].o).rep});
      work_cls[wi] = c;
      work[wi].f.rank = rank[c];
      work[wi].f.k_full = K;
    }
    ANKH_CUDA(cudaStreamSynchronize(stream_));  // the host vectors above go out of scope
  } else if (K <= 150) {
    std::map<std::pair<int, std::array<int, 3>>, Factors> reps;
    for (const auto& w : work) reps[{w.level, symmetry_of(w.o).rep}] = Factors{};
    std::vector<std::pair<int, std::array<int, 3>>> keys;
    for (const auto& kv : reps) keys.push_back(kv.first);
    std::vector<Factors> fac(keys.size());
    parallel_for(static_cast<int>(keys.size()), threads, [&](int i) {
      const int level = keys[i].first;
      const double rad = rb / (1 << level);
      fac[i] = compress_m2l(m2l_dense(L, rad, keys[i].second, cfg.xi), K, cfg.svd_tol, 0);
    });
    for (std::size_t i = 0; i < keys.size(); ++i) reps[keys[i]] = std::move(fac[i]);
    parallel_for(static_cast<int>(work.size()), threads, [&](int wi) {
      OffsetWork& w = work[wi];
      const Symmetry sym = symmetry_of(w.o);
      const Factors& r = reps.at({w.level, sym.rep});
      const std::vector<int> perm = node_permutation(sym, L);
      w.f.rank = r.rank;
      w.f.k_full = K;
      w.f.lmat.assign(r.lmat.size(), 0.0);
      w.f.rmat.assign(r.rmat.size(), 0.0);
      for (int row = 0; row < r.rank; ++row)
        for (int k = 0; k < K; ++k) {
          w.f.lmat[static_cast<std::size_t>(row) * K + perm[k]] = r.lmat[static_cast<std::size_t>(row) * K + k];
          w.f.rmat[static_cast<std::size_t>(row) * K + perm[k]] = r.rmat[static_cast<std::size_t>(row) * K + k];
        }
    });
  } else {
    parallel_for(static_cast<int>(work.size()), threads, [&](int wi) {
      OffsetWork& w = work[wi];
      const double rad = rb / (1 << w.level);
      const std::int64_t key = offset_key(w.o);
      w.f = compress_m2l(m2l_dense(L, rad, w.o, cfg.xi), K, cfg.svd_tol, m2l_seed(w.level, key));
    });
  }
  stamp("factors");
  // device operators: row blocks of <= 128 ranks, L then R, zero padded.
  // Layout pass (serial, per operator) then a parallel fill.
  std::vector<M2LTile> tiles;
  h_ops_.clear();
  double rank_sum = 0.0;
  far_flops = 0.0;
  m2l_instances = 0;
  struct Block {
    int work, r0, rows;
  };
  std::vector<Block> blocks;
  std::vector<std::size_t> inst_begin(work.size());
  std::size_t n_inst = 0, n_fac = 0;
  for (std::size_t wi = 0; wi < work.size(); ++wi) {
    const OffsetWork& w = work[wi];
    const int rank = w.f.rank;
    OpInfo info{w.level, offset_key(w.o), rank, static_cast<int>(h_ops_.size()), 0};
    inst_begin[wi] = n_inst;
    for (int r0 = 0; r0 < rank; r0 += 8 * kMaxKp8) {
      const int rows = std::min(8 * kMaxKp8, rank - r0);
      const int kp = ceil_div(rows, 8) * 8;
      M2LOp op;
      op.factor_off = static_cast<long long>(n_fac);
      op.kp = kp;
      op.rank = rows;
      n_fac += 2 * static_cast<std::size_t>(kp) * Kp;
      const int op_index = static_cast<int>(h_ops_.size());
      h_ops_.push_back(op);
      blocks.push_back({static_cast<int>(wi), r0, rows});
      ++info.n_blocks;
      for (int b = 0; b < static_cast<int>(w.count); b += kM2LTile)
        tiles.push_back({op_index, w.level, static_cast<int>(n_inst) + b,
                         std::min(kM2LTile, static_cast<int>(w.count) - b)});
    }
    op_info_[{w.level, info.key}] = info;
    rank_sum += rank;
    n_inst += w.count;
    far_flops += static_cast<double>(w.count) * (4.0 * rank * K + 2.0 * rank);
  }
  m2l_instances = n_inst;
  std::vector<uint2> inst(gpu_inst ? 0 : n_inst);  // host enumeration: gathered for the upload
  if (!gpu_inst)
    parallel_for(static_cast<int>(work.size()), threads, [&](int wi) {
      std::copy(work[wi].inst.begin(), work[wi].inst.end(), inst.begin() + inst_begin[wi]);
    });
  std::vector<double> h_factors;  // host-built operator blocks (host SVD paths)
  std::vector<M2LPack> packs;     // GPU path: block descriptors for k_m2l_pack
  std::vector<int> perms;
  int max_rows = 0;
  if (gpu_fac) {
    std::map<std::array<int, 3>, int> perm_off;  // one permutation per distinct offset
    std::vector<int> work_perm(work.size());
    for (std::size_t wi = 0; wi < work.size(); ++wi) {
      auto it = perm_off.find(work[wi].o);
      if (it == perm_off.end()) {
        it = perm_off.emplace(work[wi].o, static_cast<int>(perms.size())).first;
        const std::vector<int> p = node_permutation(symmetry_of(work[wi].o), L);
        perms.insert(perms.end(), p.begin(), p.end());
      }
      work_perm[wi] = it->second;
    }
    packs.resize(blocks.size());
    for (std::size_t bi = 0; bi < blocks.size(); ++bi) {
      const Block& b = blocks[bi];
      packs[bi] = {h_ops_[bi].factor_off, work_cls[b.work], b.r0, b.rows, h_ops_[bi].kp,
                   work_perm[b.work]};
      max_rows = std::max(max_rows, b.rows);
    }
  } else {
    h_factors.assign(n_fac, 0.0);
    parallel_for(static_cast<int>(blocks.size()), threads, [&](int bi) {
      const Block& b = blocks[bi];
      const Factors& f = work[b.work].f;
      double* dl = h_factors.data() + h_ops_[bi].factor_off;
      double* dr = dl + static_cast<std::size_t>(h_ops_[bi].kp) * Kp;
      for (int r = 0; r < b.rows; ++r)
        for (int k = 0; k < K; ++k) {
          dl[static_cast<std::size_t>(r) * Kp + k] = f.lmat[static_cast<std::size_t>(b.r0 + r) * K + k];
          dr[static_cast<std::size_t>(r) * Kp + k] = f.rmat[static_cast<std::size_t>(b.r0 + r) * K + k];
        }
    });
  }
  m2l_operators = work.size();
  m2l_rank_mean = work.empty() ? 0.0 : rank_sum / work.size();
  n_tiles_ = static_cast<int>(tiles.size());
  std::vector<int> owned(tiles.size());
  std::iota(owned.begin(), owned.end(), 0);
  // group owned tiles by kp class
  class_range_.assign(kMaxKp8 + 1, {0, 0});
  std::vector<int> ids;
  class_leaf_.assign(kMaxKp8 + 1, 0);
  for (int c = 1; c <= kMaxKp8; ++c) {
    // leaf-level tiles first: they need no M2M and can run beside it
    const int begin = static_cast<int>(ids.size());
    for (int t : owned)
      if (h_ops_[tiles[t].op].kp / 8 == c && tiles[t].level == depth) ids.push_back(t);
    class_leaf_[c] = static_cast<int>(ids.size()) - begin;
    for (int t : owned)
      if (h_ops_[tiles[t].op].kp / 8 == c && tiles[t].level != depth) ids.push_back(t);
    class_range_[c] = {begin, static_cast<int>(ids.size()) - begin};
  }
  stamp("pack");
  n_factors_ = n_fac;
  d_factors_ = static_cast<double*>(dalloc(std::max<std::size_t>(n_fac, 1) * sizeof(double)));
  d_ops_ = static_cast<M2LOp*>(dalloc(h_ops_.size() * sizeof(M2LOp)));
  d_tiles_ = static_cast<M2LTile*>(dalloc(tiles.size() * sizeof(M2LTile)));
  if (!gpu_inst) d_inst_ = static_cast<uint2*>(dalloc(std::max<std::size_t>(inst.size(), 1) * sizeof(uint2)));
  d_tile_ids_ = static_cast<int*>(dalloc(std::max<std::size_t>(ids.size(), 1) * sizeof(int)));
  d_far_part_ = static_cast<double*>(dalloc(std::max<std::size_t>(tiles.size(), 1) * sizeof(double)));
  if (gpu_fac) {
    M2LPack* d_packs = svd_tmp.alloc<M2LPack>(std::max<std::size_t>(packs.size(), 1));
    int* d_perms = svd_tmp.alloc<int>(std::max<std::size_t>(perms.size(), 1));
    ANKH_CUDA(cudaMemsetAsync(d_factors_, 0, n_fac * sizeof(double), stream_));
    ANKH_CUDA(cudaMemcpyAsync(d_packs, packs.data(), packs.size() * sizeof(M2LPack),
                              cudaMemcpyHostToDevice, stream_));
    ANKH_CUDA(cudaMemcpyAsync(d_perms, perms.data(), perms.size() * sizeof(int),
                              cudaMemcpyHostToDevice, stream_));
    launch_m2l_pack(d_packs, static_cast<int>(packs.size()), max_rows, d_perms, d_lf, d_rf, K, Kp,
                    d_factors_, stream_);
    ANKH_CUDA(cudaGetLastError());
  } else {
    ANKH_CUDA(cudaMemcpyAsync(d_factors_, h_factors.data(), h_factors.size() * sizeof(double),
                              cudaMemcpyHostToDevice, stream_));
  }
  ANKH_CUDA(cudaMemcpyAsync(d_ops_, h_ops_.data(), h_ops_.size() * sizeof(M2LOp),
                            cudaMemcpyHostToDevice, stream_));
  ANKH_CUDA(cudaMemcpyAsync(d_tiles_, tiles.data(), tiles.size() * sizeof(M2LTile),
                            cudaMemcpyHostToDevice, stream_));
  if (!gpu_inst)
    ANKH_CUDA(cudaMemcpyAsync(d_inst_, inst.data(), inst.size() * sizeof(uint2),
                              cudaMemcpyHostToDevice, stream_));
  if (!ids.empty())
    ANKH_CUDA(cudaMemcpyAsync(d_tile_ids_, ids.data(), ids.size() * sizeof(int),
                              cudaMemcpyHostToDevice, stream_));
  ANKH_CUDA(cudaMemsetAsync(d_far_part_, 0, std::max<std::size_t>(tiles.size(), 1) * sizeof(double), stream_));
  ANKH_CUDA(cudaStreamSynchronize(stream_));
  stamp("upload");
}

// build_periodic_operator (fmm.cpp:333-377): generator on the GPU, its r2c
// spectrum (FFTW layout, spectral.cpp:47-62) on the host, real part uploaded.
// ANKH-FFT engine (k_fft.cu): the equispaced transfer E (L_u x L_c), the
// circulant spectrum of the leaf-level far-field operator (generator + 6-D
// DFT on the device), the evaluation's work arrays, one far partial per
// energy CTA (summed by k_finalize as the far field), no M2L classes.
void Plan::build_fft() {
  const int Lu = cfg.order_equi;  // limits checked in the constructor, before any allocation
  fft_shape_ = fft_shape(depth, Lu);
  const FftShape& s = fft_shape_;
  const std::vector<double> E = transfer_equi(Lu, cheb_nodes(L));  // Lu x L
  d_fft_E_ = static_cast<double*>(dalloc(E.size() * sizeof(double)));
  ANKH_CUDA(cudaMemcpyAsync(d_fft_E_, E.data(), E.size() * sizeof(double), cudaMemcpyHostToDevice, stream_));
  const std::size_t cells = static_cast<std::size_t>(s.Pc) * s.Pc * s.Pc;
  d_fft_diag_ = static_cast<double*>(dalloc(cells * s.NF * sizeof(double)));
  d_fft_x0_ = static_cast<double2*>(dalloc(cells * s.NF * sizeof(double2)));  // precompute size (largest)
  d_fft_x1_ = static_cast<double2*>(dalloc(cells * s.NF * sizeof(double2)));
  launch_fft_precompute(s, depth, rb, cfg.xi, periodic ? 1 : 0, d_fft_x0_, d_fft_x1_, d_fft_diag_, stream_);
  ANKH_CUDA(cudaGetLastError());
  n_tiles_ = static_cast<int>(s.energy_blocks);
  d_far_part_ = static_cast<double*>(dalloc(static_cast<std::size_t>(n_tiles_) * sizeof(double)));
  class_range_.assign(kMaxKp8 + 1, {0, 0});
  class_leaf_.assign(kMaxKp8 + 1, 0);
  far_flops = 0.0;
  m2l_instances = 0;
  m2l_operators = 0;
  ANKH_CUDA(cudaStreamSynchronize(stream_));
}

void Plan::build_periodic() {
  const int eb = 2 * L - 1;
  const std::size_t m = static_cast<std::size_t>(eb) * eb * eb;
  double* d_gen = static_cast<double*>(dalloc(m * sizeof(double)));
  d_gen_ = d_gen;  // kept: the forces' periodic term applies the operator directly
  launch_periodic_gen(d_gen, L, rb, cfg.xi, cfg.p, stream_);
  ANKH_CUDA(cudaGetLastError());
  std::vector<double> gen(m);
  ANKH_CUDA(cudaMemcpyAsync(gen.data(), d_gen, m * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  ANKH_CUDA(cudaStreamSynchronize(stream_));
  const std::vector<double> spec = r2c_3d(gen, eb, eb, eb);
  std::vector<double> re(spec.size() / 2);
  for (std::size_t i = 0; i < re.size(); ++i) re[i] = spec[2 * i];
  d_spec_re_ = static_cast<double*>(dalloc(re.size() * sizeof(double)));
  ANKH_CUDA(cudaMemcpyAsync(d_spec_re_, re.data(), re.size() * sizeof(double),
                            cudaMemcpyHostToDevice, stream_));
  ANKH_CUDA(cudaStreamSynchronize(stream_));
}

void Plan::validate_only(const double* d_pos, const double* d_src, cudaStream_t st) {
  // per-particle flags and duplicates (types.cpp:16-63) without a tree
  launch_init_result(d_res_, st);
  const int nax8 = 256;  // depth-8 bins keep the duplicate scan local
  const double inv_side = nax8 / (2.0 * rb);
  launch_bin(d_pos, d_src, n, rb, inv_side, nax8, d_keys_, d_idx_, nullptr, d_res_, st);
  launch_sort(d_temp_, temp_bytes_, d_keys_, d_keys2_, d_idx_, d_idx2_, n, 24, st);
  launch_dup_check(d_keys2_, d_idx2_, d_pos, n, d_res_, st);
  ANKH_CUDA(cudaMemcpyAsync(h_res_, d_res_, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
  launches_ = 3;
}

// the upward pass for parent levels first .. top (whole subtrees from
// p_begin): the chained one-launch kernel for the compiled orders, per-level
// runtime-order launches past them
void Plan::launch_m2m(int first, int top, cudaStream_t st, unsigned p_begin, unsigned p_count) {
  if (L <= kMaxOrderCompiled)
    launch_m2m_chain(d_exp_, d_level_off_, first, top, L, d_m2m_, d_m2m_cnt_, st, p_begin, p_count);
  else
    launch_m2m_generic(d_exp_, level_off_.data(), first, top, L, d_m2m_, d_m2m_scratch_, st, p_begin, p_count);
}

void Plan::launch_all(const double* d_pos, const double* d_src, cudaStream_t st, int mode) {
  const bool timing = cfg.phase_timing != 0 && (mode == 0 || mode == 3);
  std::uint32_t launches = 0;
  if (timing) ANKH_CUDA(cudaEventRecord(ev_[0], st));
  if (mode == 3) {
    // positions validated and sorted by set_positions: start from their flags,
    // validate the moments, gather the records through the sorted index
    ANKH_CUDA(cudaMemcpyAsync(d_res_, d_res_pos_, sizeof(DevResult), cudaMemcpyDeviceToDevice, st));
    ANKH_CUDA(cudaMemsetAsync(d_leaf_mp_, 0, static_cast<std::size_t>(n_leaves) * sizeof(unsigned), st));
    launch_src_gather(d_pos, d_src, d_idx2_, n, d_res_, d_part_, st, d_keys_, d_leaf_mp_);
    launches += 2;
  } else if (mode != 2) {
    // sliced moments: other slices' multipoles are unseen, so the kernels
    // that branch on the global flag take the multipole path (same energies)
    launch_init_result(d_res_, st, slice_src_ ? 1 : 0, d_counts_, static_cast<unsigned>(n_leaves + 1));
    ++launches;
    // binning + sort + gather (build_tree, octree.cpp:27-45)
    const double inv_side = nax / (2.0 * rb);  // octree.cpp:35
    // moments: checked by the record gather when it visits every leaf (one
    // read of them), by a slice pass on sliced shards, else by k_bin
    const bool gather_src = gather_checks_src();
    launch_bin(d_pos, (slice_src_ || gather_src) ? nullptr : d_src, n, rb, inv_side, nax, d_keys_, d_idx_,
               d_counts_, d_res_, st, d_need_);
    ++launches;
    if (slice_src_ && src_i1_ > src_i0_) {  // this shard's moment slice (self partials, flags)
      launch_src_chunk(d_pos, d_src, nullptr, src_i0_, src_i1_, d_res_, nullptr, st);
      ++launches;
    }
    // counting sort by leaf: d_idx_ holds the arrival slots, d_keys2_ the
    // scattered indices, d_idx2_ the leaf CSR's ascending indices
    launch_bucket_gather(scan_, d_pos, d_src, d_keys_, d_idx_, d_counts_, d_off_,
                         d_keys2_, d_idx_, d_idx2_, n, n_leaves, d_need_, d_part_, st, gather_src, d_res_,
                         d_leaf_mp_);
    launches += 2;
  }
  if (csr_only_) {
    launches_ = launches;
    return;
  }
  // The far-field chain (P2M -> M2M -> M2L -> periodic) and the near field
  // (P2P) only share the sorted particle records: without phase timing they
  // run concurrently on two streams (P2M/M2M are latency-bound and hide under
  // P2P).  With phase timing -- or when the caller drives the two halves
  // itself (mode 1/2, in-process shard exchange) -- they run back to back.
  const bool serial = timing || mode == 1 || mode == 2;
  const bool do_periodic = periodic && include_self_;
  cudaStream_t far = st;
  if (!serial) {
    ANKH_CUDA(cudaEventRecord(ev_fork_, st));
    ANKH_CUDA(cudaStreamWaitEvent(side_stream_, ev_fork_, 0));
    far = side_stream_;
  }
  if (timing) ANKH_CUDA(cudaEventRecord(ev_[1], st));
  // interpolation: P2M over this shard's Morton leaf range (fmm.cpp:181-201) ...
  if (mode != 2) {
    launch_p2m(d_part_, d_off_, depth, L, rb, d_hd_, d_exp_ + level_off_[depth], d_res_, d_self_leaf_, cfg.xi,
               static_cast<unsigned>(p2m_begin_), static_cast<unsigned>(p2m_end_), far);
    ++launches;
  }
  if (mode == 1) {
    launches_ = launches;
    return;
  }
  // ... the leaf level completed by the shard exchange, then M2M (fmm.cpp:203-236)
  m2m_top_ = depth - 1;
  if (mode == 0 || mode == 3) launches += exchange_upward(far);
  if (serial) {
    if (m2m_top_ >= 0) {
      launch_m2m(m2m_top_, 0, far);
      ++launches;
    }
    if (timing) ANKH_CUDA(cudaEventRecord(ev_[2], st));
    // far field: M2L (fmm.cpp:238-276); the periodic term follows P2P below
    for (int c = 1; c <= kMaxKp8; ++c) {
      const auto r = class_range_[c];
      if (r.second == 0) continue;
      launch_m2l(d_exp_, d_level_off_, d_factors_, d_ops_, d_tiles_, r.second, c, d_tile_ids_ + r.first, d_inst_,
                 K, Kp, d_far_part_, far);
      ++launches;
    }
    if (fft_) launches += launch_fft(far);
    if (timing) ANKH_CUDA(cudaEventRecord(ev_[3], st));
  } else {
    // M2M, M2L and the periodic far images (counted once, rank 0) in branches
    launches += launch_far_chain(far, true, do_periodic);
  }
  if (!serial) ANKH_CUDA(cudaEventRecord(ev_join_, far));
  // near field: P2P (fmm.cpp:278-327)
  const int n_near_parts =
      launch_p2p(d_part_, d_off_, d_leaf_mp_, depth, periodic ? 1 : 0, 2.0 * rb, cfg.xi, radial_,
                 p2p_cap_, leaf_begin_, leaf_end_,
                 d_near_part_, d_pair_count_, d_res_, st);
  ++launches;
  if (timing) ANKH_CUDA(cudaEventRecord(ev_[4], st));
  if (serial && do_periodic) {
    launch_periodic_eval(d_exp_, d_to_equi_, d_spec_re_, L, d_per_, st, d_per_scratch_);
    ++launches;
  }
  if (!serial) ANKH_CUDA(cudaStreamWaitEvent(st, ev_join_, 0));
  if (timing) ANKH_CUDA(cudaEventRecord(ev_[5], st));
  // self energy: per-leaf sums from P2M over this shard's P2M rows -- split
  // across shards when P2M is (shard_upward_), else counted by rank 0
  const bool count_self = include_self_ || shard_upward_;
  launch_finalize(d_near_part_, n_near_parts, d_pair_count_, leaf_end_ - leaf_begin_, d_far_part_,
                  n_tiles_, d_self_leaf_ + p2m_begin_, static_cast<int>(p2m_end_ - p2m_begin_),
                  -cfg.xi * kInvSqrtPi, d_per_, do_periodic ? 1 : 0, count_self ? 1 : 0, d_fin_scratch_, d_res_,
                  st);
  ++launches;
  // shards: one all-reduce of the energy / counter / flag vector (the path's
  // only exchange besides the leaf all-gather), grouped with the MIN of the
  // first-violation indices when the moment pass is sliced
  static_assert(offsetof(DevResult, min_outside) == offsetof(DevResult, min_nonfinite) + 8,
                "min_nonfinite / min_outside are MIN-reduced as one pair");
  if (coll_) {
    if (slice_src_)
      coll_->allreduce_sum_min(d_res_->red, kRedShared, &d_res_->min_nonfinite, 2, st);
    else
      coll_->allreduce_sum(d_res_->red, kRedShared, st);
  }
  if (timing) ANKH_CUDA(cudaEventRecord(ev_[6], st));
  ANKH_CUDA(cudaMemcpyAsync(h_res_, d_res_, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
  ANKH_CUDA(cudaGetLastError());
  launches_ = launches;
}

// The far chain after the leaf level is complete: M2M (fmm.cpp:203-236),
// M2L by rank class (fmm.cpp:238-276; one kernel instantiation per padded
// rank) and, with `with_periodic`, the far-image term (fmm.cpp:421-427).
// Unforked: back to back on `far`.  Forked: the classes' leaf-level tiles
// (no M2M dependency) start at once on the kM2LStreams side branches while
// the M2M chain runs on `far`; the coarse-level tiles and the periodic term
// follow M2M on the least-loaded branches (greedy by tiles x padded rank);
// every branch joins back into `far`.
std::uint32_t Plan::launch_fft(cudaStream_t s) {
  launch_fft_far(fft_shape_, d_exp_ + level_off_[depth], Kp, depth, L, d_fft_E_, d_fft_x0_, d_fft_x1_, d_fft_diag_,
                 d_far_part_, s);
  return 4;
}

std::uint32_t Plan::launch_far_chain(cudaStream_t far, bool fork, bool with_periodic) {
  std::uint32_t launches = 0;
  std::vector<int> cls;
  for (int c = 1; c <= kMaxKp8; ++c)
    if (class_range_[c].second > 0) cls.push_back(c);
  auto work = [&](int c, int tiles) { return static_cast<long long>(tiles) * c; };
  auto m2l = [&](int c, int first, int count, cudaStream_t s) {
    if (count <= 0) return;
    launch_m2l(d_exp_, d_level_off_, d_factors_, d_ops_, d_tiles_, count, c, d_tile_ids_ + first, d_inst_, K, Kp,
               d_far_part_, s);
    ++launches;
  };
  auto m2m = [&](cudaStream_t s) {
    if (m2m_top_ < 0) return;  // (levels below m2m_top_ are done by exchange_upward)
    launch_m2m(m2m_top_, 0, s);
    ++launches;
  };
  if (!fork) {
    m2m(far);
    if (fft_) launches += launch_fft(far);
    for (int c : cls) m2l(c, class_range_[c].first, class_range_[c].second, far);
    if (with_periodic) {
      launch_periodic_eval(d_exp_, d_to_equi_, d_spec_re_, L, d_per_, far, d_per_scratch_);
      ++launches;
    }
    return launches;
  }
  cudaStream_t lane[1 + kM2LStreams] = {far};
  for (int k = 0; k < kM2LStreams; ++k) lane[1 + k] = m2l_streams_[k];
  long long load[1 + kM2LStreams] = {};
  bool forked[1 + kM2LStreams] = {true}, after_m2m[1 + kM2LStreams] = {true};
  ANKH_CUDA(cudaEventRecord(ev_m2l_fork_, far));
  auto pick = [&](int first) {
    int k = first;
    for (int j = first; j <= kM2LStreams; ++j)
      if (load[j] < load[k]) k = j;
    if (!forked[k]) {
      ANKH_CUDA(cudaStreamWaitEvent(lane[k], ev_m2l_fork_, 0));
      forked[k] = true;
    }
    return k;
  };
  // leaf-level tiles beside the M2M chain, largest first
  std::vector<int> order = cls;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return work(a, class_leaf_[a]) > work(b, class_leaf_[b]); });
  for (int c : order) {
    if (class_leaf_[c] == 0 || !m2l_split_) continue;
    const int k = pick(1);
    load[k] += work(c, class_leaf_[c]);
    m2l(c, class_range_[c].first, class_leaf_[c], lane[k]);
  }
  if (fft_) {  // the ANKH-FFT far field needs only the leaf level: beside M2M
    const int k = pick(1);
    load[k] += 1;
    launches += launch_fft(lane[k]);
  }
  m2m(far);
  ANKH_CUDA(cudaEventRecord(ev_m2m_done_, far));
  auto after = [&](int k) {
    if (!after_m2m[k]) {
      ANKH_CUDA(cudaStreamWaitEvent(lane[k], ev_m2m_done_, 0));
      after_m2m[k] = true;
    }
  };
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    const int ra = class_range_[a].second - (m2l_split_ ? class_leaf_[a] : 0);
    const int rb_ = class_range_[b].second - (m2l_split_ ? class_leaf_[b] : 0);
    return work(a, ra) > work(b, rb_);
  });
  for (int c : order) {
    const int skip = m2l_split_ ? class_leaf_[c] : 0;
    const int rest = class_range_[c].second - skip;
    if (rest <= 0) continue;
    const int k = pick(0);
    after(k);
    load[k] += work(c, rest);
    m2l(c, class_range_[c].first + skip, rest, lane[k]);
  }
  if (with_periodic) {
    const int k = pick(0);
    after(k);
    launch_periodic_eval(d_exp_, d_to_equi_, d_spec_re_, L, d_per_, lane[k], d_per_scratch_);
    ++launches;
  }
  for (int k = 1; k <= kM2LStreams; ++k)
    if (forked[k]) {
      ANKH_CUDA(cudaEventRecord(ev_m2l_join_[k - 1], lane[k]));
      ANKH_CUDA(cudaStreamWaitEvent(far, ev_m2l_join_[k - 1], 0));
    }
  return launches;
}

// Halo lists of the deep levels: for every peer q, the rows
// of this shard's cells q's M2L reads (send) and of q's cells this shard's
// M2L reads (receive), at levels halo_level_ .. depth.  Both sides enumerate
// a pair's list with the same rule in the same order, so the packed buffers
// line up without any index exchange.  ANKH_SHARD_ALLGATHER=1 keeps the
// whole-level all-gather (A/B).
void Plan::build_halo() {
  halo_level_ = depth + 1;
  halo_.clear();
  exchange_recv_bytes = exchange_send_bytes = 0;
  if (!shard_upward_ || cfg.world <= 1) return;
  const int G = cfg.world, r = cfg.rank;
  if (!std::getenv("ANKH_SHARD_ALLGATHER")) halo_level_ = shard_halo_level(depth, G);
  // the all-gathered levels exch_level_ .. halo_level_ - 1
  for (int l = exch_level_; l < std::min(halo_level_, depth + 1); ++l) {
    const std::size_t rows = static_cast<std::size_t>(1ll << (3 * l));
    exchange_recv_bytes += (rows - rows / G) * Kp * sizeof(double);
    exchange_send_bytes += (rows / G) * Kp * sizeof(double);
  }
  if (halo_level_ > depth) return;
  std::vector<long long> send_off, recv_off;    // row offsets (doubles) into d_exp_
  std::vector<std::size_t> send_at, recv_at;     // per peer: first packed row
  for (int q = 0; q < G; ++q) {
    if (q == r) continue;
    send_at.push_back(send_off.size());
    recv_at.push_back(recv_off.size());
    for (int l = halo_level_; l <= depth; ++l) {
      for (std::uint32_t m : shard_halo_cells(l, depth, periodic, r, q, G))
        send_off.push_back(level_off_[l] + static_cast<long long>(m) * Kp);
      for (std::uint32_t m : shard_halo_cells(l, depth, periodic, q, r, G))
        recv_off.push_back(level_off_[l] + static_cast<long long>(m) * Kp);
    }
  }
  send_at.push_back(send_off.size());
  recv_at.push_back(recv_off.size());
  halo_send_rows_ = static_cast<long long>(send_off.size());
  halo_recv_rows_ = static_cast<long long>(recv_off.size());
  d_halo_send_off_ = static_cast<long long*>(dalloc(std::max<std::size_t>(send_off.size(), 1) * sizeof(long long)));
  d_halo_recv_off_ = static_cast<long long*>(dalloc(std::max<std::size_t>(recv_off.size(), 1) * sizeof(long long)));
  d_halo_send_ = static_cast<double*>(dalloc(std::max<std::size_t>(send_off.size(), 1) * Kp * sizeof(double)));
  d_halo_recv_ = static_cast<double*>(dalloc(std::max<std::size_t>(recv_off.size(), 1) * Kp * sizeof(double)));
  ANKH_CUDA(cudaMemsetAsync(d_halo_recv_, 0, std::max<std::size_t>(recv_off.size(), 1) * Kp * sizeof(double), stream_));
  if (!send_off.empty())
    ANKH_CUDA(cudaMemcpyAsync(d_halo_send_off_, send_off.data(), send_off.size() * sizeof(long long),
                              cudaMemcpyHostToDevice, stream_));
  if (!recv_off.empty())
    ANKH_CUDA(cudaMemcpyAsync(d_halo_recv_off_, recv_off.data(), recv_off.size() * sizeof(long long),
                              cudaMemcpyHostToDevice, stream_));
  for (int q = 0, k = 0; q < G; ++q) {
    if (q == r) continue;
    halo_.push_back({q, d_halo_send_ + send_at[k] * Kp, (send_at[k + 1] - send_at[k]) * Kp,
                     d_halo_recv_ + recv_at[k] * Kp, (recv_at[k + 1] - recv_at[k]) * Kp});
    ++k;
  }
  exchange_recv_bytes += recv_off.size() * Kp * sizeof(double);
  exchange_send_bytes += send_off.size() * Kp * sizeof(double);
  ANKH_CUDA(cudaStreamSynchronize(stream_));
}

double* Plan::halo_recv_from(int src) const {
  for (const HaloPeer& h : halo_)
    if (h.peer == src) return h.recv;
  return nullptr;
}

// Sharded upward pass with a collective attached: M2M of this shard's own
// subtree cells for the parent levels exch_level_ .. depth-1 (at level l the
// shard owns Morton cells [r 8^l / G, (r+1) 8^l / G) -- whole subtrees, since
// G | 8^exch_level_), then ONE exchange group: an in-place all-gather of the
// coarse levels exch_level_ .. halo_level_-1 and the M2L halo rows of the deep
// levels (packed before, unpacked after); the levels above exch_level_ are
// completed redundantly by every shard (m2m_top_).  Returns the launches.
std::uint32_t Plan::exchange_upward(cudaStream_t st) {
  m2m_top_ = depth - 1;
  if (!coll_ || !shard_upward_) return 0;
  std::uint32_t launches = 0;
  const long long G = cfg.world, r = cfg.rank;
  if (depth - 1 >= exch_level_) {  // this shard's subtrees, parent levels depth-1 .. exch_level_
    const long long cells = 1ll << (3 * (depth - 1));
    launch_m2m(depth - 1, exch_level_, st, static_cast<unsigned>(cells * r / G), static_cast<unsigned>(cells / G));
    ++launches;
  }
  std::vector<double*> recv;
  std::vector<std::size_t> count;
  for (int l = exch_level_; l <= std::min(halo_level_ - 1, depth); ++l) {
    recv.push_back(d_exp_ + level_off_[l]);
    count.push_back(static_cast<std::size_t>((1ll << (3 * l)) / G) * Kp);
  }
  if (halo_send_rows_ > 0) {
    launch_halo_rows(d_exp_, d_halo_send_off_, halo_send_rows_, Kp, d_halo_send_, false, st);
    ++launches;
  }
  coll_->upward_exchange(recv.data(), count.data(), static_cast<int>(recv.size()), halo_, st);
  if (halo_recv_rows_ > 0) {
    launch_halo_rows(d_exp_, d_halo_recv_off_, halo_recv_rows_, Kp, d_halo_recv_, true, st);
    ++launches;
  }
  m2m_top_ = exch_level_ - 1;
  return launches;
}

void Plan::enqueue(const double* d_pos, const double* d_src, cudaStream_t st) {
  if (!st) st = stream_;
  last_stream_ = st;
  evaluated_ = true;
  streamed_last_ = false;
  bound_ = stream_bound_ = false;  // a full evaluation re-bins: bound positions are superseded
  if (n == 0) return;
  if (pending_code_ != 0) {
    validate_only(d_pos, d_src, st);
    return;
  }
  if (shard_upward_ && !coll_)
    throw AnkhError(ANKH_RUNTIME_ERROR,
                    "sharded plan (world > 1) needs ankh_plan_attach_nccl_v1 or the "
                    "ankh_plan_enqueue_phase_v1 exchange");
  // Repeated evaluations on the same input buffers replay a CUDA graph of the
  // whole launch sequence (captured on the second such call, after the first
  // has set every kernel attribute); phase timing keeps plain launches.
  if (cfg.phase_timing || csr_only_) {
    launch_all(d_pos, d_src, st);
    return;
  }
  if (graph_exec_ && graph_pos_ == d_pos && graph_src_ == d_src) {
    ANKH_CUDA(cudaGraphLaunch(graph_exec_, st));
    return;
  }
  if (graph_warm_pos_ == d_pos && graph_warm_src_ == d_src) {
    if (graph_exec_) {
      cudaGraphExecDestroy(graph_exec_);
      graph_exec_ = nullptr;
    }
    cudaGraph_t g = nullptr;
    ANKH_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      launch_all(d_pos, d_src, st);
    } catch (...) {
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    ANKH_CUDA(cudaStreamEndCapture(st, &g));
    const cudaError_t e = cudaGraphInstantiate(&graph_exec_, g, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(g);
    ANKH_CUDA(e);
    graph_pos_ = d_pos;
    graph_src_ = d_src;
    ANKH_CUDA(cudaGraphLaunch(graph_exec_, st));
    return;
  }
  graph_warm_pos_ = d_pos;
  graph_warm_src_ = d_src;
  launch_all(d_pos, d_src, st);
}

bool Plan::stream_eligible() const {
  const char* e = std::getenv("ANKH_STREAM_INPUT");  // "0": never, "1": any size
  if (e && e[0] == '0') return false;
  const std::size_t min_n = (e && e[0] == '1') ? 1 : 65536;
  return n >= min_n && cfg.world <= 1 && !shard_upward_ && !coll_ && !csr_only_ &&
         pending_code_ == 0 && L <= 6;
}

void Plan::stream_setup() {
  if (stream_init_) return;
  {
    if (const char* c = std::getenv("ANKH_STREAM_CHUNKS")) stream_chunks_ = std::atoi(c);
    stream_chunks_ = std::max(1, std::min(stream_chunks_, kMaxStreamChunks));
    d_inv_ = static_cast<unsigned*>(dalloc(n * sizeof(unsigned)));
    d_ready_ = static_cast<unsigned char*>(dalloc(2 * static_cast<std::size_t>(n_leaves)));
    d_scnt_ = static_cast<unsigned*>(dalloc(4 * kMaxStreamChunks * sizeof(unsigned)));  // list counts, cursors
    d_sbounds_ = static_cast<unsigned*>(dalloc(2 * (kMaxStreamChunks + 1) * sizeof(unsigned)));
    ANKH_CUDA(cudaMallocHost(&h_sbounds_, 2 * (kMaxStreamChunks + 1) * sizeof(unsigned)));
    d_list_p2m_ = static_cast<unsigned*>(dalloc(static_cast<std::size_t>(n_leaves) * sizeof(unsigned)));
    d_list_p2p_ = static_cast<unsigned*>(dalloc(static_cast<std::size_t>(n_leaves) * sizeof(unsigned)));
    ANKH_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, device_));
    ANKH_CUDA(cudaStreamCreateWithFlags(&p2p_stream2_, cudaStreamNonBlocking));
    ANKH_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
    ANKH_CUDA(cudaStreamCreateWithPriority(&gather_stream_, cudaStreamNonBlocking, hi_prio_));
    for (cudaEvent_t* e : {&ev_s_start_, &ev_s_binned_, &ev_s_lists_, &ev_s_sorted_, &ev_s_inv_, &ev_s_p2p2_})
      ANKH_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (int c = 0; c < kMaxStreamChunks; ++c) {
      ANKH_CUDA(cudaEventCreateWithFlags(&ev_s_chunk_[c], cudaEventDisableTiming));
      ANKH_CUDA(cudaEventCreateWithFlags(&ev_s_gath_[c], cudaEventDisableTiming));
      ANKH_CUDA(cudaEventCreateWithFlags(&ev_s_posc_[c], cudaEventDisableTiming));
    }
    // chunk schedules in whole 256-particle blocks (k_bin's block layout):
    // the moments' first chunk is half a regular one (the evaluation starts
    // as soon as it lands), the rest equal; positions in equal chunks
    if (const char* c = std::getenv("ANKH_STREAM_POS_CHUNKS")) stream_pos_chunks_ = std::atoi(c);
    stream_pos_chunks_ = std::max(1, std::min(stream_pos_chunks_, kMaxStreamChunks));
    const std::size_t blocks = (n + 255) / 256;
    auto schedule = [&](int C, double first) {
      StreamChunks ch{};
      std::vector<std::size_t> b(1, 0);
      const double w0 = first / (first + (C - 1));
      if (C > 1) b.push_back(std::max<std::size_t>(1, static_cast<std::size_t>(w0 * blocks + 0.5)));
      for (int c = static_cast<int>(b.size()); c < C; ++c) {
        const std::size_t rest = blocks - b[1];
        b.push_back(b[1] + (rest * (c - 1) + (C - 2)) / (C - 1));
      }
      b.push_back(blocks);
      for (std::size_t c = 0; c + 1 < b.size(); ++c)
        if (b[c + 1] > b[c]) ch.start[ch.n++] = static_cast<unsigned>(std::min(n, 256 * b[c]));
      ch.start[ch.n] = static_cast<unsigned>(n);
      return ch;
    };
    double first = 0.5;
    if (const char* f = std::getenv("ANKH_STREAM_FIRST")) first = std::atof(f);
    sch_ = schedule(stream_chunks_, first);
    pch_ = schedule(stream_pos_chunks_, 1.0);
    for (auto& e : ev_t_) ANKH_CUDA(cudaEventCreate(&e));
    ANKH_CUDA(cudaStreamSynchronize(stream_));  // pool allocations complete before other streams use them
    stream_init_ = true;
  }
}

// positions half of the streamed path: validation and binning of each
// positions chunk as it lands (pos_ev; nullptr: all in), then the per-leaf
// sort (build_tree, as set_positions) with the inverse permutation on `st`,
// and -- beside it on side_stream_ -- the per-chunk leaf lists (their bounds
// stay on the device: the chunk kernels read them there).  `after_inverse`
// is recorded once the inverse permutation -- all the chunk gathers need --
// is in; on return `st` has also joined the lists.
void Plan::stream_positions(cudaStream_t st, DevResult* res, const cudaEvent_t* pos_ev,
                            const std::function<void(const std::string&)>& mark, cudaEvent_t after_inverse) {
  launch_init_result(res, st, 0, d_counts_, static_cast<unsigned>(2 * (n_leaves + 1)));
  const double inv_side = nax / (2.0 * rb);  // octree.cpp:35
  for (int p = 0; p < pch_.n; ++p) {
    if (pos_ev) ANKH_CUDA(cudaStreamWaitEvent(st, pos_ev[p], 0));
    launch_bin(d_pos_, nullptr, n, rb, inv_side, nax, d_keys_, d_idx_, d_counts_, res, st, nullptr, pch_.start[p],
               pch_.start[p + 1], d_leafmax_);
  }
  if (mark) mark("  binned");
  ANKH_CUDA(cudaEventRecord(ev_s_binned_, st));
  ANKH_CUDA(cudaStreamWaitEvent(side_stream_, ev_s_binned_, 0));
  launch_stream_lists(d_leafmax_, depth, periodic ? 1 : 0, sch_, d_ready_, d_scnt_, d_sbounds_, d_list_p2m_,
                      d_list_p2p_, side_stream_);
  ANKH_CUDA(cudaEventRecord(ev_s_lists_, side_stream_));
  launch_bucket_gather(scan_, d_pos_, nullptr, d_keys_, d_idx_, d_counts_, d_off_, d_keys2_, d_idx_, d_idx2_, n,
                       n_leaves, nullptr, nullptr, st, false, nullptr, nullptr, d_inv_);
  if (after_inverse) ANKH_CUDA(cudaEventRecord(after_inverse, st));
  if (mark) mark("  leaf CSR + inverse");
  ANKH_CUDA(cudaStreamWaitEvent(st, ev_s_lists_, 0));
}

namespace {
bool page_locked(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}
}  // namespace

void Plan::enqueue_streamed(const double* h_pos, const double* h_src, cudaStream_t st) {
  // Repeated calls on the same page-locked host buffers replay a graph of the
  // whole streamed evaluation (its copies read the buffers' current
  // contents); pageable buffers, traces and phase timing launch directly.
  const bool graphable = !cfg.phase_timing && std::getenv("ANKH_STREAM_TRACE") == nullptr &&
                         std::getenv("ANKH_STREAM_NO_GRAPH") == nullptr && page_locked(h_pos) &&
                         page_locked(h_src);
  if (!graphable) {
    enqueue_streamed_launch(h_pos, h_src, st);
    return;
  }
  auto replayed = [&]() {  // host state an evaluation leaves behind
    last_stream_ = st;
    evaluated_ = true;
    if (h_pos) bound_ = stream_bound_ = false;
    streamed_last_ = true;
    launches_ = sgraph_launches_;
  };
  // the graph's chunk grids were sized from the lists of the evaluation
  // before its capture: when the last replay's lists (h_sbounds_) outgrow
  // them or shrink to under half (new positions), capture again
  if (sgraph_exec_ && sgraph_pos_ == h_pos && sgraph_src_ == h_src) {
    const int C = sch_.n;
    for (int k = 0; k < 2 * C; ++k) {
      const int set = k / C, c = k - set * C;
      const long long cnt = static_cast<long long>(h_sbounds_[set * (C + 1) + c + 1]) - h_sbounds_[set * (C + 1) + c];
      const long long g = sgraph_grid_[k];
      if (cnt > g || 2 * cnt + 16 < g) {
        cudaGraphExecDestroy(sgraph_exec_);
        sgraph_exec_ = nullptr;
        break;
      }
    }
  }
  if (sgraph_exec_ && sgraph_pos_ == h_pos && sgraph_src_ == h_src) {
    ANKH_CUDA(cudaGraphLaunch(sgraph_exec_, st));
    replayed();
    return;
  }
  if (sgraph_warm_ && sgraph_warm_pos_ == h_pos && sgraph_warm_src_ == h_src) {
    if (sgraph_exec_) {
      cudaGraphExecDestroy(sgraph_exec_);
      sgraph_exec_ = nullptr;
    }
    cudaGraph_t g = nullptr;
    ANKH_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_streamed_launch(h_pos, h_src, st);
    } catch (...) {
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    ANKH_CUDA(cudaStreamEndCapture(st, &g));
    const cudaError_t e = cudaGraphInstantiate(&sgraph_exec_, g, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(g);
    ANKH_CUDA(e);
    sgraph_pos_ = h_pos;
    sgraph_src_ = h_src;
    sgraph_launches_ = launches_;
    sgraph_grid_ = last_grids_;
    ANKH_CUDA(cudaGraphLaunch(sgraph_exec_, st));
    return;
  }
  sgraph_warm_ = true;
  sgraph_warm_pos_ = h_pos;
  sgraph_warm_src_ = h_src;
  enqueue_streamed_launch(h_pos, h_src, st);
}

void Plan::enqueue_streamed_launch(const double* h_pos, const double* h_src, cudaStream_t st) {
  // ANKH_STREAM_TRACE=1: stage timestamps (ms after the call) on stderr
  const bool trace = std::getenv("ANKH_STREAM_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  auto mark = [&](const std::string& what, cudaStream_t s) {
    if (!trace) return;
    cudaEvent_t e = nullptr;
    ANKH_CUDA(cudaEventCreate(&e));
    ANKH_CUDA(cudaEventRecord(e, s));
    marks.emplace_back(what, e);
  };
  // h_pos == nullptr: positions bound by set_positions (flags in d_res_pos_,
  // sorted order and per-chunk lists already built) -- stream the moments only
  const bool bound_pos = h_pos == nullptr;
  last_stream_ = st;
  evaluated_ = true;
  if (!bound_pos) bound_ = stream_bound_ = false;
  streamed_last_ = true;
  const bool timing = cfg.phase_timing != 0;
  stream_setup();
  const int C = sch_.n;
  // copies: positions, then the moment chunks (after the previous evaluation)
  ANKH_CUDA(cudaEventRecord(ev_s_start_, st));
  if (timing) ANKH_CUDA(cudaEventRecord(ev_t_[0], st));
  mark("start", st);
  ANKH_CUDA(cudaStreamWaitEvent(copy_stream_, ev_s_start_, 0));
  if (!bound_pos) {
    for (int p = 0; p < pch_.n; ++p) {
      const std::size_t i0 = pch_.start[p], i1 = pch_.start[p + 1];
      ANKH_CUDA(cudaMemcpyAsync(d_pos_ + 3 * i0, h_pos + 3 * i0, (i1 - i0) * 3 * sizeof(double),
                                cudaMemcpyHostToDevice, copy_stream_));
      ANKH_CUDA(cudaEventRecord(ev_s_posc_[p], copy_stream_));
    }
    mark("copy positions done", copy_stream_);
  }
  for (int c = 0; c < C; ++c) {
    const std::size_t i0 = sch_.start[c], i1 = sch_.start[c + 1];
    ANKH_CUDA(cudaMemcpyAsync(d_src_ + 10 * i0, h_src + 10 * i0, (i1 - i0) * 10 * sizeof(double),
                              cudaMemcpyHostToDevice, copy_stream_));
    ANKH_CUDA(cudaEventRecord(ev_s_chunk_[c], copy_stream_));
    mark("copy chunk " + std::to_string(c), copy_stream_);
  }
  if (!bound_pos) {
    stream_positions(st, d_res_, ev_s_posc_,
                     trace ? std::function<void(const std::string&)>([&](const std::string& w) { mark(w, st); })
                           : std::function<void(const std::string&)>(),
                     ev_s_inv_);
  } else {
    ANKH_CUDA(cudaMemcpyAsync(d_res_, d_res_pos_, sizeof(DevResult), cudaMemcpyDeviceToDevice, st));
    ANKH_CUDA(cudaEventRecord(ev_s_inv_, st));
  }
  ANKH_CUDA(cudaEventRecord(ev_s_sorted_, st));
  if (timing) ANKH_CUDA(cudaEventRecord(ev_t_[1], st));
  // this evaluation's list bounds for the next one's grids (D2H engine; read
  // by the host only after the caller's synchronisation)
  ANKH_CUDA(cudaMemcpyAsync(h_sbounds_, d_sbounds_, 2 * (C + 1) * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  mark("sorted + lists", st);
  ANKH_CUDA(cudaGetLastError());
  // No host wait: the chunk kernels read their leaf-list bounds on the device,
  // with grids sized by upper bounds (warps / CTAs stride over the list).
  // Records (gather stream) start once the inverse permutation is in; P2M
  // (far stream) and P2P wait for the lists; P2P chunks alternate between two
  // streams so one chunk's tail overlaps the next chunk's start.
  std::uint32_t launches = 9;
  ANKH_CUDA(cudaStreamWaitEvent(gather_stream_, ev_s_inv_, 0));
  // per-leaf multipole flags: OR-ed by the chunk gathers below
  ANKH_CUDA(cudaMemsetAsync(d_leaf_mp_, 0, static_cast<std::size_t>(n_leaves) * sizeof(unsigned), gather_stream_));
  ANKH_CUDA(cudaStreamWaitEvent(side_stream_, ev_s_sorted_, 0));
  ANKH_CUDA(cudaStreamWaitEvent(p2p_stream2_, ev_s_sorted_, 0));
  // P2P chunk grids: one CTA per listed leaf, sized from the previous
  // evaluation's list (the block scheduler balances short-lived CTAs, and the
  // far chain's higher-priority CTAs interleave as they exit); the first
  // evaluation strides two waves over each list.  (A persistent work-counter
  // variant kept P2P's CTAs resident and pushed M2L behind it: 6.28 vs 6.16
  // ms per streamed call at config 3.)
  const bool sized = h_sbounds_valid_ && std::getenv("ANKH_P2P_STRIDE") == nullptr;
  int p2p_group = 1;
  if (const char* g = std::getenv("ANKH_STREAM_P2P_GROUP")) p2p_group = std::max(1, std::atoi(g));
  auto p2p_grid = [&](int c) {
    if (!sized) return static_cast<int>(std::min<long long>(n_leaves, 6ll * sm_count_));
    const long long cnt = static_cast<long long>(h_sbounds_[C + 1 + c + 1]) - h_sbounds_[C + 1 + c];
    return static_cast<int>(std::max(1ll, std::min<long long>(n_leaves, cnt + cnt / 16 + 8)));
  };
  // P2M: one warp per listed leaf, sized the same way (else 32 warps per SM striding)
  last_grids_.assign(2 * static_cast<std::size_t>(C), 0);
  auto p2m_cap = [&](int c) {
    if (!sized) return static_cast<unsigned>(std::min<long long>(n_leaves, 32ll * sm_count_));
    const long long cnt = static_cast<long long>(h_sbounds_[c + 1]) - h_sbounds_[c];
    return static_cast<unsigned>(std::max(1ll, std::min<long long>(n_leaves, cnt + cnt / 16 + 8)));
  };
  const bool do_periodic = periodic && include_self_;
  int n_near_parts = leaf_end_ - leaf_begin_;
  for (int c = 0; c < C; ++c) {
    const std::size_t i0 = sch_.start[c], i1 = sch_.start[c + 1];
    ANKH_CUDA(cudaStreamWaitEvent(gather_stream_, ev_s_chunk_[c], 0));
    launch_src_chunk(d_pos_, d_src_, d_inv_, i0, i1, d_res_, d_part_, gather_stream_, d_keys_, d_leaf_mp_);
    ANKH_CUDA(cudaEventRecord(ev_s_gath_[c], gather_stream_));
    mark("gather " + std::to_string(c), gather_stream_);
    ANKH_CUDA(cudaStreamWaitEvent(side_stream_, ev_s_gath_[c], 0));
    launch_p2m(d_part_, d_off_, depth, L, rb, d_hd_, d_exp_ + level_off_[depth], d_res_, d_self_leaf_, cfg.xi, 0u,
               0u, side_stream_, d_list_p2m_, d_sbounds_ + c, p2m_cap(c));
    last_grids_[c] = p2m_cap(c);
    mark("p2m " + std::to_string(c), side_stream_);
    // P2P for the lists of chunks [c0, c] once every `group` chunks (one
    // launch over consecutive lists; ANKH_STREAM_P2P_GROUP, default 1 --
    // config 3, 16 chunks: groups of 1 / 2 / 4 measured 5.89 / 5.98 / 6.14 ms
    // per streamed call: the launch tails are not what the path loses)
    if ((c + 1) % p2p_group != 0 && c != C - 1) {
      launches += 2;
      continue;
    }
    const int c0 = c - (c % p2p_group);  // the first chunk of this group
    long long grid_sum = 0;
    for (int cc = c0; cc <= c; ++cc) grid_sum += p2p_grid(cc);
    const int pgrid = static_cast<int>(std::min<long long>(n_leaves, grid_sum));
    cudaStream_t ps = ((c / p2p_group) & 1) ? p2p_stream2_ : st;
    ANKH_CUDA(cudaStreamWaitEvent(ps, ev_s_gath_[c], 0));
    if (timing && c0 == 0) ANKH_CUDA(cudaEventRecord(ev_t_[2], st));
    n_near_parts = launch_p2p(d_part_, d_off_, d_leaf_mp_, depth, periodic ? 1 : 0, 2.0 * rb, cfg.xi, radial_,
                              p2p_cap_, leaf_begin_, leaf_end_, d_near_part_, d_pair_count_, d_res_, ps,
                              d_list_p2p_, d_sbounds_ + (C + 1) + c0, pgrid, c - c0 + 1);
    for (int cc = c0; cc <= c; ++cc) last_grids_[C + cc] = p2p_grid(cc);
    mark("p2p " + std::to_string(c), ps);
    launches += 3;
  }
  // the last chunk's records are in before the tail (far stream waits below)
  ANKH_CUDA(cudaStreamWaitEvent(side_stream_, ev_s_gath_[C - 1], 0));
  ANKH_CUDA(cudaEventRecord(ev_s_p2p2_, p2p_stream2_));
  ANKH_CUDA(cudaStreamWaitEvent(st, ev_s_p2p2_, 0));
  ANKH_CUDA(cudaStreamWaitEvent(st, ev_s_gath_[C - 1], 0));
  if (timing) ANKH_CUDA(cudaEventRecord(ev_t_[3], st));
  if (timing) {  // phase spans: M2M, M2L, periodic back to back
    launch_m2m(depth - 1, 0, side_stream_);
    ++launches;
    ANKH_CUDA(cudaEventRecord(ev_t_[4], side_stream_));
    for (int c = 1; c <= kMaxKp8; ++c) {
      const auto r = class_range_[c];
      if (r.second == 0) continue;
      launch_m2l(d_exp_, d_level_off_, d_factors_, d_ops_, d_tiles_, r.second, c, d_tile_ids_ + r.first, d_inst_,
                 K, Kp, d_far_part_, side_stream_);
      ++launches;
    }
    if (fft_) launches += launch_fft(side_stream_);
    ANKH_CUDA(cudaEventRecord(ev_t_[5], side_stream_));
    if (do_periodic) {
      launch_periodic_eval(d_exp_, d_to_equi_, d_spec_re_, L, d_per_, side_stream_, d_per_scratch_);
      ++launches;
    }
    ANKH_CUDA(cudaEventRecord(ev_t_[6], side_stream_));
  } else {
    m2m_top_ = depth - 1;
    launches += launch_far_chain(side_stream_, true, do_periodic);
  }
  mark("far chain (m2m, m2l, periodic)", side_stream_);
  ANKH_CUDA(cudaEventRecord(ev_join_, side_stream_));
  ANKH_CUDA(cudaStreamWaitEvent(st, ev_join_, 0));
  if (timing) ANKH_CUDA(cudaEventRecord(ev_t_[7], st));
  launch_finalize(d_near_part_, n_near_parts, d_pair_count_, leaf_end_ - leaf_begin_, d_far_part_, n_tiles_,
                  d_self_leaf_, n_leaves, -cfg.xi * kInvSqrtPi, d_per_, do_periodic ? 1 : 0,
                  include_self_ ? 1 : 0, d_fin_scratch_, d_res_, st);
  ++launches;
  if (timing) ANKH_CUDA(cudaEventRecord(ev_t_[8], st));
  ANKH_CUDA(cudaMemcpyAsync(h_res_, d_res_, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
  mark("finalize + result copy", st);
  ANKH_CUDA(cudaGetLastError());
  launches_ = launches;
  h_sbounds_valid_ = true;
  if (trace) {
    ANKH_CUDA(cudaStreamSynchronize(st));
    for (auto& m : marks) {
      float ms = 0.f;
      ANKH_CUDA(cudaEventElapsedTime(&ms, marks[0].second, m.second));
      std::fprintf(stderr, "[ankh stream] %8.3f ms  %s\n", ms, m.first.c_str());
    }
    for (auto& m : marks) cudaEventDestroy(m.second);
  }
}

void Plan::enqueue_host(const double* h_pos, const double* h_src, cudaStream_t st) {
  if (!st) st = stream_;
  if (stream_eligible()) {
    enqueue_streamed(h_pos, h_src, st);
    return;
  }
  if (n > 0) {
    ANKH_CUDA(cudaMemcpyAsync(d_pos_, h_pos, n * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
    // a shard with a sliced moment pass reads moments only for the leaves it
    // touches and for its index slice: from page-locked host memory it reads
    // them in place (mapped, over PCIe) instead of copying all N
    if (slice_src_ && pending_code_ == 0 && std::getenv("ANKH_SHARD_COPY_SRC") == nullptr) {
      cudaPointerAttributes a{};
      if (cudaPointerGetAttributes(&a, h_src) == cudaSuccess && a.type == cudaMemoryTypeHost &&
          a.devicePointer != nullptr) {
        enqueue(d_pos_, static_cast<const double*>(a.devicePointer), st);
        return;
      }
      cudaGetLastError();
    }
    ANKH_CUDA(cudaMemcpyAsync(d_src_, h_src, n * 10 * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  enqueue(d_pos_, d_src_, st);
}

void Plan::set_positions(const double* h_pos, cudaStream_t st) {
  if (!st) st = stream_;
  bound_ = stream_bound_ = false;
  if (n == 0) {
    bound_ = true;
    return;
  }
  if (stream_eligible()) {  // energy_sources will stream the moments chunk by chunk
    stream_setup();
    ANKH_CUDA(cudaMemcpyAsync(d_pos_, h_pos, n * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
    stream_positions(st, d_res_pos_, nullptr);
    ANKH_CUDA(cudaStreamSynchronize(st));
    bound_ = stream_bound_ = true;
    return;
  }
  ANKH_CUDA(cudaMemcpyAsync(d_pos_, h_pos, n * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
  if (pending_code_ == 0 && !csr_only_) {
    launch_init_result(d_res_pos_, st, 0, d_counts_, static_cast<unsigned>(n_leaves + 1));
    const double inv_side = nax / (2.0 * rb);  // octree.cpp:35
    launch_bin(d_pos_, nullptr, n, rb, inv_side, nax, d_keys_, d_idx_, d_counts_, d_res_pos_, st, d_need_);
    launch_bucket_gather(scan_, d_pos_, nullptr, d_keys_, d_idx_, d_counts_,
                         d_off_, d_keys2_, d_idx_, d_idx2_, n, n_leaves, d_need_, nullptr, st);
  }
  ANKH_CUDA(cudaGetLastError());
  bound_ = true;
}

void Plan::enqueue_sources(const double* h_src, cudaStream_t st) {
  if (!bound_) throw AnkhError(ANKH_RUNTIME_ERROR, "plan positions are not set (ankh_plan_set_positions_v1)");
  if (!st) st = stream_;
  if (stream_bound_ && stream_eligible()) {
    enqueue_streamed(nullptr, h_src, st);
    return;
  }
  last_stream_ = st;
  evaluated_ = true;
  streamed_last_ = false;
  if (n == 0) return;
  ANKH_CUDA(cudaMemcpyAsync(d_src_, h_src, n * 10 * sizeof(double), cudaMemcpyHostToDevice, st));
  if (pending_code_ != 0) {
    validate_only(d_pos_, d_src_, st);
    return;
  }
  if (shard_upward_ && !coll_)
    throw AnkhError(ANKH_RUNTIME_ERROR,
                    "sharded plan (world > 1) needs ankh_plan_attach_nccl_v1");
  if (cfg.phase_timing) {
    launch_all(d_pos_, d_src_, st, 3);
    return;
  }
  // same CUDA-graph policy as enqueue: plain launches once, then capture and replay
  if (!graph_src_exec_ && graph_src_warm_ > 0) {
    cudaGraph_t g = nullptr;
    ANKH_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      launch_all(d_pos_, d_src_, st, 3);
    } catch (...) {
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    ANKH_CUDA(cudaStreamEndCapture(st, &g));
    const cudaError_t e = cudaGraphInstantiate(&graph_src_exec_, g, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(g);
    ANKH_CUDA(e);
  }
  if (graph_src_exec_) {
    ANKH_CUDA(cudaGraphLaunch(graph_src_exec_, st));
    return;
  }
  ++graph_src_warm_;
  launch_all(d_pos_, d_src_, st, 3);
}

void Plan::result(ankh_report_v1* out) {
  if (!evaluated_) throw AnkhError(ANKH_RUNTIME_ERROR, "plan has not been evaluated");
  std::memset(out, 0, sizeof(*out));
  out->depth = depth;
  out->order_cheb = L;
  if (n == 0) {
    if (pending_code_ != 0) throw AnkhError(pending_code_, pending_msg_);
    return;
  }
  ANKH_CUDA(cudaStreamSynchronize(last_stream_));
  check_guards();
  const DevResult& r = *h_res_;
  // validate_system precedence: first per-particle violation, then duplicates
  if (r.min_nonfinite != ~0ull || r.min_outside != ~0ull) {
    const bool nf = r.min_nonfinite <= r.min_outside;
    throw AnkhError(ANKH_INVALID_ARGUMENT,
                    std::string("fmm_energy: invalid system: ") +
                        (nf ? "non-finite coordinate or moment" : "outside box"));
  }
  if (r.red[kDuplicate] > 0.0)
    throw AnkhError(ANKH_INVALID_ARGUMENT, "fmm_energy: invalid system: duplicate position");
  if (pending_code_ != 0) throw AnkhError(pending_code_, pending_msg_);
  if (r.red[kCoincident] > 0.0)
    throw AnkhError(ANKH_DOMAIN_ERROR, "pair_interaction: coincident points");
  out->e_self = r.red[kESelf];
  out->e_near = r.red[kENear];
  out->e_far = r.red[kEFar];
  out->e_periodic_far = r.red[kEPeriodic];
  out->e_reciprocal = 0.0;
  // EnergyReport::component_sum order (types.hpp:132-134)
  out->e_total = out->e_self + out->e_near + out->e_far + out->e_periodic_far + out->e_reciprocal;
  out->near_pairs = static_cast<std::uint64_t>(r.red[kNearPairs]);
  out->far_instances = m2l_instances;  // this shard's (the instance lists are per shard)
  out->far_flops = far_flops;
  out->gpu_launches = launches_;
  if (cfg.phase_timing && streamed_last_) {
    // overlapped phases: wall-clock span of each (they may sum to more than
    // the total); interpolation = chunk gathers + P2M + M2M, precompute =
    // the positions copy, binning and sort
    auto span = [&](int a, int b) {
      float ms = 0.f;
      ANKH_CUDA(cudaEventElapsedTime(&ms, ev_t_[a], ev_t_[b]));
      return ms * 1e-3;
    };
    out->t_precompute = span(0, 1);
    out->t_interpolation = span(1, 4);
    out->t_far_field = span(4, 5);
    out->t_near_field = span(2, 3);
    out->t_periodic_far = span(5, 6);
    out->t_self = span(7, 8);
    out->t_total = span(0, 8);
  } else if (cfg.phase_timing) {
    float ms[6];
    for (int i = 0; i < 6; ++i) ANKH_CUDA(cudaEventElapsedTime(&ms[i], ev_[i], ev_[i + 1]));
    out->t_precompute = ms[0] * 1e-3;
    out->t_interpolation = ms[1] * 1e-3;
    out->t_far_field = ms[2] * 1e-3;
    out->t_near_field = ms[3] * 1e-3;
    out->t_periodic_far = ms[4] * 1e-3;
    out->t_self = ms[5] * 1e-3;  // finalize (self energy is fused into binning)
    float all = 0.f;
    ANKH_CUDA(cudaEventElapsedTime(&all, ev_[0], ev_[6]));
    out->t_total = all * 1e-3;  // the evaluation on the device
  }
  if (!precompute_reported) {
    out->t_precompute += precompute_seconds;
    out->t_total += precompute_seconds;  // the plan build is part of the first call
    precompute_reported = true;
  }
}

// Force buffers and tables (first forces() call): per-cell dE/dM in the
// expansion layout, near / far / output force arrays, H D^n for n = 0..3,
// the (level, offset) -> operator table and the dE/dM tiles (level, parity
// class, first class index, count <= 32) of k_m2l_local.
void Plan::force_setup() {
  if (force_init_) return;
  const std::size_t nn = std::max<std::size_t>(n, 1);
  d_loc_ = static_cast<double*>(dalloc(level_off_[depth + 1] * sizeof(double)));
  d_fnear_ = static_cast<double*>(dalloc(nn * 3 * sizeof(double)));
  d_ffar_ = static_cast<double*>(dalloc(nn * 3 * sizeof(double)));
  d_fout_ = static_cast<double*>(dalloc(nn * 3 * sizeof(double)));
  const auto hd = diff_operator(L);
  std::vector<double> hd4;
  for (const auto& m : hd) hd4.insert(hd4.end(), m.begin(), m.end());
  const std::vector<double> d3 = diff_operator_hd3(L);
  hd4.insert(hd4.end(), d3.begin(), d3.end());
  d_hd4_ = static_cast<double*>(dalloc(hd4.size() * sizeof(double)));
  ANKH_CUDA(cudaMemcpyAsync(d_hd4_, hd4.data(), hd4.size() * sizeof(double), cudaMemcpyHostToDevice, stream_));
  std::vector<int2> op_of(static_cast<std::size_t>(depth + 1) * 343, make_int2(-1, 0));
  for (int level = 1; level <= depth; ++level)
    for (int ox = -3; ox <= 3; ++ox)
      for (int oy = -3; oy <= 3; ++oy)
        for (int oz = -3; oz <= 3; ++oz) {
          auto it = op_info_.find({level, offset_key({ox, oy, oz})});
          if (it == op_info_.end()) continue;
          op_of[level * 343 + ((ox + 3) * 7 + (oy + 3)) * 7 + (oz + 3)] =
              make_int2(it->second.first_op, it->second.n_blocks);
        }
  d_op_of_ = static_cast<int2*>(dalloc(op_of.size() * sizeof(int2)));
  ANKH_CUDA(cudaMemcpyAsync(d_op_of_, op_of.data(), op_of.size() * sizeof(int2), cudaMemcpyHostToDevice, stream_));
  std::vector<int4> tiles;
  for (int level = 1; level <= depth; ++level) {
    const int per_class = 1 << (3 * (level - 1));
    for (int cls = 0; cls < 8; ++cls)
      for (int j0 = 0; j0 < per_class; j0 += 32) tiles.push_back(make_int4(level, cls, j0, std::min(32, per_class - j0)));
  }
  n_loc_tiles_ = static_cast<int>(tiles.size());
  d_loc_tiles_ = static_cast<int4*>(dalloc(std::max<std::size_t>(tiles.size(), 1) * sizeof(int4)));
  if (!tiles.empty())
    ANKH_CUDA(cudaMemcpyAsync(d_loc_tiles_, tiles.data(), tiles.size() * sizeof(int4), cudaMemcpyHostToDevice,
                              stream_));
  const double per_leaf = static_cast<double>(n) / n_leaves;
  force_cap_ = static_cast<int>(std::ceil(27.0 * per_leaf * 1.3 / 32.0)) * 32;
  force_cap_ = std::max(256, std::min(force_cap_, force_max_cap()));
  // forces without moment derivatives: the half shell (own leaf + 13 neighbours)
  force_half_cap_ = static_cast<int>(std::ceil(14.0 * per_leaf * 1.25 / 32.0)) * 32;
  force_half_cap_ = std::max(128, std::min(force_half_cap_, force_half_max_cap()));
  force_half_ = std::getenv("ANKH_FORCE_FULL_STENCIL") == nullptr;
  ANKH_CUDA(cudaStreamSynchronize(stream_));
  force_init_ = true;
}

void Plan::forces(const double* h_pos, const double* h_src, double* h_forces, ankh_report_v1* out) {
  derivatives(h_pos, h_src, h_forces, nullptr, out);
}

void Plan::derivatives(const double* h_pos, const double* h_src, double* h_forces, double* h_dsrc,
                       ankh_report_v1* out) {
  if (cfg.world > 1) throw AnkhError(ANKH_RUNTIME_ERROR, "forces: sharded plans (world > 1) are not supported");
  if (L > kMaxOrderCompiled && pending_code_ == 0)
    throw AnkhError(ANKH_RUNTIME_ERROR, "forces: order_cheb > 10 is not supported (energy only)");
  if (fft_) throw AnkhError(ANKH_RUNTIME_ERROR, "forces: not available on the fft engine (energy only)");
  if (n == 0 || pending_code_ != 0 || csr_only_) {
    enqueue_host(h_pos, h_src, nullptr);
    result(out);  // raises the deferred error, if any
    return;
  }
  // energies, records, leaf CSR, expansions of every level: the energy call's
  // own host path (large systems stream the inputs in chunks under the
  // kernels; its side streams are joined on stream_ before the final sums)
  enqueue_host(h_pos, h_src, stream_);
  force_setup();
  cudaStream_t st = stream_;
  ANKH_CUDA(cudaMemsetAsync(d_loc_, 0, level_off_[depth + 1] * sizeof(double), st));
  const bool dsrc = h_dsrc != nullptr;
  if (dsrc && !d_dnear_) {
    const std::size_t nn = std::max<std::size_t>(n, 1);
    d_dnear_ = static_cast<double*>(dalloc(nn * 10 * sizeof(double)));
    d_dfar_ = static_cast<double*>(dalloc(nn * 10 * sizeof(double)));
    d_dout_ = static_cast<double*>(dalloc(nn * 10 * sizeof(double)));
  }
  // forces alone: every neighbour pair once (Newton's third law), the
  // neighbours' sums in 13 direction slots that launch_force_out adds
  const bool half = force_half_ && !dsrc;
  const std::size_t slot_stride = std::max<std::size_t>(n, 1) * 3;
  if (half) {
    if (!d_fslot_) d_fslot_ = static_cast<double*>(dalloc(13 * slot_stride * sizeof(double)));
    ANKH_CUDA(cudaMemsetAsync(d_fslot_, 0, 13 * slot_stride * sizeof(double), st));
  }
  launch_force_near(d_part_, d_off_, d_leaf_mp_, depth, periodic ? 1 : 0, 2.0 * rb, cfg.xi, radial_,
                    half ? force_half_cap_ : force_cap_, (dsrc && !h_forces) ? nullptr : d_fnear_, st,
                    dsrc ? d_dnear_ : nullptr,
                    half ? d_fslot_ : nullptr, slot_stride);
  launch_m2l_local(d_exp_, d_loc_, d_level_off_, d_factors_, d_ops_, d_op_of_, d_loc_tiles_, n_loc_tiles_, Kp,
                   periodic ? 1 : 0, st);
  if (periodic) launch_periodic_local(d_exp_, d_to_equi_, d_gen_, L, d_loc_, st);
  for (int l = 0; l < depth; ++l) launch_l2l(d_loc_ + level_off_[l], d_loc_ + level_off_[l + 1], l, L, d_m2m_, st);
  launch_l2p(d_part_, d_off_, depth, L, rb, d_hd4_, d_loc_ + level_off_[depth], d_ffar_, st,
             dsrc ? d_dfar_ : nullptr);
  if (h_forces) {
    launch_force_out(d_fnear_, d_ffar_, d_idx2_, n, d_fout_, st, half ? d_fslot_ : nullptr, slot_stride);
    ANKH_CUDA(cudaMemcpyAsync(h_forces, d_fout_, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  if (dsrc) {
    launch_dsrc_out(d_dnear_, d_dfar_, d_part_, d_idx2_, n, cfg.xi, include_self_ ? 1 : 0, d_dout_, st);
    ANKH_CUDA(cudaMemcpyAsync(h_dsrc, d_dout_, n * 10 * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  ANKH_CUDA(cudaGetLastError());
  last_stream_ = st;
  result(out);
}

void Plan::expansions(double* out, std::size_t count) {
  ANKH_CUDA(cudaStreamSynchronize(last_stream_ ? last_stream_ : stream_));
  // reference layout: levels 0..depth, lex cell order, K doubles per cell
  // (device rows are Morton-ordered and padded to Kp)
  const std::size_t total = static_cast<std::size_t>(level_off_[depth + 1]);
  std::vector<double> padded(total);
  ANKH_CUDA(cudaMemcpy(padded.data(), d_exp_, total * sizeof(double), cudaMemcpyDeviceToHost));
  std::size_t o = 0;
  for (int l = 0; l <= depth; ++l) {
    const unsigned nl = 1u << l;
    for (unsigned c = 0; c < (1u << (3 * l)); ++c, o += K) {
      if (o + K > count) return;
      const unsigned m = morton3(c / (nl * nl), (c / nl) % nl, c % nl);
      std::memcpy(out + o, padded.data() + level_off_[l] + static_cast<std::size_t>(m) * Kp,
                  K * sizeof(double));
    }
  }
}

void Plan::enqueue_phase(int phase, const double* d_pos, const double* d_src, cudaStream_t st) {
  streamed_last_ = false;
  if (!st) st = stream_;
  last_stream_ = st;
  bound_ = false;
  if (phase == 1) evaluated_ = true;
  if (n == 0 || pending_code_ != 0) {
    if (phase == 1) enqueue(d_pos, d_src, st);
    return;
  }
  launch_all(d_pos, d_src, st, phase == 1 ? 1 : 2);
}

double* Plan::leaf_level(std::int64_t* begin, std::int64_t* end, int* row_stride) {
  if (begin) *begin = p2m_begin_;
  if (end) *end = p2m_end_;
  if (row_stride) *row_stride = Kp;
  return d_exp_ + level_off_[depth];
}

void Plan::attach_collective(Collective* c) {
  if (c && (c->world() != cfg.world || c->rank() != cfg.rank)) {
    delete c;
    throw AnkhError(ANKH_INVALID_ARGUMENT, "collective rank/world does not match the plan's shard");
  }
  coll_.reset(c);
  if (graph_src_exec_) {
    cudaGraphExecDestroy(graph_src_exec_);
    graph_src_exec_ = nullptr;
    graph_src_warm_ = 0;
  }
  if (graph_exec_) {  // recapture with the collectives in the graph
    cudaGraphExecDestroy(graph_exec_);
    graph_exec_ = nullptr;
    graph_pos_ = graph_src_ = graph_warm_pos_ = graph_warm_src_ = nullptr;
  }
}

void Plan::m2l_factors(int level, const int* offset, double* lmat, double* rmat, int max_rank,
                       int* rank) {
  const std::int64_t key = offset_key({offset[0], offset[1], offset[2]});
  auto it = op_info_.find({level, key});
  if (it == op_info_.end()) {
    *rank = 0;
    return;
  }
  const OpInfo& info = it->second;
  *rank = info.rank;
  if (info.rank > max_rank) return;
  int row = 0;
  for (int b = 0; b < info.n_blocks; ++b) {
    const M2LOp& op = h_ops_[info.first_op + b];
    std::vector<double> blk(2 * static_cast<std::size_t>(op.kp) * Kp);
    ANKH_CUDA(cudaMemcpy(blk.data(), d_factors_ + op.factor_off, blk.size() * sizeof(double),
                         cudaMemcpyDeviceToHost));
    const double* Lb = blk.data();
    const double* Rb = Lb + static_cast<std::size_t>(op.kp) * Kp;
    for (int r = 0; r < op.rank; ++r, ++row)
      for (int k = 0; k < K; ++k) {
        lmat[static_cast<std::size_t>(row) * K + k] = Lb[static_cast<std::size_t>(r) * Kp + k];
        rmat[static_cast<std::size_t>(row) * K + k] = Rb[static_cast<std::size_t>(r) * Kp + k];
      }
  }
}

void Plan::energies_to_device(double* d_out, cudaStream_t st) {
  if (!st) st = stream_;
  if (n == 0) {
    ANKH_CUDA(cudaMemsetAsync(d_out, 0, 4 * sizeof(double), st));
    return;
  }
  static_assert(offsetof(DevResult, red) == 0 && kESelf == 0 && kEPeriodic == 3,
                "DevResult energy layout");
  ANKH_CUDA(cudaMemcpyAsync(d_out, d_res_, 4 * sizeof(double), cudaMemcpyDeviceToDevice, st));
}

void Plan::leaf_csr(std::uint32_t* offsets, std::uint32_t* indices) {
  ANKH_CUDA(cudaStreamSynchronize(last_stream_ ? last_stream_ : stream_));
  ANKH_CUDA(cudaMemcpy(offsets, d_off_, (n_leaves + 1) * sizeof(unsigned), cudaMemcpyDeviceToHost));
  if (n) ANKH_CUDA(cudaMemcpy(indices, d_idx2_, n * sizeof(unsigned), cudaMemcpyDeviceToHost));
}

}  // namespace ankh_b200
