// C-ABI of libankh_b200.so (declared in include/ankh_b200.h).
#include <chrono>
#include <string>
#include <cmath>
#include <cstring>
#include <vector>
#include <list>
#include <memory>
#include <mutex>

#include "host_numerics.hpp"
#include "plan.hpp"
#include "shard.hpp"

using ankh_b200::AnkhError;
using ankh_b200::Plan;

struct ankh_plan_v1 {
  std::unique_ptr<Plan> plan;
  std::mutex mu;
};

namespace {

int set_err(char* err, std::size_t errlen, const char* msg, int code) {
  if (err && errlen) {
    std::strncpy(err, msg, errlen - 1);
    err[errlen - 1] = '\0';
  }
  return code;
}

template <class F>
int guarded(char* err, std::size_t errlen, F&& f) {
  try {
    f();
    if (err && errlen) err[0] = '\0';
    return ANKH_OK;
  } catch (const AnkhError& e) {
    return set_err(err, errlen, e.what(), e.code);
  } catch (const std::bad_alloc&) {
    return set_err(err, errlen, "host allocation failed", ANKH_RUNTIME_ERROR);
  } catch (const std::exception& e) {
    return set_err(err, errlen, e.what(), ANKH_RUNTIME_ERROR);
  }
}

// Process-wide cache of plans for the one-shot drop-in call: the geometry-only
// precompute (M2L factors, periodic spectrum, buffers) is reused whenever the
// particle count, box radius, configuration and (resolved) device repeat.
// The cache lock covers only the lookup / insert; an evaluation holds its
// plan's own mutex, so calls on different GPUs (or different systems) run
// concurrently, as the reference's reentrant call does.  Entries are shared:
// an entry evicted while a call still uses it lives until that call returns.
struct CacheEntry {
  std::size_t n;
  double rb;
  ankh_config_v1 cfg;
  int device;
  std::shared_ptr<ankh_plan_v1> h;
};
std::mutex g_cache_mu;
std::list<CacheEntry> g_cache;
constexpr std::size_t kCacheMax = 4;

bool same_cfg(const ankh_config_v1& a, const ankh_config_v1& b) {
  return a.xi == b.xi && a.p == b.p && a.order_cheb == b.order_cheb &&
         a.order_equi == b.order_equi && a.depth == b.depth && a.svd_tol == b.svd_tol &&
         a.recip_cutoff == b.recip_cutoff && a.rank == b.rank && a.world == b.world &&
         a.phase_timing == b.phase_timing;
}

int resolve_device(const ankh_config_v1& c) {
  if (c.device >= 0) return c.device;
  int d = 0;
  ANKH_CUDA(cudaGetDevice(&d));
  return d;
}

// Run f(plan) on the plan's device (the caller's current device restored
// after) under the plan's mutex.
template <class F>
void on_plan(ankh_plan_v1* h, F&& f) {
  if (!h || !h->plan) throw AnkhError(ANKH_INVALID_ARGUMENT, "null plan");
  std::lock_guard<std::mutex> lock(h->mu);
  ankh_b200::DeviceGuard dev(h->plan->device());
  f(*h->plan);
}

}  // namespace

extern "C" {

void ankh_config_default_v1(ankh_config_v1* c) {
  std::memset(c, 0, sizeof(*c));
  c->xi = 0.01;
  c->p = 15;
  c->order_cheb = 8;
  c->order_equi = 8;
  c->depth = 0;
  c->svd_tol = 1e-7;
  c->recip_cutoff = 12;
  c->threads = 0;
  c->device = -1;
  c->rank = 0;
  c->world = 1;
  c->phase_timing = 1;
}

const char* ankh_version_v1(void) { return "ankh_b200 0.1.0 (sm_100a)"; }

int ankh_fmm_energy_v1(size_t n, const double* positions, const double* sources, double box_radius,
                       const ankh_config_v1* cfg, ankh_report_v1* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!cfg || !out) throw AnkhError(ANKH_INVALID_ARGUMENT, "null config or report");
    if (n > 0 && (!positions || !sources)) throw AnkhError(ANKH_INVALID_ARGUMENT, "null input buffer");
    ankh_b200::validate_config(*cfg);
    const auto t0 = std::chrono::steady_clock::now();
    const int dev = resolve_device(*cfg);
    std::shared_ptr<ankh_plan_v1> h;
    {
      std::lock_guard<std::mutex> lock(g_cache_mu);
      for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (it->n == n && it->rb == box_radius && it->device == dev && same_cfg(it->cfg, *cfg)) {
          g_cache.splice(g_cache.begin(), g_cache, it);
          h = g_cache.front().h;
          break;
        }
      }
    }
    if (!h) {  // built outside the cache lock (plan builds on other devices proceed)
      ankh_config_v1 c = *cfg;
      c.device = dev;
      h = std::make_shared<ankh_plan_v1>();
      h->plan = std::make_unique<Plan>(n, box_radius, c);
      std::lock_guard<std::mutex> lock(g_cache_mu);
      while (g_cache.size() >= kCacheMax) g_cache.pop_back();
      g_cache.push_front({n, box_radius, *cfg, dev, h});
    }
    on_plan(h.get(), [&](Plan& plan) {
      plan.enqueue_host(positions, sources, nullptr);
      plan.result(out);
    });
    // wall_times["total"]: the whole call, as fmm.cpp:433 times it
    out->t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int ankh_fmm_forces_v1(size_t n, const double* positions, const double* sources, double box_radius,
                       const ankh_config_v1* cfg, double* forces, ankh_report_v1* out, char* err,
                       size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!cfg || !out) throw AnkhError(ANKH_INVALID_ARGUMENT, "null config or report");
    if (n > 0 && (!positions || !sources || !forces)) throw AnkhError(ANKH_INVALID_ARGUMENT, "null input buffer");
    ankh_b200::validate_config(*cfg);
    const auto t0 = std::chrono::steady_clock::now();
    const int dev = resolve_device(*cfg);
    std::shared_ptr<ankh_plan_v1> h;
    {
      std::lock_guard<std::mutex> lock(g_cache_mu);
      for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (it->n == n && it->rb == box_radius && it->device == dev && same_cfg(it->cfg, *cfg)) {
          g_cache.splice(g_cache.begin(), g_cache, it);
          h = g_cache.front().h;
          break;
        }
      }
    }
    if (!h) {
      ankh_config_v1 c = *cfg;
      c.device = dev;
      h = std::make_shared<ankh_plan_v1>();
      h->plan = std::make_unique<Plan>(n, box_radius, c);
      std::lock_guard<std::mutex> lock(g_cache_mu);
      while (g_cache.size() >= kCacheMax) g_cache.pop_back();
      g_cache.push_front({n, box_radius, *cfg, dev, h});
    }
    on_plan(h.get(), [&](Plan& plan) { plan.forces(positions, sources, forces, out); });
    out->t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int ankh_plan_forces_v1(ankh_plan_v1* plan, const double* positions, const double* sources, double* forces,
                        ankh_report_v1* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out) throw AnkhError(ANKH_INVALID_ARGUMENT, "null report");
    on_plan(plan, [&](Plan& p) {
      if (p.n > 0 && (!positions || !sources || !forces)) throw AnkhError(ANKH_INVALID_ARGUMENT, "null input buffer");
      p.forces(positions, sources, forces, out);
    });
  });
}

int ankh_plan_derivatives_v1(ankh_plan_v1* plan, const double* positions, const double* sources, double* forces,
                             double* dsrc, ankh_report_v1* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out) throw AnkhError(ANKH_INVALID_ARGUMENT, "null report");
    on_plan(plan, [&](Plan& p) {
      if (p.n > 0 && (!positions || !sources || (!forces && !dsrc)))
        throw AnkhError(ANKH_INVALID_ARGUMENT, "null input buffer");
      p.derivatives(positions, sources, forces, dsrc, out);
    });
  });
}

int ankh_plan_create_v1(size_t n, double box_radius, const ankh_config_v1* cfg, ankh_plan_v1** plan,
                        char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!cfg || !plan) throw AnkhError(ANKH_INVALID_ARGUMENT, "null config or plan pointer");
    auto h = std::make_unique<ankh_plan_v1>();
    h->plan = std::make_unique<Plan>(n, box_radius, *cfg);
    *plan = h.release();
  });
}

int ankh_plan_create_fft_v1(size_t n, double box_radius, const ankh_config_v1* cfg, ankh_plan_v1** plan,
                            char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!cfg || !plan) throw AnkhError(ANKH_INVALID_ARGUMENT, "null config or plan pointer");
    auto h = std::make_unique<ankh_plan_v1>();
    h->plan = std::make_unique<Plan>(n, box_radius, *cfg, false, /*engine=*/1);
    *plan = h.release();
  });
}

void ankh_plan_destroy_v1(ankh_plan_v1* plan) { delete plan; }  // ~Plan selects its own device

int ankh_check_call_v1(const ankh_config_v1* cfg, double box_radius, size_t n_positions,
                       size_t n_sources, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!cfg) throw AnkhError(ANKH_INVALID_ARGUMENT, "null config");
    ankh_b200::validate_config(*cfg);  // fmm.cpp:384
    // validate_system's system-level rules, in order (types.cpp:20-26)
    if (!(box_radius > 0.0) || !std::isfinite(box_radius))
      throw AnkhError(ANKH_INVALID_ARGUMENT, "fmm_energy: invalid system: box_radius must be positive and finite");
    if (n_positions != n_sources)
      throw AnkhError(ANKH_INVALID_ARGUMENT,
                      "fmm_energy: invalid system: positions and sources must have equal length");
  });
}

int ankh_plan_energy_v1(ankh_plan_v1* plan, const double* positions, const double* sources,
                        ankh_report_v1* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!plan || !out) throw AnkhError(ANKH_INVALID_ARGUMENT, "null plan or report");
    on_plan(plan, [&](Plan& p) {
      if (p.n > 0 && (!positions || !sources)) throw AnkhError(ANKH_INVALID_ARGUMENT, "null input buffer");
      p.enqueue_host(positions, sources, nullptr);
      p.result(out);
    });
  });
}

int ankh_plan_set_positions_v1(ankh_plan_v1* plan, const double* positions, char* err,
                               size_t errlen) {
  return guarded(err, errlen, [&] {
    on_plan(plan, [&](Plan& p) {
      if (p.n > 0 && !positions) throw AnkhError(ANKH_INVALID_ARGUMENT, "null input buffer");
      p.set_positions(positions, nullptr);
    });
  });
}

int ankh_plan_energy_sources_v1(ankh_plan_v1* plan, const double* sources, ankh_report_v1* out,
                                char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out) throw AnkhError(ANKH_INVALID_ARGUMENT, "null report");
    on_plan(plan, [&](Plan& p) {
      if (p.n > 0 && !sources) throw AnkhError(ANKH_INVALID_ARGUMENT, "null input buffer");
      p.enqueue_sources(sources, nullptr);
      p.result(out);
    });
  });
}

int ankh_plan_energy_device_v1(ankh_plan_v1* plan, const double* d_positions,
                               const double* d_sources, void* stream, ankh_report_v1* out,
                               char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out) throw AnkhError(ANKH_INVALID_ARGUMENT, "null report");
    on_plan(plan, [&](Plan& p) {
      p.enqueue(d_positions, d_sources, static_cast<cudaStream_t>(stream));
      p.result(out);
    });
  });
}

int ankh_plan_enqueue_v1(ankh_plan_v1* plan, const double* d_positions, const double* d_sources,
                         void* stream, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    on_plan(plan, [&](Plan& p) { p.enqueue(d_positions, d_sources, static_cast<cudaStream_t>(stream)); });
  });
}

int ankh_plan_result_v1(ankh_plan_v1* plan, ankh_report_v1* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out) throw AnkhError(ANKH_INVALID_ARGUMENT, "null report");
    on_plan(plan, [&](Plan& p) { p.result(out); });
  });
}

int ankh_plan_info_v1(const ankh_plan_v1* plan, int* depth, int* order, size_t* n_cells_leaf,
                      size_t* m2l_instances, size_t* m2l_operators, double* m2l_rank_mean,
                      size_t* device_bytes) {
  if (!plan) return ANKH_INVALID_ARGUMENT;
  const Plan& p = *plan->plan;
  if (depth) *depth = p.depth;
  if (order) *order = p.L;
  if (n_cells_leaf) *n_cells_leaf = static_cast<size_t>(p.n_leaves);
  if (m2l_instances) *m2l_instances = p.m2l_instances;
  if (m2l_operators) *m2l_operators = p.m2l_operators;
  if (m2l_rank_mean) *m2l_rank_mean = p.m2l_rank_mean;
  if (device_bytes) *device_bytes = p.device_bytes;
  return ANKH_OK;
}

int ankh_plan_expansions_v1(ankh_plan_v1* plan, double* out, size_t count, char* err,
                            size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out) throw AnkhError(ANKH_INVALID_ARGUMENT, "null buffer");
    on_plan(plan, [&](Plan& p) { p.expansions(out, count); });
  });
}

int ankh_leaf_csr_v1(size_t n, const double* positions, double box_radius, int depth,
                     uint32_t* leaf_offsets, uint32_t* indices, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (depth < 1 || depth > 8) throw AnkhError(ANKH_INVALID_ARGUMENT, "build_tree: depth must be in [1, 8]");
    ankh_config_v1 cfg;
    ankh_config_default_v1(&cfg);
    cfg.depth = depth;
    cfg.order_cheb = 2;
    cfg.order_equi = 2;
    cfg.p = 0;
    cfg.phase_timing = 0;
    Plan plan(n, box_radius, cfg, /*csr_only=*/true);
    std::vector<double> zeros(n * 10, 0.0);
    plan.enqueue_host(positions, zeros.data(), nullptr);
    plan.leaf_csr(leaf_offsets, indices);  // build_tree does not validate (octree.cpp:27-45)
  });
}

int ankh_plan_m2l_factors_v1(ankh_plan_v1* plan, int level, const int* offset, double* lmat,
                             double* rmat, int max_rank, int* rank, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!offset || !rank) throw AnkhError(ANKH_INVALID_ARGUMENT, "null argument");
    on_plan(plan, [&](Plan& p) { p.m2l_factors(level, offset, lmat, rmat, max_rank, rank); });
  });
}

int ankh_plan_energies_device_v1(ankh_plan_v1* plan, double* d_out, void* stream, char* err,
                                 size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!d_out) throw AnkhError(ANKH_INVALID_ARGUMENT, "null buffer");
    on_plan(plan, [&](Plan& p) { p.energies_to_device(d_out, static_cast<cudaStream_t>(stream)); });
  });
}

int ankh_plan_enqueue_phase_v1(ankh_plan_v1* plan, int phase, const double* d_positions,
                               const double* d_sources, void* stream, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (phase != 1 && phase != 2) throw AnkhError(ANKH_INVALID_ARGUMENT, "bad phase");
    on_plan(plan, [&](Plan& p) {
      p.enqueue_phase(phase, d_positions, d_sources, static_cast<cudaStream_t>(stream));
    });
  });
}

int ankh_plan_leaf_level_v1(ankh_plan_v1* plan, double** d_leaf_level, int64_t* row_begin,
                            int64_t* row_end, int* row_stride) {
  if (!plan || !d_leaf_level) return ANKH_INVALID_ARGUMENT;
  *d_leaf_level = plan->plan->leaf_level(row_begin, row_end, row_stride);
  return ANKH_OK;
}

int ankh_device_copy_v1(void* dst, const void* src, size_t bytes, void* stream, char* err,
                        size_t errlen) {
  return guarded(err, errlen, [&] {
    ANKH_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice,
                              static_cast<cudaStream_t>(stream)));
  });
}

int ankh_nccl_unique_id_v1(unsigned char* id128, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!id128) throw AnkhError(ANKH_INVALID_ARGUMENT, "null id buffer");
    ankh_b200::nccl_unique_id(id128);
  });
}

int ankh_plan_attach_nccl_v1(ankh_plan_v1* plan, const unsigned char* id128, char* err,
                             size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!id128) throw AnkhError(ANKH_INVALID_ARGUMENT, "null id");
    on_plan(plan, [&](Plan& p) {
      p.attach_collective(ankh_b200::make_nccl_collective(id128, p.cfg.rank, p.cfg.world));
    });
  });
}

int ankh_nccl_selftest_v1(char* err, size_t errlen) {
  return guarded(err, errlen, [&] { ankh_b200::nccl_selftest(); });
}

int ankh_plan_attach_loopback_v1(ankh_plan_v1* plan, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    on_plan(plan, [&](Plan& p) {
      p.attach_collective(ankh_b200::make_loopback_collective(p.cfg.rank, p.cfg.world));
    });
  });
}

int ankh_plan_attach_push_group_v1(ankh_plan_v1** plans, int world, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!plans || world < 1) throw AnkhError(ANKH_INVALID_ARGUMENT, "bad plan group");
    std::vector<double*> bases(world);
    for (int r = 0; r < world; ++r) {
      if (!plans[r] || plans[r]->plan->cfg.world != world || plans[r]->plan->cfg.rank != r)
        throw AnkhError(ANKH_INVALID_ARGUMENT, "plan group must hold ranks 0..world-1 of one sharding");
      bases[r] = plans[r]->plan->expansions_base();
    }
    std::vector<std::vector<double*>> halo_recv(world, std::vector<double*>(world, nullptr));
    for (int q = 0; q < world; ++q)
      for (int r = 0; r < world; ++r) halo_recv[q][r] = plans[q]->plan->halo_recv_from(r);
    for (int r = 0; r < world; ++r)
      on_plan(plans[r], [&](Plan& p) {
        p.attach_collective(ankh_b200::make_push_collective(r, world, bases, halo_recv));
      });
  });
}

int ankh_shard_leaf_range_v1(int depth, int rank, int world, int64_t* begin, int64_t* end) {
  if (depth < 1 || depth > 8 || world < 1 || rank < 0 || rank >= world || !begin || !end)
    return ANKH_INVALID_ARGUMENT;
  ankh_b200::shard_leaf_range(depth, rank, world, begin, end);
  return ANKH_OK;
}

int ankh_shard_src_slice_v1(size_t n, int rank, int world, size_t* i0, size_t* i1) {
  if (world < 1 || rank < 0 || rank >= world || !i0 || !i1) return ANKH_INVALID_ARGUMENT;
  ankh_b200::shard_src_slice(n, rank, world, i0, i1);
  return ANKH_OK;
}

int ankh_shard_exchange_level_v1(int depth, int world) {
  if (depth < 1 || depth > 8 || world < 1) return -1;
  return ankh_b200::shard_exchange_level(depth, world);
}

int ankh_shard_halo_cells_v1(int level, int depth, int periodic, int src, int dst, int world,
                             uint32_t* morton, size_t capacity, size_t* count) {
  if (level < 0 || level > depth || depth < 1 || depth > 8 || world < 1 || src < 0 || src >= world ||
      dst < 0 || dst >= world || !count)
    return ANKH_INVALID_ARGUMENT;
  try {
    const auto cells = ankh_b200::shard_halo_cells(level, depth, periodic != 0, src, dst, world);
    *count = cells.size();
    if (morton)
      for (size_t k = 0; k < cells.size() && k < capacity; ++k) morton[k] = cells[k];
    return ANKH_OK;
  } catch (...) {
    return ANKH_RUNTIME_ERROR;
  }
}

int ankh_shard_exchange_bytes_v1(int depth, int periodic, int order, int rank, int world, int halo,
                                 size_t* recv_bytes, size_t* send_bytes) {
  if (depth < 1 || depth > 8 || order < 2 || world < 1 || rank < 0 || rank >= world || !recv_bytes ||
      !send_bytes)
    return ANKH_INVALID_ARGUMENT;
  try {
    ankh_b200::shard_exchange_bytes(depth, periodic != 0, ankh_b200::exp_stride(order * order * order), rank,
                                    world, halo != 0, recv_bytes, send_bytes);
    return ANKH_OK;
  } catch (...) {
    return ANKH_RUNTIME_ERROR;
  }
}

int ankh_shard_cell_owner_v1(int level, uint32_t cell, int depth, int world) {
  if (level < 0 || level > depth || depth > 8 || world < 1) return -1;
  return ankh_b200::shard_cell_owner(level, cell, depth, world);
}

int ankh_shard_m2l_instances_v1(int depth, int periodic, int rank, int world, uint32_t* level,
                                uint32_t* t, uint32_t* s, int32_t* offset, size_t capacity,
                                size_t* count) {
  if (depth < 1 || depth > 8 || world < 1 || rank >= world || !count) return ANKH_INVALID_ARGUMENT;
  try {
    const auto groups = ankh_b200::enumerate_m2l(depth, periodic != 0, rank, world, 0);
    size_t c = 0;
    for (const auto& g : groups) {
      for (size_t k = 0; k < g.t.size(); ++k, ++c) {
        if (c >= capacity) continue;
        if (level) level[c] = static_cast<uint32_t>(g.level);
        if (t) t[c] = g.t[k];
        if (s) s[c] = g.s[k];
        if (offset)
          for (int a = 0; a < 3; ++a) offset[3 * c + a] = g.offset[a];
      }
    }
    *count = c;
    return ANKH_OK;
  } catch (...) {
    return ANKH_RUNTIME_ERROR;
  }
}

int ankh_radial_fit_v1(double s_max, int* nterms, double* s_lim, double* p, double* g,
                       double* max_err) {
  try {
    const ankh_b200::RadialFit f = ankh_b200::fit_radial(s_max);
    if (nterms) *nterms = f.nterms;
    if (s_lim) *s_lim = f.s_lim;
    if (max_err) *max_err = f.max_err;
    if (p) std::memcpy(p, f.p, sizeof f.p);
    if (g) std::memcpy(g, f.g, sizeof f.g);
    return ANKH_OK;
  } catch (...) {
    return ANKH_RUNTIME_ERROR;
  }
}

double ankh_probe_dmma_tflops_v1(int shape, int iters) {
  try {
    return ankh_b200::probe_dmma_tflops(shape, iters > 0 ? iters : 4096);
  } catch (...) {
    return 0.0;
  }
}

double ankh_probe_fp64_mix_ms_v1(int mode, int iters_dfma, int iters_dmma) {
  try {
    return ankh_b200::probe_fp64_mix_ms(mode, iters_dfma, iters_dmma);
  } catch (...) {
    return 0.0;
  }
}

double ankh_probe_fp64_tflops_v1(int iters) {
  try {
    return ankh_b200::probe_fp64_tflops(iters > 0 ? iters : 4096);
  } catch (...) {
    return 0.0;
  }
}

}  // extern "C"
