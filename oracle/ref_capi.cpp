// TEST INFRASTRUCTURE ONLY (oracle).  Never linked into the product.
//
// A C-ABI around the UNMODIFIED reference sources (/root/reference/proj/core),
// compiled by oracle/Makefile against the shim headers in oracle/shim into
// oracle/_ref/libankh_ref.so.  Used by tests/ (parity checker), by
// __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
// --impl reference legs.  Everything here forwards to the reference's own
// functions; no algorithm is restated in this file.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "ankh/chebyshev.hpp"
#include "ankh/fmm.hpp"
#include "ankh/kernel.hpp"
#include "ankh/octree.hpp"
#include "ankh/types.hpp"

namespace {

ankh::ParticleSystem make_system(std::size_t n, const double* pos, const double* src, double r) {
  static_assert(sizeof(ankh::Vec3) == 3 * sizeof(double), "Vec3 layout");
  static_assert(sizeof(ankh::MultipoleSource) == 10 * sizeof(double), "MultipoleSource layout");
  ankh::ParticleSystem s;
  s.box_radius = r;
  s.positions.resize(n);
  s.sources.resize(n);
  if (n) {
    std::memcpy(s.positions.data(), pos, n * 3 * sizeof(double));
    if (src) std::memcpy(s.sources.data(), src, n * 10 * sizeof(double));
  }
  return s;
}

ankh::EwaldConfig make_config(const double* dcfg, const int* icfg) {
  // dcfg = {xi, svd_tol}; icfg = {p, order_cheb, order_equi, depth, recip_cutoff}
  ankh::EwaldConfig c;
  c.xi = dcfg[0];
  c.svd_tol = dcfg[1];
  c.p = icfg[0];
  c.order_cheb = icfg[1];
  c.order_equi = icfg[2];
  c.depth = icfg[3];
  c.recip_cutoff = icfg[4];
  return c;
}

int fail(const char* what, char* err, std::size_t errlen, int code) {
  if (err && errlen) {
    std::strncpy(err, what, errlen - 1);
    err[errlen - 1] = '\0';
  }
  return code;
}

template <class F>
int guarded(char* err, std::size_t errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e.what(), err, errlen, 1);
  } catch (const std::domain_error& e) {
    return fail(e.what(), err, errlen, 2);
  } catch (const std::runtime_error& e) {
    return fail(e.what(), err, errlen, 3);
  } catch (const std::exception& e) {
    return fail(e.what(), err, errlen, 5);
  }
}

}  // namespace

extern "C" {

// out[0..5] = e_total, e_self, e_near, e_far, e_periodic_far, e_reciprocal
// out[6..12] = wall_times precompute, interpolation, far_field, near_field,
//              periodic_far, self, total
int ref_fmm_energy(std::size_t n, const double* pos, const double* src, double box_radius,
                   const double* dcfg, const int* icfg, int threads, double* out, char* err,
                   std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ankh::ParticleSystem sys = make_system(n, pos, src, box_radius);
    const ankh::EwaldConfig cfg = make_config(dcfg, icfg);
    const ankh::EnergyReport r = ankh::fmm_energy(sys, cfg, threads);
    out[0] = r.e_total;
    out[1] = r.e_self;
    out[2] = r.e_near;
    out[3] = r.e_far;
    out[4] = r.e_periodic_far;
    out[5] = r.e_reciprocal;
    const char* keys[7] = {"precompute", "interpolation", "far_field", "near_field",
                           "periodic_far", "self", "total"};
    for (int i = 0; i < 7; ++i) {
      auto it = r.wall_times.find(keys[i]);
      out[6 + i] = it == r.wall_times.end() ? 0.0 : it->second;
    }
  });
}

// fmm_energy on a system whose position and source arrays differ in length
// (the reference's size-mismatch rule, types.cpp:23-26): only the exception
// is of interest; returns the code / message of the call.
int ref_fmm_energy_sized(std::size_t n_pos, std::size_t n_src, const double* pos, const double* src,
                         double box_radius, const double* dcfg, const int* icfg, char* err,
                         std::size_t errlen) {
  return guarded(err, errlen, [&] {
    ankh::ParticleSystem s;
    s.box_radius = box_radius;
    s.positions.resize(n_pos);
    s.sources.resize(n_src);
    if (n_pos) std::memcpy(s.positions.data(), pos, n_pos * 3 * sizeof(double));
    if (n_src) std::memcpy(s.sources.data(), src, n_src * 10 * sizeof(double));
    ankh::fmm_energy(s, make_config(dcfg, icfg), 1);
  });
}

// Leaf CSR of build_tree (octree.cpp:27-45): offsets[8^depth + 1], indices[n].
int ref_leaf_csr(std::size_t n, const double* pos, double box_radius, int depth,
                 std::uint32_t* offsets, std::uint32_t* indices, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ankh::ParticleSystem sys = make_system(n, pos, nullptr, box_radius);
    const ankh::PerfectOctree tree = ankh::build_tree(sys, depth);
    std::uint32_t acc = 0;
    for (std::size_t leaf = 0; leaf < tree.leaf_buckets.size(); ++leaf) {
      offsets[leaf] = acc;
      for (std::uint32_t u : tree.leaf_buckets[leaf]) indices[acc++] = u;
    }
    offsets[tree.leaf_buckets.size()] = acc;
  });
}

// Per-level expansions after P2M + M2M (fmm.cpp:181-236), levels 0..depth
// concatenated in level order, each level in lex cell order, K per cell.
int ref_expansions(std::size_t n, const double* pos, const double* src, double box_radius,
                   int depth, int order, double* out, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ankh::ParticleSystem sys = make_system(n, pos, src, box_radius);
    const ankh::PerfectOctree tree = ankh::build_tree(sys, depth);
    const ankh::DiffOperator op(order);
    const ankh::LevelExpansions ex =
        ankh::upward_pass(tree, ankh::leaf_expansions(sys, tree, op, 1), order);
    std::size_t o = 0;
    for (int level = 0; level <= depth; ++level)
      for (const auto& cell : ex[static_cast<std::size_t>(level)])
        for (double v : cell) out[o++] = v;
  });
}

// Far-field pieces: e_far (fmm.cpp:238-276), and the summed rank statistics of
// the M2L cache (fmm.cpp:141-179) for diagnostics.
int ref_far_field(std::size_t n, const double* pos, const double* src, double box_radius,
                  int depth, int order, double xi, double svd_tol, int periodic, int threads,
                  double* out, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ankh::ParticleSystem sys = make_system(n, pos, src, box_radius);
    const ankh::PerfectOctree tree = ankh::build_tree(sys, depth);
    const ankh::InteractionLists lists = ankh::interaction_lists(tree, periodic != 0);
    const ankh::DiffOperator op(order);
    const ankh::Grid1D grid = ankh::Grid1D::chebyshev(order);
    const ankh::M2LCache cache = ankh::build_m2l_cache(tree, lists, grid, xi, svd_tol, threads);
    const ankh::LevelExpansions ex =
        ankh::upward_pass(tree, ankh::leaf_expansions(sys, tree, op, threads), order);
    out[0] = ankh::far_field_energy(tree, lists, ex, cache, threads);
    out[1] = ankh::far_field_energy(tree, lists, ex, cache, threads, /*mutual=*/false);
    double ranks = 0.0, count = 0.0;
    for (const auto& lvl : cache.ops)
      for (const auto& kv : lvl) {
        ranks += kv.second.rank();
        count += 1.0;
      }
    out[2] = ranks;
    out[3] = count;
  });
}

// M2L factors for one (level-radius, offset): lmat and rmat (k x K, row-major
// as in Eigen's col-major storage transposed) -> returns rank in *rank_out.
int ref_m2l_factors(int order, double cell_radius, const int* offset, double xi, double svd_tol,
                    std::uint64_t seed, double* lmat, double* rmat, int max_rank, int* rank_out,
                    char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ankh::Grid1D grid = ankh::Grid1D::chebyshev(order);
    const Eigen::MatrixXd c = ankh::m2l_dense(grid, cell_radius, {offset[0], offset[1], offset[2]}, xi);
    const ankh::M2LOperator op = ankh::compress_m2l(c, svd_tol, seed);
    const int k = op.rank();
    *rank_out = k;
    if (k > max_rank) return;
    const Eigen::Index kk = c.rows();
    for (int i = 0; i < k; ++i)
      for (Eigen::Index j = 0; j < kk; ++j) {
        lmat[i * kk + j] = op.lmat(i, j);
        rmat[i * kk + j] = op.rmat(i, j);
      }
  });
}

// Dense M2L block (fmm.cpp:60-96), row-major K x K.
int ref_m2l_dense(int order, double cell_radius, const int* offset, double xi, double* out,
                  char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ankh::Grid1D grid = ankh::Grid1D::chebyshev(order);
    const Eigen::MatrixXd c = ankh::m2l_dense(grid, cell_radius, {offset[0], offset[1], offset[2]}, xi);
    for (Eigen::Index i = 0; i < c.rows(); ++i)
      for (Eigen::Index j = 0; j < c.cols(); ++j) out[i * c.cols() + j] = c(i, j);
  });
}

// Interaction-list sizes (octree.cpp:47-112): lambda sizes for every cell at
// `level` and neighbour counts for every leaf.
int ref_list_sizes(int depth, int periodic, int level, std::uint32_t* lambda_sizes,
                   std::uint32_t* neighbor_sizes, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    ankh::PerfectOctree tree;
    tree.depth = depth;
    tree.box_radius = 1.0;
    tree.leaf_buckets.assign(tree.cell_count(depth), {});
    const ankh::InteractionLists lists = ankh::interaction_lists(tree, periodic != 0);
    for (std::size_t t = 0; t < tree.cell_count(level); ++t)
      lambda_sizes[t] = static_cast<std::uint32_t>(lists.lambda[static_cast<std::size_t>(level)][t].size());
    for (std::size_t t = 0; t < tree.cell_count(depth); ++t)
      neighbor_sizes[t] = static_cast<std::uint32_t>(lists.leaf_neighbors[t].size());
  });
}

double ref_erfc_screen(double z) { return ankh::erfc_screen(z); }

int ref_pair_interaction(const double* xa, const double* sa, const double* xb, const double* sb,
                         double xi, double* out, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    ankh::Vec3 a{xa[0], xa[1], xa[2]}, b{xb[0], xb[1], xb[2]};
    ankh::MultipoleSource s1, s2;
    std::memcpy(&s1, sa, sizeof(s1));
    std::memcpy(&s2, sb, sizeof(s2));
    *out = ankh::pair_interaction(a, s1, b, s2, xi);
  });
}

double ref_self_energy(std::size_t n, const double* src, double xi) {
  ankh::ParticleSystem s;
  s.sources.resize(n);
  if (n) std::memcpy(s.sources.data(), src, n * 10 * sizeof(double));
  return ankh::self_energy(s, xi);
}

int ref_default_depth(std::size_t n) { return ankh::default_depth(n); }

// Periodic far-image energy of a given root Chebyshev expansion
// (fmm.cpp:333-381, 421-427).
int ref_periodic_far(double box_radius, int order, double xi, int p, const double* root_cheb,
                     int threads, double* out, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ankh::PeriodicOperator op = ankh::build_periodic_operator(box_radius, order, xi, p, threads);
    const ankh::Grid1D grid = ankh::Grid1D::chebyshev(order);
    const ankh::Grid1D equi = ankh::Grid1D::equispaced(order);
    const Eigen::MatrixXd to_equi = ankh::transfer_1d(equi, grid.nodes);
    const std::size_t k = static_cast<std::size_t>(order) * order * order;
    const std::vector<double> root(root_cheb, root_cheb + k);
    const std::vector<double> root_equi = ankh::tensor3_apply(to_equi, to_equi, to_equi, root);
    *out = 0.5 * ankh::periodic_far_energy(op, root_equi);
  });
}

}  // extern "C"
