// C++ drop-in for the reference's energy call, header-only over the C-ABI of
// libankh_b200.so (include/ankh_b200.h).
//
// A caller of the reference (proj/core/include/ankh/fmm.hpp) replaces
//     #include "ankh/fmm.hpp"      and links libankh_core
// with
//     #include "ankh_b200.hpp"     and links libankh_b200.so
// and keeps calling ankh::fmm_energy(system, config, threads).  The types
// below are layout-compatible re-declarations of the reference's value types
// (types.hpp:13-135); the exceptions are the same standard types with the
// same messages (types.cpp:65-79, fmm.cpp:385-388, octree.cpp:28,
// chebyshev.cpp:86, kernel.cpp:161).
//
// If the reference's own ankh/types.hpp is already included (the caller keeps
// it for its own code), define ANKH_B200_USE_REFERENCE_TYPES before including
// this header and only ankh::b200::fmm_energy is declared, taking the
// reference's types.
#pragma once

#include <array>
#include <cmath>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "ankh_b200.h"

namespace ankh {

#ifndef ANKH_B200_USE_REFERENCE_TYPES
struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  double& operator[](int i) { return (&x)[i]; }
  double operator[](int i) const { return (&x)[i]; }
};

struct SymMat3 {
  std::array<double, 6> m{0, 0, 0, 0, 0, 0};  // xx, xy, xz, yy, yz, zz
};

struct MultipoleSource {
  double q = 0.0;
  Vec3 mu{};
  SymMat3 theta{};
};

struct ParticleSystem {
  std::vector<Vec3> positions;
  std::vector<MultipoleSource> sources;
  double box_radius = 1.0;
  std::size_t size() const { return positions.size(); }
};

struct EwaldConfig {
  double xi = 0.01;
  int p = 15;
  int order_cheb = 8;
  int order_equi = 8;
  int depth = 0;
  double svd_tol = 1e-7;
  int recip_cutoff = 12;
};

struct EnergyReport {
  double e_total = 0.0;
  double e_self = 0.0;
  double e_near = 0.0;
  double e_far = 0.0;
  double e_periodic_far = 0.0;
  double e_reciprocal = 0.0;
  std::map<std::string, double> wall_times;
  double component_sum() const { return e_self + e_near + e_far + e_periodic_far + e_reciprocal; }
};
#endif

namespace b200 {

inline void rethrow(int code, const char* err) {
  switch (code) {
    case ANKH_OK:
      return;
    case ANKH_INVALID_ARGUMENT:
      throw std::invalid_argument(err);
    case ANKH_DOMAIN_ERROR:
      throw std::domain_error(err);
    default:
      throw std::runtime_error(err);
  }
}

template <class Config>
ankh_config_v1 to_c(const Config& config, int threads) {
  ankh_config_v1 c;
  ankh_config_default_v1(&c);
  c.xi = config.xi;
  c.p = config.p;
  c.order_cheb = config.order_cheb;
  c.order_equi = config.order_equi;
  c.depth = config.depth;
  c.svd_tol = config.svd_tol;
  c.recip_cutoff = config.recip_cutoff;
  c.threads = threads;
  return c;
}

template <class Report>
Report from_c(const ankh_report_v1& r);

template <class System, class Config, class Report = EnergyReport>
Report fmm_energy(const System& system, const Config& config, int threads = 1) {
  static_assert(sizeof(system.positions[0]) == 3 * sizeof(double), "Vec3 layout");
  static_assert(sizeof(system.sources[0]) == 10 * sizeof(double), "MultipoleSource layout");
  const ankh_config_v1 c = to_c(config, threads);
  ankh_report_v1 r;
  char err[512];
  // validate_config, box radius, size mismatch: the reference's order (fmm.cpp:384-388)
  rethrow(ankh_check_call_v1(&c, system.box_radius, system.positions.size(), system.sources.size(),
                             err, sizeof(err)),
          err);
  const int code = ankh_fmm_energy_v1(
      system.positions.size(), reinterpret_cast<const double*>(system.positions.data()),
      reinterpret_cast<const double*>(system.sources.data()), system.box_radius, &c, &r, err,
      sizeof(err));
  rethrow(code, err);
  return from_c<Report>(r);
}

template <class Report>
Report from_c(const ankh_report_v1& r) {
  Report out;
  out.e_total = r.e_total;
  out.e_self = r.e_self;
  out.e_near = r.e_near;
  out.e_far = r.e_far;
  out.e_periodic_far = r.e_periodic_far;
  out.e_reciprocal = r.e_reciprocal;
  out.wall_times["precompute"] = r.t_precompute;
  out.wall_times["interpolation"] = r.t_interpolation;
  out.wall_times["far_field"] = r.t_far_field;
  out.wall_times["near_field"] = r.t_near_field;
  out.wall_times["periodic_far"] = r.t_periodic_far;
  out.wall_times["self"] = r.t_self;
  out.wall_times["total"] = r.t_total;
  return out;
}

/// Repeated evaluation (the plan API of include/ankh_b200.h): geometry-only
/// precompute once per (n, box radius, config); positions may be bound once
/// when only the moments change (ankh_plan_set_positions_v1).
template <class Config, class Report = EnergyReport>
class Plan {
 public:
  Plan(std::size_t n, double box_radius, const Config& config, int threads = 0) : n_(n) {
    const ankh_config_v1 c = to_c(config, threads);
    char err[512];
    rethrow(ankh_plan_create_v1(n, box_radius, &c, &plan_, err, sizeof(err)), err);
  }
  ~Plan() { ankh_plan_destroy_v1(plan_); }
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;

  /// Full evaluation of host positions (n Vec3) and moments (n MultipoleSource).
  template <class P, class S>
  Report energy(const std::vector<P>& positions, const std::vector<S>& sources) {
    check(positions.size(), sources.size());
    ankh_report_v1 r;
    char err[512];
    rethrow(ankh_plan_energy_v1(plan_, reinterpret_cast<const double*>(positions.data()),
                                reinterpret_cast<const double*>(sources.data()), &r, err,
                                sizeof(err)),
            err);
    return from_c<Report>(r);
  }
  /// Energy plus forces F = -dE/dx (moments fixed): `forces`
  /// receives n x 3 doubles (any 24-byte Vec3-like element type).
  template <class P, class S, class F>
  Report forces(const std::vector<P>& positions, const std::vector<S>& sources, std::vector<F>& forces) {
    static_assert(sizeof(F) == 3 * sizeof(double), "force element layout");
    check(positions.size(), sources.size());
    forces.resize(n_);
    ankh_report_v1 r;
    char err[512];
    rethrow(ankh_plan_forces_v1(plan_, reinterpret_cast<const double*>(positions.data()),
                                reinterpret_cast<const double*>(sources.data()),
                                reinterpret_cast<double*>(forces.data()), &r, err, sizeof(err)),
            err);
    return from_c<Report>(r);
  }
  /// Energy plus the moment gradient dE/ds (n x 10 doubles in the
  /// MultipoleSource layout: potential, minus the field, field gradient per
  /// stored component) -- the induced-dipole machinery; any 80-byte element.
  template <class P, class S, class G>
  Report moment_gradient(const std::vector<P>& positions, const std::vector<S>& sources, std::vector<G>& dsrc) {
    static_assert(sizeof(G) == 10 * sizeof(double), "moment-gradient element layout");
    check(positions.size(), sources.size());
    dsrc.resize(n_);
    ankh_report_v1 r;
    char err[512];
    rethrow(ankh_plan_derivatives_v1(plan_, reinterpret_cast<const double*>(positions.data()),
                                     reinterpret_cast<const double*>(sources.data()), nullptr,
                                     reinterpret_cast<double*>(dsrc.data()), &r, err, sizeof(err)),
            err);
    return from_c<Report>(r);
  }
  /// Bind positions once (copied, validated, binned) ...
  template <class P>
  void set_positions(const std::vector<P>& positions) {
    check(positions.size(), n_);
    char err[512];
    rethrow(ankh_plan_set_positions_v1(plan_, reinterpret_cast<const double*>(positions.data()),
                                       err, sizeof(err)),
            err);
  }
  /// ... then evaluate new moments at the bound positions.
  template <class S>
  Report energy_sources(const std::vector<S>& sources) {
    check(n_, sources.size());
    ankh_report_v1 r;
    char err[512];
    rethrow(ankh_plan_energy_sources_v1(plan_, reinterpret_cast<const double*>(sources.data()),
                                        &r, err, sizeof(err)),
            err);
    return from_c<Report>(r);
  }

 private:
  void check(std::size_t a, std::size_t b) const {
    if (a != b || a != n_)
      throw std::invalid_argument(
          "fmm_energy: invalid system: positions and sources must have equal length");
  }
  std::size_t n_;
  ankh_plan_v1* plan_ = nullptr;
};

}  // namespace b200

#ifndef ANKH_B200_USE_REFERENCE_TYPES
/// Drop-in for ankh::fmm_energy (fmm.hpp:98-99).
inline EnergyReport fmm_energy(const ParticleSystem& system, const EwaldConfig& config,
                               int threads = 1) {
  return b200::fmm_energy<ParticleSystem, EwaldConfig, EnergyReport>(system, config, threads);
}
#endif

}  // namespace ankh
