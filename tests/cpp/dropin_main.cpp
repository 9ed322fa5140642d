// Drop-in check: a reference-style caller of ankh::fmm_energy compiled against
// include/ankh_b200.hpp and linked with libankh_b200.so.  Reads a SPEC
// particle file: '#' comments, "N r_B", then N rows of
// x y z q mux muy muz Txx Txy Txz Tyy Tyz Tzz.
//   dropin_main <file> <order_cheb> <depth> <p>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#ifdef ANKH_B200_USE_REFERENCE_TYPES
#include "ankh/types.hpp"  // the reference's own value types (types.hpp:13-135)
#endif
#include "ankh_b200.hpp"

static ankh::EnergyReport call(const ankh::ParticleSystem& s, const ankh::EwaldConfig& c) {
#ifdef ANKH_B200_USE_REFERENCE_TYPES
  return ankh::b200::fmm_energy(s, c, 1);
#else
  return ankh::fmm_energy(s, c, 1);
#endif
}

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s file order depth p\n", argv[0]);
    return 2;
  }
  std::ifstream in(argv[1]);
  std::string line;
  ankh::ParticleSystem sys;
  std::size_t n = 0;
  bool header = false;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ss(line);
    if (!header) {
      ss >> n >> sys.box_radius;
      header = true;
      continue;
    }
    ankh::Vec3 p;
    ankh::MultipoleSource s;
    ss >> p.x >> p.y >> p.z >> s.q >> s.mu.x >> s.mu.y >> s.mu.z;
    for (double& t : s.theta.m) ss >> t;
    sys.positions.push_back(p);
    sys.sources.push_back(s);
  }
  if (sys.positions.size() != n) return 3;
  ankh::EwaldConfig cfg;
  cfg.order_cheb = std::atoi(argv[2]);
  cfg.order_equi = cfg.order_cheb;
  cfg.depth = std::atoi(argv[3]);
  cfg.p = std::atoi(argv[4]);
  const ankh::EnergyReport r = call(sys, cfg);
  std::printf("%.17g %.17g %.17g %.17g %.17g\n", r.e_total, r.e_self, r.e_near, r.e_far,
              r.e_periodic_far);
  {
    // repeated evaluation with bound positions (ankh::b200::Plan), moments halved:
    // the energy is quadratic in the moments, so e_total scales by exactly 1/4
    // up to the self-energy and rounding -- printed for the Python side to check
    ankh::b200::Plan<ankh::EwaldConfig, ankh::EnergyReport> plan(n, sys.box_radius, cfg);
    plan.set_positions(sys.positions);
    const ankh::EnergyReport a = plan.energy_sources(sys.sources);
    std::vector<ankh::MultipoleSource> half = sys.sources;
    for (auto& s : half) {
      s.q *= 0.5;
      s.mu.x *= 0.5;
      s.mu.y *= 0.5;
      s.mu.z *= 0.5;
      for (double& t : s.theta.m) t *= 0.5;
    }
    const ankh::EnergyReport b = plan.energy_sources(half);
    std::printf("plan %.17g %.17g\n", a.e_total, b.e_total);
    // forces into the caller's own Vec3 vector
    std::vector<ankh::Vec3> f;
    const ankh::EnergyReport c = plan.forces(sys.positions, sys.sources, f);
    std::printf("forces %.17g %.17g %.17g %.17g\n", c.e_total, f[0].x, f[0].y, f[n - 1].z);
    // the moment gradient (potential, -field, field gradient) into the
    // caller's own MultipoleSource vector (same 10-double layout)
    std::vector<ankh::MultipoleSource> g;
    const ankh::EnergyReport d = plan.moment_gradient(sys.positions, sys.sources, g);
    std::printf("mgrad %.17g %.17g %.17g %.17g\n", d.e_total, g[0].q, g[0].mu.x, g[n - 1].theta.m[1]);
  }
  try {
    ankh::EwaldConfig bad = cfg;
    bad.xi = -1.0;
    call(sys, bad);
    return 4;
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what());
  }
  return 0;
}
