// ref_adapter_driver.cpp -- TEST INFRASTRUCTURE ONLY (built by oracle/build_ref.py into
// oracle/_ref/, run by tests/test_ref_adapter_gpu.py on the GPU box).
//
// A caller of the REFERENCE library (its unmodified headers under /root/reference/proj/include,
// compiled against oracle/eigen_shim) switches to the device through include/tpmg_b200_ref.hpp:
// it builds the reference's own MultigridHierarchy<double> exactly as the reference's fixture
// does (tests/fixtures.hpp:18-62: icosahedral hierarchy, balanced-flow factorised profiles with
// vertical advection, geometric grading, block-Jacobi relax = 0.9, nu = 2 + 2), hands it to
// tpmg_b200::ref::DeviceMultigrid, and calls the device versions of v_cycle, apply_operator,
// smooth, restrict_field[_transpose], prolongate_field and measure_cycle_rate with the
// reference's own Field<double> objects.  Every result is compared with the reference's own
// CPU call on the same inputs: bitwise for the element-wise operations, 1e-12 for the
// norm-based cycle rate.  Prints one line per check and exits non-zero on any mismatch.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "tpmg/multigrid.hpp"
#include "tpmg_b200_ref.hpp"

using namespace tpmg;

static int g_fail = 0;

static Field<double> random_field(int level, Index nr, Index nc, unsigned seed) {
  Field<double> u(level, nr, nc);
  std::mt19937 rng(seed);
  std::normal_distribution<double> dist;
  for (Index i = 0; i < u.values.size(); ++i) u.values.data()[i] = dist(rng);
  return u;
}

static void same(const char* what, const Field<double>& a, const Field<double>& b) {
  bool ok = a.level == b.level && a.values.rows() == b.values.rows() &&
            a.values.cols() == b.values.cols();
  Index bad = 0;
  double worst = 0.0;
  if (ok)
    for (Index i = 0; i < a.values.size(); ++i) {
      const double x = a.values.data()[i], y = b.values.data()[i];
      if (!(x == y) || std::signbit(x) != std::signbit(y)) {
        ++bad;
        worst = std::fmax(worst, std::fabs(x - y));
      }
    }
  ok = ok && bad == 0;
  std::printf("%-40s %s (%lld values%s)\n", what, ok ? "bitwise" : "MISMATCH",
              (long long)a.values.size(),
              ok ? "" : (", " + std::to_string(bad) + " differ, max " + std::to_string(worst)).c_str());
  if (!ok) ++g_fail;
}

int main() {
  const int L = 2;
  const Index nr = 8;
  const PhysicalConstants<double> consts{};
  const auto hier = build_icosahedral_hierarchy<double>(L);
  const auto vert = build_vertical_grid<double>(nr, 80.0 / 6371.229, VerticalGrading::geometric, 1.2);
  const BalancedFlow<double> flow(0.022, consts);
  const auto op = OperatorParameters<double>::courant_default(hier.finest(), consts);
  const auto fac = factorize_balanced_flow(hier.finest(), vert, flow, op);
  SmootherConfig<double> sm;
  sm.kind = SmootherKind::block_jacobi;
  sm.relax = 0.9;

  tpmg_b200::Context ctx(0);
  const Index ncL = hier.finest().n_cells();
  const auto u = random_field(L, nr, ncL, 1);
  const auto f = random_field(L, nr, ncL, 2);
  const auto u0 = random_field(L, nr, ncL, 3);

  const std::pair<ProlongationKind, RestrictionKind> pairs[3] = {
      {ProlongationKind::linear, RestrictionKind::summation},
      {ProlongationKind::linear, RestrictionKind::transpose},
      {ProlongationKind::injection, RestrictionKind::summation}};
  for (int c = 0; c < 3; ++c) {
    TransferConfig tr;
    tr.prolongation = pairs[c].first;
    tr.restriction = pairs[c].second;
    const auto m = build_hierarchy_coefficients(fac, hier, vert, op.omega, sm, tr, 2, 2, 0);
    tpmg_b200::ref::DeviceMultigrid dm(ctx, m);  // the reference's own hierarchy object
    const std::string s = " [pair " + std::to_string(c) + "]";
    if (c == 0) {
      // apply_operator, discretization.hpp:262-278
      Field<double> y_ref, y_dev;
      apply_operator(m.coeff(L), m.grid(L), u, y_ref);
      tpmg_b200::ref::apply_operator(dm, L, u, y_dev);
      same("apply_operator (finest)", y_ref, y_dev);
      for (int l = 0; l < L; ++l) {  // every level
        const auto ul = random_field(l, nr, hier.grid(l).n_cells(), 40 + l);
        Field<double> a, b;
        apply_operator(m.coeff(l), m.grid(l), ul, a);
        tpmg_b200::ref::apply_operator(dm, l, ul, b);
        same(("apply_operator level " + std::to_string(l)).c_str(), a, b);
      }
      // smooth, relaxation.hpp:63-97: two block-Jacobi sweeps
      auto us_ref = u, us_dev = u;
      smooth(m.coeff(L), m.grid(L), us_ref, f, sm, 2);
      tpmg_b200::ref::smooth(dm, L, us_dev, f, 2);
      same("smooth (2 sweeps)", us_ref, us_dev);
      // transfers, multigrid.hpp:29-100 (all kinds, independent of the TransferConfig)
      for (int lc = 0; lc < L; ++lc) {
        const auto fine = random_field(lc + 1, nr, hier.grid(lc + 1).n_cells(), 10 + lc);
        const auto coarse = random_field(lc, nr, hier.grid(lc).n_cells(), 20 + lc);
        const std::string t = " " + std::to_string(lc);
        same(("restrict_field" + t).c_str(), restrict_field(fine, hier, lc),
             tpmg_b200::ref::restrict_field(dm, fine, lc));
        same(("restrict_field_transpose" + t).c_str(), restrict_field_transpose(fine, hier, lc),
             tpmg_b200::ref::restrict_field_transpose(dm, fine, lc));
        same(("prolongate_field linear" + t).c_str(),
             prolongate_field(coarse, hier, lc, ProlongationKind::linear),
             tpmg_b200::ref::prolongate_field(dm, coarse, lc, ProlongationKind::linear));
        same(("prolongate_field injection" + t).c_str(),
             prolongate_field(coarse, hier, lc, ProlongationKind::injection),
             tpmg_b200::ref::prolongate_field(dm, coarse, lc, ProlongationKind::injection));
      }
      // the reference's error types cross the boundary
      bool shape_thrown = false;
      try {
        Field<double> y;
        tpmg_b200::ref::apply_operator(dm, L, random_field(L, nr, ncL - 1, 5), y);
      } catch (const shape_error&) {
        shape_thrown = true;
      }
      std::printf("%-40s %s\n", "shape_error on a mismatched Field", shape_thrown ? "ok" : "MISSING");
      if (!shape_thrown) ++g_fail;
    }
    // v_cycle, multigrid.hpp:276-299, nonzero initial guess
    auto uv_ref = u0, uv_dev = u0;
    v_cycle(m, L, f, uv_ref);
    tpmg_b200::ref::v_cycle(dm, L, f, uv_dev);
    same(("v_cycle" + s).c_str(), uv_ref, uv_dev);
    // measure_cycle_rate, multigrid.hpp:302-321 (norm-based: reduction order is the device's)
    const double r_ref = measure_cycle_rate(m, f, 4);
    const double r_dev = tpmg_b200::ref::measure_cycle_rate(dm, f, 4);
    const bool ok = std::fabs(r_ref - r_dev) <= 1e-12 * std::fabs(r_ref);
    std::printf("%-40s %s (%.17g vs %.17g)\n", ("measure_cycle_rate" + s).c_str(),
                ok ? "within 1e-12" : "MISMATCH", r_ref, r_dev);
    if (!ok) ++g_fail;
  }
  std::printf("%s\n", g_fail ? "FAILED" : "ALL OK");
  return g_fail ? 1 : 0;
}
