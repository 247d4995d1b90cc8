// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Runs the REFERENCE's own hot-path code (/root/reference/proj/include/tpmg/*.hpp, compiled
// unmodified against oracle/eigen_shim) on the reference's icosahedral problem and dumps
// inputs + outputs, so that the CPU oracle (oracle/tpmg_oracle.cpp, fed the same neighbour /
// edge / child tables and hatted coefficients through tpmgo_generic_create) can be pinned
// against the reference itself (tests/test_ref_pin.py).
//
// Setup mirrors the reference's test fixtures (tests/fixtures.hpp:18-62): icosahedral
// hierarchy, balanced-flow factorised profiles WITH vertical advection, ν = 2 + 2, a
// geometrically graded vertical grid, block-Jacobi smoother with relax = 0.9.
//
// Output: a flat record file (name, dtype 'd'|'q', dims, data), read by tests/ref_pin_io.py.
#include <cstdint>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "tpmg/multigrid.hpp"

using namespace tpmg;

static FILE* g_out = nullptr;

static void rec(const std::string& name, char dtype, std::vector<int64_t> dims, const void* data,
                size_t elems) {
  const uint32_t nl = static_cast<uint32_t>(name.size());
  std::fwrite(&nl, 4, 1, g_out);
  std::fwrite(name.data(), 1, nl, g_out);
  std::fwrite(&dtype, 1, 1, g_out);
  const uint32_t nd = static_cast<uint32_t>(dims.size());
  std::fwrite(&nd, 4, 1, g_out);
  std::fwrite(dims.data(), 8, nd, g_out);
  std::fwrite(data, 8, elems, g_out);
}
static void recd(const std::string& n, const Matrix<double>& m) {
  rec(n, 'd', {m.rows(), m.cols()}, m.data(), m.size());
}
static void recv(const std::string& n, const Vector<double>& v) {
  rec(n, 'd', {v.size()}, v.data(), v.size());
}
static void recq(const std::string& n, const Index3X& m) {
  std::vector<int64_t> t(m.data(), m.data() + m.size());
  rec(n, 'q', {m.cols(), 3}, t.data(), t.size());
}
static void recs(const std::string& n, double v) { rec(n, 'd', {1}, &v, 1); }

static Field<double> random_field(int level, Index nr, Index nc, unsigned seed) {
  Field<double> u(level, nr, nc);
  std::mt19937 rng(seed);
  std::normal_distribution<double> dist;
  for (Index i = 0; i < u.values.size(); ++i) u.values.data()[i] = dist(rng);
  return u;
}

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "ref_pin.bin";
  g_out = std::fopen(path, "wb");
  if (!g_out) return 2;
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
  TransferConfig tr;  // production pair: linear + summation
  const auto m = build_hierarchy_coefficients(fac, hier, vert, op.omega, sm, tr, 2, 2, 0);
  recs("omega", op.omega);
  recs("relax", sm.relax);
  const int64_t nlev = m.depth();
  rec("n_levels", 'q', {1}, &nlev, 1);
  rec("nr", 'q', {1}, &nr, 1);
  for (int l = 0; l <= L; ++l) {
    const auto& g = hier.grid(l);
    const auto& h = m.coeff(l);
    const std::string s = std::to_string(l);
    recq("nbr" + s, g.neighbors);
    recq("cedge" + s, g.cell_edges);
    recv("bh" + s, h.beta.horiz);
    recv("ah" + s, h.alpha_r.horiz);
    recv("xh" + s, h.xi_r.horiz);
    recv("sh" + s, h.alpha_s.horiz);
    if (l == L) {
      recv("bv", h.beta.vert);
      recv("sv", h.alpha_s.vert);
      recv("av", h.alpha_r.vert);
      recv("xv", h.xi_r.vert);
    }
  }
  const auto& hL = m.finest_coefficients();
  const auto& gL = hier.finest();
  const Index ncL = gL.n_cells();
  const auto u = random_field(L, nr, ncL, 1);
  const auto f = random_field(L, nr, ncL, 2);
  const auto u0 = random_field(L, nr, ncL, 3);
  recd("u", u.values);
  recd("f", f.values);
  recd("u0", u0.values);

  // operator apply (discretization.hpp:262-278) and its explicit matrix (:291-316)
  recd("apply", apply_operator(hL, gL, u).values);
  {
    const auto A = dense_assemble(hL, gL);
    std::vector<double> tv;
    for (int outer = 0; outer < A.outerSize(); ++outer)
      for (Eigen::SparseMatrix<double>::InnerIterator it(A, outer); it; ++it) {
        tv.push_back(static_cast<double>(it.row()));
        tv.push_back(static_cast<double>(it.col()));
        tv.push_back(it.value());
      }
    rec("triplets", 'd', {static_cast<int64_t>(tv.size() / 3), 3}, tv.data(), tv.size());
  }
  // smoother (relaxation.hpp:63-97), 2 sweeps
  {
    auto us = u;
    smooth(hL, gL, us, f, sm, 2);
    recd("smooth2", us.values);
  }
  // Thomas on one column (relaxation.hpp:37-52)
  {
    const auto col = column_matrix(hL, gL, 5);
    Vector<double> rhs = random_field(L, nr, 1, 4).values.col(0);
    recv("th_diag", col.diag);
    recv("th_upper", col.upper);
    recv("th_lower", col.lower);
    recv("th_rhs", rhs);
    recv("th_x", thomas_solve(col, rhs));
  }
  // transfers (multigrid.hpp:29-100)
  for (int lc = 0; lc < L; ++lc) {
    const std::string s = std::to_string(lc);
    const auto fine = random_field(lc + 1, nr, hier.grid(lc + 1).n_cells(), 10 + lc);
    const auto coarse = random_field(lc, nr, hier.grid(lc).n_cells(), 20 + lc);
    recd("tr_fine" + s, fine.values);
    recd("tr_coarse" + s, coarse.values);
    recd("restrict_sum" + s, restrict_field(fine, hier, lc).values);
    recd("restrict_T" + s, restrict_field_transpose(fine, hier, lc).values);
    recd("prolong_lin" + s, prolongate_field(coarse, hier, lc, ProlongationKind::linear).values);
    recd("prolong_inj" + s, prolongate_field(coarse, hier, lc, ProlongationKind::injection).values);
  }
  // V-cycles (multigrid.hpp:276-299) for the three transfer pairs, nonzero initial guess
  const std::pair<ProlongationKind, RestrictionKind> pairs[3] = {
      {ProlongationKind::linear, RestrictionKind::summation},
      {ProlongationKind::linear, RestrictionKind::transpose},
      {ProlongationKind::injection, RestrictionKind::summation}};
  for (int c = 0; c < 3; ++c) {
    TransferConfig t;
    t.prolongation = pairs[c].first;
    t.restriction = pairs[c].second;
    const auto mc = build_hierarchy_coefficients(fac, hier, vert, op.omega, sm, t, 2, 2, 0);
    auto uv = u0;
    v_cycle(mc, L, f, uv);
    recd("vcycle" + std::to_string(c), uv.values);
    recs("rate" + std::to_string(c), measure_cycle_rate(mc, f, 4));
  }
  std::fclose(g_out);
  std::printf("wrote %s\n", path);
  return 0;
}
