// icosa_setup.cpp -- TEST INFRASTRUCTURE (oracle side; only tests/ load it): the reference's
// own test problem set up on the host in the reference's operation order, so that the device
// can be pinned against the reference's outputs (tests/golden/ref_icosa_pin.bin) from the
// reference's own fixture without the reference: the nested icosahedral grids
// (geometry.hpp:116-290), the radial grid (:295-327), the balanced-flow profiles
// (profiles.hpp:14-176, 262-392), assemble_hatted for factorised profiles
// (discretization.hpp:70-84, 146-184) and restrict_profiles (multigrid.hpp:107-201), ending in
// the same tables and hatted coefficients build_hierarchy_coefficients (multigrid.hpp:242-272)
// would hand to the V-cycle.  This is a restatement of the reference's setup code, kept out of
// the product: the product takes such tables through its C-ABI (tpmg_hier_create_generic).
//
// Arithmetic follows the reference expression by expression (left-to-right association, no
// contraction: this file is compiled with -ffp-contract=off) with Eigen's reductions as the
// oracle's Eigen shim evaluates them (sequential sums; v / |v| per component), which is how the
// committed golden outputs of the reference were produced -- tests/test_icosa_setup.py compares
// every table and coefficient bit for bit.
#include <cstdint>

// status codes and profile kinds of the product's C-ABI (include/tpmg_b200.h), restated so the
// oracle library stays standalone
enum { TPMG_OK = 0, TPMG_E_CONFIG = 1, TPMG_E_CAP = 6 };
enum { TPMG_PROFILE_FACTORIZED = 0, TPMG_PROFILE_FULL = 2 };
typedef struct tpmgo_icosa_params {
  int levels;              // refinements of the base icosahedron (grids 0..levels)
  int64_t n_r;             // vertical cells
  double depth;            // radial depth (units of the Earth's radius)
  int geometric;           // 0 uniform, 1 geometric grading
  double ratio;            // grading ratio
  double buoyancy_frequency;
  double courant;          // <= 0: courant_default's 10
  int advection;           // 0: without_advection
} tpmgo_icosa_params;
typedef struct tpmg_icosa_s* tpmg_icosa;

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <numbers>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace {

struct SetupError : std::runtime_error {
  int code;
  SetupError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};
thread_local std::string g_icosa_error;

// ---- 3-vectors with the shim's evaluation order ---------------------------------------------
struct V3 {
  double x = 0, y = 0, z = 0;
};
V3 operator+(const V3& a, const V3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V3 operator-(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 operator-(const V3& a) { return {-a.x, -a.y, -a.z}; }
double dot(const V3& a, const V3& b) {  // s = 0; s = s + a_i b_i
  double s = 0.0;
  s = s + a.x * b.x;
  s = s + a.y * b.y;
  s = s + a.z * b.z;
  return s;
}
double norm(const V3& a) { return std::sqrt(dot(a, a)); }
V3 normalized(const V3& a) {
  const double n = norm(a);
  return {a.x / n, a.y / n, a.z / n};
}
V3 cross(const V3& a, const V3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// arc_length / spherical_triangle_area, geometry.hpp:19-36
double arc(const V3& a, const V3& b) { return std::atan2(norm(cross(a, b)), dot(a, b)); }
double tri_area(const V3& v0, const V3& v1, const V3& v2) {
  const double a = arc(v1, v2), b = arc(v2, v0), c = arc(v0, v1);
  const double s = (a + b + c) / 2.0;
  const double t = std::tan(s / 2) * std::tan((s - a) / 2) * std::tan((s - b) / 2) *
                   std::tan((s - c) / 2);
  return 4.0 * std::atan(std::sqrt(std::max(t, 0.0)));
}

using Key = std::pair<int64_t, int64_t>;
Key key_of(int64_t a, int64_t b) { return a < b ? Key{a, b} : Key{b, a}; }

// HorizontalGrid, geometry.hpp:41-71
struct Grid {
  int level = 0;
  std::vector<V3> vertices;
  std::vector<std::array<int64_t, 3>> tri;
  std::vector<V3> centers;
  std::vector<double> areas;
  std::vector<int64_t> neighbors, cell_edges;  // [T*3 + j]
  std::vector<int64_t> ea, eb, va, vb;           // edge records
  std::vector<double> lengths;
  std::vector<V3> normals, midpoints;
  int64_t n_cells() const { return (int64_t)tri.size(); }
  int64_t n_edges() const { return (int64_t)ea.size(); }
  double geometry_factor(int64_t e) const {  // geometry.hpp:66-70
    const V3 chord = centers[(size_t)eb[(size_t)e]] - centers[(size_t)ea[(size_t)e]];
    return lengths[(size_t)e] * dot(normals[(size_t)e], chord) / dot(chord, chord);
  }
};

// base_icosahedron, geometry.hpp:115-152
Grid base_icosahedron() {
  constexpr double pi = std::numbers::pi_v<double>;
  Grid g;
  g.vertices.resize(12);
  g.vertices[0] = {0, 0, 1};
  g.vertices[11] = {0, 0, -1};
  const double lat = std::atan(0.5);
  for (int j = 0; j < 5; ++j) {
    const double lon_u = 2.0 * pi * double(j) / 5.0;
    const double lon_l = 2.0 * pi * (double(j) + 0.5) / 5.0;
    g.vertices[(size_t)(1 + j)] = {std::cos(lat) * std::cos(lon_u), std::cos(lat) * std::sin(lon_u),
                                   std::sin(lat)};
    g.vertices[(size_t)(6 + j)] = {std::cos(lat) * std::cos(lon_l), std::cos(lat) * std::sin(lon_l),
                                   -std::sin(lat)};
  }
  auto U = [](int j) { return int64_t(1 + (j % 5)); };
  auto L = [](int j) { return int64_t(6 + (j % 5)); };
  for (int j = 0; j < 5; ++j) g.tri.push_back({0, U(j), U(j + 1)});
  for (int j = 0; j < 5; ++j) g.tri.push_back({U(j), L(j), U(j + 1)});
  for (int j = 0; j < 5; ++j) g.tri.push_back({L(j), L(j + 1), U(j + 1)});
  for (int j = 0; j < 5; ++j) g.tri.push_back({11, L(j + 1), L(j)});
  for (auto& t : g.tri) {  // outward orientation
    const V3 v0 = g.vertices[(size_t)t[0]], v1 = g.vertices[(size_t)t[1]], v2 = g.vertices[(size_t)t[2]];
    if (dot(v0, cross(v1, v2)) < 0.0) std::swap(t[1], t[2]);
  }
  return g;
}

// refine, geometry.hpp:154-189: children 4c..4c+3, 4c+3 the medial triangle
Grid refine(const Grid& coarse, std::map<Key, int64_t>& midpoint_of) {
  Grid fine;
  fine.level = coarse.level + 1;
  fine.vertices = coarse.vertices;
  midpoint_of.clear();
  auto midpoint = [&](int64_t a, int64_t b) {
    const Key k = key_of(a, b);
    auto it = midpoint_of.find(k);
    if (it != midpoint_of.end()) return it->second;
    const int64_t id = (int64_t)fine.vertices.size();
    fine.vertices.push_back(normalized(coarse.vertices[(size_t)a] + coarse.vertices[(size_t)b]));
    midpoint_of.emplace(k, id);
    return id;
  };
  fine.tri.resize(4 * coarse.tri.size());
  for (size_t c = 0; c < coarse.tri.size(); ++c) {
    const int64_t v0 = coarse.tri[c][0], v1 = coarse.tri[c][1], v2 = coarse.tri[c][2];
    const int64_t m01 = midpoint(v0, v1), m12 = midpoint(v1, v2), m20 = midpoint(v2, v0);
    fine.tri[4 * c + 0] = {v0, m01, m20};
    fine.tri[4 * c + 1] = {v1, m12, m01};
    fine.tri[4 * c + 2] = {v2, m20, m12};
    fine.tri[4 * c + 3] = {m01, m12, m20};
  }
  return fine;
}

// finalize, geometry.hpp:191-257: centres, areas, edge records (in order of their second
// sighting), neighbour and edge maps
void finalize(Grid& g, std::map<Key, int64_t>* edge_of = nullptr) {
  const int64_t n = g.n_cells();
  g.centers.resize((size_t)n);
  g.areas.resize((size_t)n);
  for (int64_t c = 0; c < n; ++c) {
    const auto& t = g.tri[(size_t)c];
    const V3 v0 = g.vertices[(size_t)t[0]], v1 = g.vertices[(size_t)t[1]], v2 = g.vertices[(size_t)t[2]];
    g.centers[(size_t)c] = normalized(v0 + v1 + v2);
    g.areas[(size_t)c] = tri_area(v0, v1, v2);
  }
  g.neighbors.assign((size_t)(3 * n), -1);
  g.cell_edges.assign((size_t)(3 * n), -1);
  std::map<Key, std::pair<int64_t, int>> first_seen;
  for (int64_t c = 0; c < n; ++c) {
    for (int j = 0; j < 3; ++j) {
      const int64_t a = g.tri[(size_t)c][(size_t)((j + 1) % 3)], b = g.tri[(size_t)c][(size_t)((j + 2) % 3)];
      const Key k = key_of(a, b);
      auto it = first_seen.find(k);
      if (it == first_seen.end()) {
        first_seen.emplace(k, std::make_pair(c, j));
        continue;
      }
      const int64_t c0 = it->second.first;
      const int j0 = it->second.second;
      g.neighbors[(size_t)(3 * c0 + j0)] = c;
      g.neighbors[(size_t)(3 * c + j)] = c0;
      const int64_t e = g.n_edges();
      g.cell_edges[(size_t)(3 * c0 + j0)] = e;
      g.cell_edges[(size_t)(3 * c + j)] = e;
      g.ea.push_back(std::min(c0, c));
      g.eb.push_back(std::max(c0, c));
      g.va.push_back(k.first);
      g.vb.push_back(k.second);
      if (edge_of) edge_of->emplace(k, e);
    }
  }
  const int64_t ne = g.n_edges();
  g.lengths.resize((size_t)ne);
  g.normals.resize((size_t)ne);
  g.midpoints.resize((size_t)ne);
  for (int64_t e = 0; e < ne; ++e) {
    const V3 pa = g.vertices[(size_t)g.va[(size_t)e]], pb = g.vertices[(size_t)g.vb[(size_t)e]];
    g.lengths[(size_t)e] = arc(pa, pb);
    g.midpoints[(size_t)e] = normalized(pa + pb);
    V3 nrm = normalized(cross(pa, pb));
    if (dot(nrm, g.centers[(size_t)g.eb[(size_t)e]] - g.centers[(size_t)g.ea[(size_t)e]]) < 0.0) nrm = -nrm;
    g.normals[(size_t)e] = nrm;
  }
}

// VerticalGrid / build_vertical_grid, geometry.hpp:98-111, 292-327
struct Vert {
  int64_t n_r = 0;
  std::vector<double> r, volumes, sigma;
  double r_half(int64_t k) const { return (r[(size_t)k] + r[(size_t)k + 1]) / 2.0; }
  double r_half_below(int64_t k) const {
    return k == 0 ? r[0] : (r[(size_t)k - 1] + r[(size_t)k]) / 2.0;
  }
};
Vert vertical_grid(int64_t n_r, double depth, bool geometric, double ratio) {
  if (n_r < 1) throw SetupError(TPMG_E_CONFIG, "vertical grid needs at least one cell");
  if (!(depth > 0.0)) throw SetupError(TPMG_E_CONFIG, "vertical depth must be positive");
  if (!(ratio > 0.0)) throw SetupError(TPMG_E_CONFIG, "grading ratio must be positive");
  Vert v;
  v.n_r = n_r;
  v.r.resize((size_t)n_r + 1);
  if (!geometric || ratio == 1.0) {
    for (int64_t k = 0; k <= n_r; ++k) v.r[(size_t)k] = 1.0 + depth * double(k) / double(n_r);
  } else {
    const double dr0 = depth * (ratio - 1.0) / (std::pow(ratio, double(n_r)) - 1.0);
    v.r[0] = 1.0;
    double dr = dr0;
    for (int64_t k = 0; k < n_r; ++k, dr *= ratio) v.r[(size_t)k + 1] = v.r[(size_t)k] + dr;
  }
  v.r[0] = 1.0;
  v.r[(size_t)n_r] = 1.0 + depth;
  v.volumes.resize((size_t)n_r);
  for (int64_t k = 0; k < n_r; ++k)
    v.volumes[(size_t)k] =
        (std::pow(v.r[(size_t)k + 1], 3.0) - std::pow(v.r[(size_t)k], 3.0)) / 3.0;
  v.sigma.assign((size_t)n_r + 1, 1.0);
  v.sigma[0] = 0.0;
  v.sigma[(size_t)n_r] = 0.0;
  return v;
}

// ---- balanced flow, profiles.hpp:14-176 -------------------------------------------------------
struct Consts {  // PhysicalConstants defaults
  double p_0 = 10000, T_0 = 273, R_d = 287.05, c_p = 1005.0, g = 9.80665, R_earth = 6.371229e6;
  double Omega = 2.0 * std::numbers::pi_v<double> / 86400.0;
  double kappa() const { return R_d / c_p; }
  double gamma() const { return (1.0 - kappa()) / kappa(); }
  double c_s() const { return std::sqrt(c_p * T_0 / gamma()); }
  double c_h() const { return std::sqrt(gamma()) * c_s(); }
  double N_star() const { return g / c_h(); }
};
struct Jet {
  double u_0 = 100, phi_m = std::numbers::pi_v<double> / 4.0, sigma = 0.1;
};

template <typename Fn>
double simpson_rec(const Fn& f, double a, double b, double fa, double fm, double fb,
                   double whole, double tol, int depth) {
  const double m = (a + b) / 2;
  const double lm = (a + m) / 2, rm = (m + b) / 2;
  const double flm = f(lm), frm = f(rm);
  const double left = (m - a) / 6 * (fa + 4 * flm + fm);
  const double right = (b - m) / 6 * (fm + 4 * frm + fb);
  const double delta = left + right - whole;
  if (depth <= 0 || std::abs(delta) <= 15 * tol) return left + right + delta / 15;
  return simpson_rec(f, a, m, fa, flm, fm, left, tol / 2, depth - 1) +
         simpson_rec(f, m, b, fm, frm, fb, right, tol / 2, depth - 1);
}
template <typename Fn>
double simpson(const Fn& f, double a, double b, double tol) {
  if (a == b) return 0.0;
  const double fa = f(a), fb = f(b), fm = f((a + b) / 2);
  const double whole = (b - a) / 6 * (fa + 4 * fm + fb);
  return simpson_rec(f, a, b, fa, fm, fb, whole, tol, 48);
}

double jet_velocity(double phi, const Jet& jet) {
  const double d = std::cos(phi) - std::cos(jet.phi_m);
  return jet.u_0 * std::cos(phi) / std::cos(jet.phi_m) *
         std::exp(-d * d / (2 * jet.sigma * jet.sigma));
}

double jet_function(double phi, const Jet& jet, const Consts& c) {
  const auto integrand = [&](double p) {
    const double us = jet_velocity(p, jet);
    const double d = std::cos(p) - std::cos(jet.phi_m);
    const double us2_tan = jet.u_0 * jet.u_0 * std::cos(p) * std::sin(p) /
                           (std::cos(jet.phi_m) * std::cos(jet.phi_m)) *
                           std::exp(-d * d / (jet.sigma * jet.sigma));
    return 2 * c.R_earth * c.Omega * us * std::sin(p) + us2_tan;
  };
  const double tol = 1e-8 * c.R_earth * c.Omega * jet.u_0;
  if (phi >= 0.0) return simpson(integrand, 0.0, phi, tol);
  return -simpson(integrand, phi, 0.0, tol);
}

struct Flow {
  Consts c;
  Jet jet;
  double n = 0, eps = 0;
  explicit Flow(double N) : n(N) {
    const double ns = c.N_star();
    eps = (n / ns) * (n / ns) - 1.0;
    if (eps < -1e-12) throw SetupError(TPMG_E_CONFIG, "buoyancy frequency below N*: epsilon < 0 unsupported");
    eps = std::max(eps, 0.0);
  }
  double horizontal_exp(double phi) const {
    return std::exp(-n * n / (c.g * c.g) * jet_function(phi, jet, c));
  }
  double vertical_exp(double r) const { return std::exp(-n * n * c.R_earth / c.g * (r - 1.0)); }
  static double latitude(const V3& rh) { return std::asin(std::clamp(rh.z, -1.0, 1.0)); }
  // state_from_exp, profiles.hpp:159-166
  void state(double es, double er, double& exner, double& rho) const {
    const double e = es * er;
    exner = (eps + e) / (1.0 + eps);
    rho = c.p_0 / (c.R_d * c.T_0) * std::pow(exner, c.gamma()) * e;
  }
};

struct Factorized {  // FactorizedProfileSet, profiles.hpp:196-210
  std::vector<double> beta_r, alpha_s_r, alpha_r_r, xi_r_r, beta_s, alpha_r_s, xi_r_s, alpha_s_s;
};
struct Full {  // ProfileSet, profiles.hpp:181-192 (column-major, k fastest)
  std::vector<double> beta, alpha_s, alpha_r, xi_r;
};

// factorize_balanced_flow, profiles.hpp:329-391
Factorized factorize(const Grid& g, const Vert& v, const Flow& flow, double mu_dt) {
  const Consts& c = flow.c;
  const int64_t ns = g.n_cells(), ne = g.n_edges(), nr = v.n_r;
  const double eps = flow.eps, n2 = flow.n * flow.n;
  const double lambda_bar = 1.0 / (1.0 + mu_dt * mu_dt * n2);
  const double dlog = n2 * c.R_earth / c.g;
  const double gam = c.gamma();
  struct VF {
    double beta, alpha_s, alpha_r_over_r2, xi;
  };
  auto vertical = [&](double r) {
    const double er = flow.vertical_exp(r);
    const double pi_r = (eps + er) / (1.0 + eps);
    const double rho_r = c.p_0 / (c.R_d * c.T_0) * std::pow(pi_r, gam) * er;
    const double theta_r = 1.0 / er;
    return VF{gam * rho_r / pi_r, rho_r * theta_r, lambda_bar * rho_r * theta_r,
              lambda_bar * rho_r * theta_r * dlog};
  };
  Factorized f;
  f.beta_r.resize((size_t)nr);
  f.alpha_s_r.resize((size_t)nr);
  f.alpha_r_r.resize((size_t)nr + 1);
  f.xi_r_r.resize((size_t)nr + 1);
  for (int64_t k = 0; k < nr; ++k) {
    const VF x = vertical(v.r_half(k));
    f.beta_r[(size_t)k] = x.beta;
    f.alpha_s_r[(size_t)k] = x.alpha_s;
  }
  for (int64_t k = 0; k <= nr; ++k) {
    const double rk = v.r[(size_t)k];
    f.alpha_r_r[(size_t)k] = rk * rk * vertical(rk).alpha_r_over_r2;
    f.xi_r_r[(size_t)k] = vertical(v.r_half_below(k)).xi;
  }
  auto horizontal = [&](double phi) { return std::pow(flow.horizontal_exp(phi), gam); };
  f.beta_s.resize((size_t)ns);
  f.alpha_r_s.resize((size_t)ns);
  f.xi_r_s.resize((size_t)ns);
  for (int64_t T = 0; T < ns; ++T) {
    const double h = horizontal(Flow::latitude(g.centers[(size_t)T]));
    f.beta_s[(size_t)T] = f.alpha_r_s[(size_t)T] = f.xi_r_s[(size_t)T] = h;
  }
  f.alpha_s_s.resize((size_t)ne);
  for (int64_t e = 0; e < ne; ++e)
    f.alpha_s_s[(size_t)e] = horizontal(Flow::latitude(g.midpoints[(size_t)e]));
  return f;
}

// balanced_flow_profiles + profile_factors, profiles.hpp:262-324
Full full_profiles(const Grid& g, const Vert& v, const Flow& flow, double mu_dt) {
  const Consts& c = flow.c;
  const int64_t ns = g.n_cells(), ne = g.n_edges(), nr = v.n_r;
  const double n2 = flow.n * flow.n;
  const double lambda_bar = 1.0 / (1.0 + mu_dt * mu_dt * n2);
  struct PF {
    double beta, alpha_s, alpha_r_over_r2, xi_r;
  };
  auto factors = [&](double es, double er) {
    double exner, rho;
    flow.state(es, er, exner, rho);
    const double theta_nd = 1.0 / (es * er);
    const double dlog_theta = flow.n * flow.n * c.R_earth / c.g;
    return PF{c.gamma() * rho / exner, rho * theta_nd, lambda_bar * rho * theta_nd,
              lambda_bar * rho * theta_nd * dlog_theta};
  };
  Full p;
  p.beta.resize((size_t)(nr * ns));
  p.alpha_s.resize((size_t)(nr * ne));
  p.alpha_r.resize((size_t)((nr + 1) * ns));
  p.xi_r.resize((size_t)((nr + 1) * ns));
  for (int64_t T = 0; T < ns; ++T) {
    const double es = flow.horizontal_exp(Flow::latitude(g.centers[(size_t)T]));
    for (int64_t k = 0; k < nr; ++k)
      p.beta[(size_t)(T * nr + k)] = factors(es, flow.vertical_exp(v.r_half(k))).beta;
    for (int64_t k = 0; k <= nr; ++k) {
      const double rk = v.r[(size_t)k];
      p.alpha_r[(size_t)(T * (nr + 1) + k)] =
          rk * rk * factors(es, flow.vertical_exp(rk)).alpha_r_over_r2;
      p.xi_r[(size_t)(T * (nr + 1) + k)] = factors(es, flow.vertical_exp(v.r_half_below(k))).xi_r;
    }
  }
  for (int64_t e = 0; e < ne; ++e) {
    const double es = flow.horizontal_exp(Flow::latitude(g.midpoints[(size_t)e]));
    for (int64_t k = 0; k < nr; ++k)
      p.alpha_s[(size_t)(e * nr + k)] = factors(es, flow.vertical_exp(v.r_half(k))).alpha_s;
  }
  return p;
}

// hatted coefficients of one level from factorised profiles, discretization.hpp:146-184
struct Hatted {
  std::vector<double> bv, sv, av, xv, bh, ah, xh, sh;
};
Hatted assemble(const Factorized& p, const Grid& g, const Vert& v, double omega) {
  const int64_t nr = v.n_r, ns = g.n_cells(), ne = g.n_edges();
  const double w2 = omega * omega;
  Hatted h;
  h.bv.resize((size_t)nr);
  h.sv.resize((size_t)nr);
  for (int64_t k = 0; k < nr; ++k) {
    h.bv[(size_t)k] = v.volumes[(size_t)k] * p.beta_r[(size_t)k];
    h.sv[(size_t)k] = (v.r[(size_t)k + 1] - v.r[(size_t)k]) * p.alpha_s_r[(size_t)k];
  }
  h.av.assign((size_t)nr + 1, 0.0);
  h.xv.assign((size_t)nr + 1, 0.0);
  for (int64_t k = 0; k <= nr; ++k) {  // face factors, discretization.hpp:70-84 (0 on the boundary)
    double fd = 0.0, fa = 0.0;
    if (k >= 1 && k < nr) {
      const double rk = v.r[(size_t)k], rp = v.r[(size_t)k + 1], rm = v.r[(size_t)k - 1];
      fd = 2 * rk * rk / (rp - rm);
      fa = rk * rk * (rp - rk) / (rp - rm);
    }
    h.av[(size_t)k] = fd * p.alpha_r_r[(size_t)k];
    h.xv[(size_t)k] = fa * p.xi_r_r[(size_t)k];
  }
  h.bh.resize((size_t)ns);
  h.ah.resize((size_t)ns);
  h.xh.resize((size_t)ns);
  for (int64_t T = 0; T < ns; ++T) {
    const double A = g.areas[(size_t)T];
    h.bh[(size_t)T] = A * p.beta_s[(size_t)T];
    h.ah[(size_t)T] = w2 * (A * p.alpha_r_s[(size_t)T]);
    h.xh[(size_t)T] = w2 * (A * p.xi_r_s[(size_t)T]);
  }
  h.sh.resize((size_t)ne);
  for (int64_t e = 0; e < ne; ++e) h.sh[(size_t)e] = w2 * g.geometry_factor(e) * p.alpha_s_s[(size_t)e];
  return h;
}

// restrict_profiles for a factorised set, multigrid.hpp:107-149, 171-185: cell scalars by the
// area-weighted mean of the four children, edge scalars by the mean of the two co-linear ones
Factorized restrict_fact(const Factorized& fine, const Grid& fg, int64_t ncoarse,
                         const std::vector<std::array<int64_t, 2>>& colinear) {
  Factorized c = fine;
  auto cells = [&](const std::vector<double>& f) {
    std::vector<double> out((size_t)ncoarse);
    for (int64_t T = 0; T < ncoarse; ++T) {
      double wsum = 0.0, acc = 0.0;
      for (int j = 0; j < 4; ++j) {
        const int64_t ch = 4 * T + j;
        const double w = fg.areas[(size_t)ch];
        acc = acc + w * f[(size_t)ch];
        wsum += w;
      }
      out[(size_t)T] = acc / wsum;
    }
    return out;
  };
  c.beta_s = cells(fine.beta_s);
  c.alpha_r_s = cells(fine.alpha_r_s);
  c.xi_r_s = cells(fine.xi_r_s);
  c.alpha_s_s.resize(colinear.size());
  for (size_t e = 0; e < colinear.size(); ++e)
    c.alpha_s_s[e] = (fine.alpha_s_s[(size_t)colinear[e][0]] + fine.alpha_s_s[(size_t)colinear[e][1]]) / 2.0;
  return c;
}

}  // namespace

struct tpmg_icosa_s {
  tpmgo_icosa_params prm{};
  std::vector<Grid> grids;                                   // levels 0..L
  std::vector<std::vector<std::array<int64_t, 2>>> colinear;  // [l]: coarse level l edges
  Vert vert;
  double omega = 0, mu_dt = 0, eps = 0;
  Factorized fac;   // finest level
  Full full;        // finest level
  std::vector<Hatted> hatted;  // per level
  std::vector<std::vector<double>> centers;  // per level, 3 per cell
};

namespace {

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return TPMG_OK;
  } catch (const SetupError& e) {
    g_icosa_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_icosa_error = "out of host memory";
    return TPMG_E_CAP;
  } catch (const std::exception& e) {
    g_icosa_error = e.what();
    return TPMG_E_CONFIG;
  }
}

}  // namespace

extern "C" {

const char* tpmgo_icosa_last_error(void) { return g_icosa_error.c_str(); }

int tpmgo_icosa_create(const tpmgo_icosa_params* p, tpmg_icosa* out) {
  return guard([&] {
    if (!p || !out) throw SetupError(TPMG_E_CONFIG, "tpmgo_icosa_create: null argument");
    if (p->levels < 0 || p->levels > 9)
      throw SetupError(TPMG_E_CONFIG, "level count must be in [0, 9]");
    auto ico = std::make_unique<tpmg_icosa_s>();
    ico->prm = *p;
    // build_icosahedral_hierarchy, geometry.hpp:263-290
    ico->grids.push_back(base_icosahedron());
    finalize(ico->grids[0]);
    for (int l = 0; l < p->levels; ++l) {
      std::map<Key, int64_t> midpoint_of, fine_edge_of;
      Grid fine = refine(ico->grids.back(), midpoint_of);
      finalize(fine, &fine_edge_of);
      const Grid& coarse = ico->grids.back();
      std::vector<std::array<int64_t, 2>> co((size_t)coarse.n_edges());
      for (int64_t e = 0; e < coarse.n_edges(); ++e) {
        const int64_t a = coarse.va[(size_t)e], b = coarse.vb[(size_t)e];
        const int64_t m = midpoint_of.at(key_of(a, b));
        co[(size_t)e] = {fine_edge_of.at(key_of(a, m)), fine_edge_of.at(key_of(m, b))};
      }
      ico->colinear.push_back(std::move(co));
      ico->grids.push_back(std::move(fine));
    }
    ico->vert = vertical_grid(p->n_r, p->depth, p->geometric != 0, p->ratio);
    const Flow flow(p->buoyancy_frequency);
    // OperatorParameters::courant_default, profiles.hpp:40-54 (mean_edge_length: sum / n)
    const Grid& fg = ico->grids.back();
    double sum = fg.lengths[0];
    for (size_t e = 1; e < fg.lengths.size(); ++e) sum = sum + fg.lengths[e];
    const double courant = p->courant > 0.0 ? p->courant : 10.0;
    ico->omega = courant * (sum / double(fg.lengths.size()));
    if (!(ico->omega > 0.0)) throw SetupError(TPMG_E_CONFIG, "omega must be positive");
    ico->mu_dt = ico->omega * flow.c.R_earth / flow.c.c_h();
    ico->eps = flow.eps;
    ico->fac = factorize(fg, ico->vert, flow, ico->mu_dt);
    ico->full = full_profiles(fg, ico->vert, flow, ico->mu_dt);
    if (!p->advection) {  // without_advection, profiles.hpp:393-403
      std::fill(ico->fac.xi_r_r.begin(), ico->fac.xi_r_r.end(), 0.0);
      std::fill(ico->full.xi_r.begin(), ico->full.xi_r.end(), 0.0);
    }
    // build_hierarchy_coefficients' loop, multigrid.hpp:263-268: assemble, then restrict
    const int L = p->levels;
    ico->hatted.resize((size_t)L + 1);
    Factorized prof = ico->fac;
    for (int l = L; l >= 0; --l) {
      ico->hatted[(size_t)l] = assemble(prof, ico->grids[(size_t)l], ico->vert, ico->omega);
      if (l > 0)
        prof = restrict_fact(prof, ico->grids[(size_t)l], ico->grids[(size_t)l - 1].n_cells(),
                             ico->colinear[(size_t)l - 1]);
    }
    for (const Grid& g : ico->grids) {
      std::vector<double> c;
      c.reserve((size_t)(3 * g.n_cells()));
      for (const V3& v : g.centers) {
        c.push_back(v.x);
        c.push_back(v.y);
        c.push_back(v.z);
      }
      ico->centers.push_back(std::move(c));
    }
    *out = ico.release();
  });
}

int tpmgo_icosa_destroy(tpmg_icosa ico) {
  delete ico;
  return TPMG_OK;
}

int tpmgo_icosa_info(tpmg_icosa ico, int* n_levels, double* omega, double* mu_dt,
                    double* epsilon) {
  return guard([&] {
    if (!ico) throw SetupError(TPMG_E_CONFIG, "null problem");
    if (n_levels) *n_levels = (int)ico->grids.size();
    if (omega) *omega = ico->omega;
    if (mu_dt) *mu_dt = ico->mu_dt;
    if (epsilon) *epsilon = ico->eps;
  });
}

int tpmgo_icosa_level(tpmg_icosa ico, int level, int64_t* n_cells, int64_t* n_edges,
                     const int64_t** neighbors, const int64_t** cell_edges,
                     const double** centers, const double** areas) {
  return guard([&] {
    if (!ico || level < 0 || level >= (int)ico->grids.size())
      throw SetupError(TPMG_E_CONFIG, "tpmgo_icosa_level: no such level");
    const Grid& g = ico->grids[(size_t)level];
    if (n_cells) *n_cells = g.n_cells();
    if (n_edges) *n_edges = g.n_edges();
    if (neighbors) *neighbors = g.neighbors.data();
    if (cell_edges) *cell_edges = g.cell_edges.data();
    if (centers) *centers = ico->centers[(size_t)level].data();
    if (areas) *areas = g.areas.data();
  });
}

int tpmgo_icosa_hatted(tpmg_icosa ico, int level, const double** bh, const double** ah,
                      const double** xh, const double** sh, const double** bv, const double** sv,
                      const double** av, const double** xv) {
  return guard([&] {
    if (!ico || level < 0 || level >= (int)ico->hatted.size())
      throw SetupError(TPMG_E_CONFIG, "tpmgo_icosa_hatted: no such level");
    const Hatted& h = ico->hatted[(size_t)level];
    if (bh) *bh = h.bh.data();
    if (ah) *ah = h.ah.data();
    if (xh) *xh = h.xh.data();
    if (sh) *sh = h.sh.data();
    if (bv) *bv = h.bv.data();
    if (sv) *sv = h.sv.data();
    if (av) *av = h.av.data();
    if (xv) *xv = h.xv.data();
  });
}

int tpmgo_icosa_profiles(tpmg_icosa ico, int kind, double* packed, int64_t capacity) {
  return guard([&] {
    if (!ico || !packed) throw SetupError(TPMG_E_CONFIG, "tpmgo_icosa_profiles: null argument");
    std::vector<const std::vector<double>*> parts;
    if (kind == TPMG_PROFILE_FACTORIZED) {
      const Factorized& f = ico->fac;
      parts = {&f.beta_r, &f.alpha_s_r, &f.alpha_r_r, &f.xi_r_r,
               &f.beta_s, &f.alpha_r_s, &f.xi_r_s,    &f.alpha_s_s};
    } else if (kind == TPMG_PROFILE_FULL) {
      const Full& f = ico->full;
      parts = {&f.beta, &f.alpha_s, &f.alpha_r, &f.xi_r};
    } else {
      throw SetupError(TPMG_E_CONFIG, "tpmgo_icosa_profiles: unknown kind");
    }
    int64_t n = 0;
    for (const auto* v : parts) n += (int64_t)v->size();
    if (n > capacity) throw SetupError(TPMG_E_CAP, "tpmgo_icosa_profiles: buffer too small");
    for (const auto* v : parts) {
      std::memcpy(packed, v->data(), v->size() * sizeof(double));
      packed += v->size();
    }
  });
}

}  // extern "C"
