// tpmg_b200_ref.hpp -- drop-in adapter for a caller that holds the REFERENCE's own objects
// (proj/include/tpmg/*.hpp: MultigridHierarchy<double>, Field<double>).  Include it after the
// reference's headers:
//
//   #include "tpmg/multigrid.hpp"   // the reference library
//   #include "tpmg_b200_ref.hpp"    // this adapter (C-ABI tpmg_b200.h underneath)
//
//   const auto m = tpmg::build_hierarchy_coefficients(fac, hier, vert, omega, sm, tr, 2, 2);
//   tpmg_b200::Context ctx;                        // one GPU
//   tpmg_b200::ref::DeviceMultigrid dm(ctx, m);    // device-resident copy of m (once)
//
//   reference call (CPU)                                  device call (sm_100a), same arguments
//   tpmg::v_cycle(m, L, f, u)        multigrid.hpp:276    tpmg_b200::ref::v_cycle(dm, L, f, u)
//   tpmg::apply_operator(m.coeff(l), m.grid(l), u, out)   tpmg_b200::ref::apply_operator(dm, l, u, out)
//                                    discretization.hpp:262
//   tpmg::smooth(m.coeff(l), m.grid(l), u, f, m.smoother, s)  tpmg_b200::ref::smooth(dm, l, u, f, s)
//                                    relaxation.hpp:63
//   tpmg::restrict_field(fine, *m.grids, lc)             tpmg_b200::ref::restrict_field(dm, fine, lc)
//   tpmg::restrict_field_transpose(fine, *m.grids, lc)   tpmg_b200::ref::restrict_field_transpose(dm, fine, lc)
//   tpmg::prolongate_field(c, *m.grids, lc, kind)        tpmg_b200::ref::prolongate_field(dm, c, lc, kind)
//                                    multigrid.hpp:29-100
//   tpmg::measure_cycle_rate(m, f, n) multigrid.hpp:302  tpmg_b200::ref::measure_cycle_rate(dm, f, n)
//
// The Field arguments are the reference's own (values: n_r x n_cells, column-major, k fastest,
// discretization.hpp:14-19); they cross the boundary in that layout (TPMG_LAYOUT_K_FASTEST).
// The device hierarchy takes the reference's grid tables (neighbors / cell_edges, child_of(Tc, j)
// = 4 Tc + j, geometry.hpp:51-53, 89-90) and its separable hatted coefficients as they are
// (tpmg_hier_create_generic), so every element-wise result is bitwise the reference's
// (tests/test_ref_adapter_gpu.py).  Limits, raised as the reference's own exception types
// (types.hpp:24-58): the device smoother is block-Jacobi (block-SOR is sequential by contract,
// relaxation.hpp:13-16), coefficients must be separable (the factorised profile set), and
// v_cycle / measure_cycle_rate run from the finest level of m.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "tpmg_b200.hpp"

namespace tpmg_b200 {
namespace ref {

// Status -> the reference's exception types (types.hpp:24-58).
inline void check_ref(int rc, tpmg_context ctx = nullptr) {
  if (rc == TPMG_OK) return;
  const std::string msg = std::string(tpmg_status_string(rc)) + ": " + tpmg_last_error(ctx);
  switch (rc) {
    case TPMG_E_CONFIG: throw tpmg::config_error(msg);
    case TPMG_E_SHAPE: throw tpmg::shape_error(msg);
    case TPMG_E_NONFINITE: throw tpmg::nonfinite_error(msg);
    case TPMG_E_FINGERPRINT: throw tpmg::fingerprint_error(msg);
    case TPMG_E_SINGULAR: throw tpmg::singular_error(msg);
    case TPMG_E_CAP: throw tpmg::cap_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// build_hierarchy_coefficients' result (multigrid.hpp:207-272), uploaded once.
class DeviceMultigrid {
 public:
  DeviceMultigrid(const Context& ctx, const tpmg::MultigridHierarchy<double>& m)
      : ctx_(ctx.get()), coarsest_(m.coarsest_level), finest_(m.finest_level()) {
    if (!m.grids) throw tpmg::config_error("MultigridHierarchy without grids");
    if (m.smoother.kind != tpmg::SmootherKind::block_jacobi)
      throw tpmg::config_error("device smoother is block-Jacobi (block-SOR is sequential)");
    const int nl = m.depth();
    const tpmg::Index nr = m.finest_coefficients().n_r();
    std::vector<int64_t> nc, ne;
    std::vector<std::vector<int64_t>> nbr, ced, chd;
    std::vector<const int64_t*> pn, pc, pch;
    std::vector<const double*> bh, ah, xh, sh;
    for (int l = coarsest_; l <= finest_; ++l) {
      const auto& g = m.grid(l);
      const auto& h = m.coeff(l);
      if (!h.fully_separable())
        throw tpmg::config_error("device hierarchy needs separable (factorised) coefficients");
      nc.push_back(g.n_cells());
      ne.push_back(g.n_edges());
      nbr.emplace_back(g.neighbors.data(), g.neighbors.data() + g.neighbors.size());
      ced.emplace_back(g.cell_edges.data(), g.cell_edges.data() + g.cell_edges.size());
      std::vector<int64_t> ch;
      if (l > coarsest_) {  // GridHierarchy::child_of(Tc, j) = 4 Tc + j
        const tpmg::Index ncc = m.grid(l - 1).n_cells();
        ch.resize(static_cast<size_t>(4 * ncc));
        for (tpmg::Index tc = 0; tc < ncc; ++tc)
          for (int j = 0; j < 4; ++j)
            ch[static_cast<size_t>(4 * tc + j)] = tpmg::GridHierarchy<double>::child_of(tc, j);
      }
      chd.push_back(std::move(ch));
      bh.push_back(h.beta.horiz.data());
      ah.push_back(h.alpha_r.horiz.data());
      xh.push_back(h.xi_r.horiz.data());
      sh.push_back(h.alpha_s.horiz.data());
    }
    for (int i = 0; i < nl; ++i) {
      pn.push_back(nbr[static_cast<size_t>(i)].data());
      pc.push_back(ced[static_cast<size_t>(i)].data());
      pch.push_back(chd[static_cast<size_t>(i)].empty() ? nullptr : chd[static_cast<size_t>(i)].data());
    }
    // pre/post sweeps: refined levels share nu (the coarsest is 1 + 0, multigrid.hpp:269-270)
    const int nu_pre = nl > 1 ? m.pre_sweeps(finest_) : 1;
    const int nu_post = nl > 1 ? m.post_sweeps(finest_) : 0;
    for (int l = coarsest_ + 1; l <= finest_; ++l)
      if (m.pre_sweeps(l) != nu_pre || m.post_sweeps(l) != nu_post)
        throw tpmg::config_error("device hierarchy needs the same nu on every refined level");
    // linear prolongation's corner rule (multigrid.hpp:88-95): corner child j takes the coarse
    // neighbours across edges (j+1)%3 and (j+2)%3, the centre child (j = 3) none
    const int d1[4] = {1, 2, 0, -1}, d2[4] = {2, 0, 1, -1};
    const auto& hf = m.finest_coefficients();
    check_ref(tpmg_hier_create_generic(
                  ctx_, nl, static_cast<int>(nr), 3, 4, nc.data(), ne.data(), pn.data(), pc.data(),
                  pch.data(), d1, d2, hf.beta.vert.data(), hf.alpha_s.vert.data(),
                  hf.alpha_r.vert.data(), hf.xi_r.vert.data(), bh.data(), ah.data(), xh.data(),
                  sh.data(), m.smoother.relax,
                  m.transfers.prolongation == tpmg::ProlongationKind::linear ? TPMG_PROLONG_LINEAR
                                                                             : TPMG_PROLONG_INJECTION,
                  m.transfers.restriction == tpmg::RestrictionKind::summation ? TPMG_RESTRICT_SUMMATION
                                                                              : TPMG_RESTRICT_TRANSPOSE,
                  nu_pre, nu_post, &h_),
              ctx_);
    n_r_ = nr;
  }
  ~DeviceMultigrid() { tpmg_hier_destroy(h_); }
  DeviceMultigrid(const DeviceMultigrid&) = delete;
  DeviceMultigrid& operator=(const DeviceMultigrid&) = delete;

  tpmg_hierarchy get() const { return h_; }
  tpmg_context context() const { return ctx_; }
  int coarsest_level() const { return coarsest_; }
  int finest_level() const { return finest_; }
  tpmg::Index n_r() const { return n_r_; }
  // device level of reference level l
  int dev(int l) const {
    if (l < coarsest_ || l > finest_) throw tpmg::shape_error("level outside the hierarchy");
    return l - coarsest_;
  }

 private:
  tpmg_context ctx_;
  tpmg_hierarchy h_ = nullptr;
  int coarsest_, finest_;
  tpmg::Index n_r_ = 0;
};

namespace detail {
// A device field holding a reference Field's values (k fastest at the boundary).
struct DevField {
  tpmg_context ctx;
  tpmg_field f = nullptr;
  DevField(const DeviceMultigrid& dm, int level) : ctx(dm.context()) {
    check_ref(tpmg_field_create(dm.get(), dm.dev(level), &f), ctx);
  }
  ~DevField() { tpmg_field_destroy(f); }
  void up(const tpmg::Field<double>& a, tpmg::Index n_cells) {
    if (a.values.rows() != 0 && a.values.cols() != n_cells)
      throw tpmg::shape_error("field does not match the grid level");
    check_ref(tpmg_field_upload(f, a.values.data(), TPMG_LAYOUT_K_FASTEST), ctx);
  }
  void down(tpmg::Field<double>& a, int level, tpmg::Index n_r, tpmg::Index n_cells) {
    a.level = level;
    a.values.resize(n_r, n_cells);
    check_ref(tpmg_field_download(f, a.values.data(), TPMG_LAYOUT_K_FASTEST), ctx);
  }
};
inline tpmg::Index cells(const DeviceMultigrid& dm, int level) {
  int64_t nx = 0, ny = 0, nz = 0, x0 = 0, y0 = 0;
  check_ref(tpmg_hier_level_shape(dm.get(), dm.dev(level), &nx, &ny, &nz, &x0, &y0), dm.context());
  return static_cast<tpmg::Index>(nx * ny);
}
inline void need(const tpmg::Field<double>& a, int level, tpmg::Index n_r, tpmg::Index n_cells) {
  if (a.level != level || a.values.rows() != n_r || a.values.cols() != n_cells)
    throw tpmg::shape_error("field does not match the hierarchy level");
}
}  // namespace detail

// apply_operator(h, grid, u, out), discretization.hpp:262-278: out is resized like the reference's
inline void apply_operator(const DeviceMultigrid& dm, int level, const tpmg::Field<double>& u,
                           tpmg::Field<double>& out) {
  const tpmg::Index nc = detail::cells(dm, level);
  detail::need(u, level, dm.n_r(), nc);
  detail::DevField du(dm, level), dy(dm, level);
  du.up(u, nc);
  check_ref(tpmg_apply(dm.get(), du.f, dy.f), dm.context());
  dy.down(out, level, dm.n_r(), nc);
}

// smooth(h, grid, u, f, cfg, sweeps), relaxation.hpp:63-97 (block-Jacobi, cfg.relax of the hierarchy)
inline void smooth(const DeviceMultigrid& dm, int level, tpmg::Field<double>& u,
                   const tpmg::Field<double>& f, int sweeps) {
  const tpmg::Index nc = detail::cells(dm, level);
  detail::need(u, level, dm.n_r(), nc);
  detail::need(f, level, dm.n_r(), nc);
  detail::DevField du(dm, level), df(dm, level);
  du.up(u, nc);
  df.up(f, nc);
  check_ref(tpmg_smooth(dm.get(), du.f, df.f, sweeps), dm.context());
  du.down(u, level, dm.n_r(), nc);
}

namespace detail {
inline tpmg::Field<double> restrict_impl(const DeviceMultigrid& dm, const tpmg::Field<double>& fine,
                                         int coarse_level, bool transpose) {
  if (fine.level != coarse_level + 1)
    throw tpmg::shape_error("restrict: fine field is not one level above the target");
  const tpmg::Index ncf = cells(dm, coarse_level + 1), ncc = cells(dm, coarse_level);
  need(fine, coarse_level + 1, dm.n_r(), ncf);
  DevField df(dm, coarse_level + 1), dc(dm, coarse_level);
  df.up(fine, ncf);
  check_ref(tpmg_restrict_kind(dm.get(), df.f, dc.f,
                               transpose ? TPMG_RESTRICT_TRANSPOSE : TPMG_RESTRICT_SUMMATION),
            dm.context());
  tpmg::Field<double> out;
  dc.down(out, coarse_level, dm.n_r(), ncc);
  return out;
}
}  // namespace detail

// restrict_field / restrict_field_transpose, multigrid.hpp:29-69
inline tpmg::Field<double> restrict_field(const DeviceMultigrid& dm, const tpmg::Field<double>& fine,
                                          int coarse_level) {
  return detail::restrict_impl(dm, fine, coarse_level, false);
}
inline tpmg::Field<double> restrict_field_transpose(const DeviceMultigrid& dm,
                                                    const tpmg::Field<double>& fine,
                                                    int coarse_level) {
  return detail::restrict_impl(dm, fine, coarse_level, true);
}

// prolongate_field(coarse, hier, coarse_level, kind), multigrid.hpp:74-100
inline tpmg::Field<double> prolongate_field(const DeviceMultigrid& dm,
                                            const tpmg::Field<double>& coarse, int coarse_level,
                                            tpmg::ProlongationKind kind) {
  if (coarse.level != coarse_level) throw tpmg::shape_error("prolongate: field level does not match");
  const tpmg::Index ncc = detail::cells(dm, coarse_level), ncf = detail::cells(dm, coarse_level + 1);
  detail::need(coarse, coarse_level, dm.n_r(), ncc);
  detail::DevField dc(dm, coarse_level), df(dm, coarse_level + 1);
  dc.up(coarse, ncc);
  check_ref(tpmg_prolong_kind(dm.get(), dc.f, df.f,
                              kind == tpmg::ProlongationKind::linear ? TPMG_PROLONG_LINEAR
                                                                     : TPMG_PROLONG_INJECTION,
                              0),
            dm.context());
  tpmg::Field<double> out;
  df.down(out, coarse_level + 1, dm.n_r(), ncf);
  return out;
}

// v_cycle(m, level, f, u), multigrid.hpp:276-299 (from the finest level of m)
inline void v_cycle(const DeviceMultigrid& dm, int level, const tpmg::Field<double>& f,
                    tpmg::Field<double>& u) {
  if (level != dm.finest_level())
    throw tpmg::config_error("device v_cycle starts at the finest level of the hierarchy");
  const tpmg::Index nc = detail::cells(dm, level);
  detail::need(f, level, dm.n_r(), nc);
  detail::need(u, level, dm.n_r(), nc);
  detail::DevField df(dm, level), du(dm, level);
  df.up(f, nc);
  du.up(u, nc);
  check_ref(tpmg_vcycle(dm.get(), df.f, du.f), dm.context());
  du.down(u, level, dm.n_r(), nc);
}

// measure_cycle_rate(m, f, n_cycles), multigrid.hpp:302-321
inline double measure_cycle_rate(const DeviceMultigrid& dm, const tpmg::Field<double>& f,
                                 int n_cycles) {
  const int L = dm.finest_level();
  const tpmg::Index nc = detail::cells(dm, L);
  detail::need(f, L, dm.n_r(), nc);
  detail::DevField df(dm, L);
  df.up(f, nc);
  double rate = 0.0;
  check_ref(tpmg_measure_cycle_rate(dm.get(), df.f, n_cycles, &rate), dm.context());
  return rate;
}

}  // namespace ref
}  // namespace tpmg_b200
