// tpmg_b200.hpp -- header-only C++ adapter over the C-ABI (tpmg_b200.h) that restores the
// reference's call shapes (proj/include/tpmg/*.hpp) for device-resident fields:
//
//   reference (CPU, Eigen)                              this adapter (sm_100a)
//   apply_operator(h, grid, u, out)   discr.hpp:262      apply_operator(H, u, out)
//   smooth(h, grid, u, f, cfg, s)     relax.hpp:63       smooth(H, u, f, s)
//   restrict_field(fine, hier, lc)    multigrid.hpp:29   restrict_field(H, fine, coarse)
//   prolongate_field(c, hier, lc, k)  multigrid.hpp:74   prolongate_field(H, coarse, fine)
//   v_cycle(m, L, f, u)               multigrid.hpp:276  v_cycle(H, f, u)
//   measure_cycle_rate(m, f, n)       multigrid.hpp:302  measure_cycle_rate(H, f, n)
//   (SPEC.md:402-419 Krylov driver)                      pcg_solve(H, f, x, tol, max_iter)
//
// Errors are thrown as the reference's exception types (types.hpp:24-58).  Handles are RAII;
// a Hierarchy must not outlive its Context, a Field must not outlive its Hierarchy (the same
// lifetime rule as MultigridHierarchy::grids, multigrid.hpp:203-209).
#pragma once

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tpmg_b200.h"

namespace tpmg_b200 {

struct config_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct shape_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct nonfinite_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct singular_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct device_error : std::runtime_error { using std::runtime_error::runtime_error; };

inline void check(int rc, tpmg_context ctx = nullptr) {
  if (rc == TPMG_OK) return;
  const std::string msg = std::string(tpmg_status_string(rc)) + ": " + tpmg_last_error(ctx);
  switch (rc) {
    case TPMG_E_CONFIG: throw config_error(msg);
    case TPMG_E_SHAPE: throw shape_error(msg);
    case TPMG_E_NONFINITE: throw nonfinite_error(msg);
    case TPMG_E_SINGULAR: throw singular_error(msg);
    default: throw device_error(msg);
  }
}

class Context {
 public:
  explicit Context(int device = 0, int rank = 0, int world = 1, int px = 1, int py = 1,
                   const void* nccl_id = nullptr) {
    tpmg_context_params p{device, rank, world, px, py, nccl_id};
    check(tpmg_init(&p, &ctx_));
  }
  ~Context() { tpmg_finalize(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  tpmg_context get() const { return ctx_; }

 private:
  tpmg_context ctx_ = nullptr;
};

// build_hierarchy_coefficients(profiles, hier, vertical, omega, smoother, transfers, nu_pre,
// nu_post, depth) -- multigrid.hpp:242-272, for the Cartesian grid of tpmg_grid_desc.
class Hierarchy {
 public:
  Hierarchy(const Context& ctx, const tpmg_grid_desc& grid, const tpmg_factorized_profiles& prof,
            double omega, const tpmg_mg_config& cfg)
      : ctx_(ctx.get()) {
    check(tpmg_hier_create(ctx_, &grid, &prof, omega, &cfg, &h_), ctx_);
    check(tpmg_hier_n_levels(h_, &levels_), ctx_);
  }
  ~Hierarchy() { tpmg_hier_destroy(h_); }
  Hierarchy(const Hierarchy&) = delete;
  Hierarchy& operator=(const Hierarchy&) = delete;
  tpmg_hierarchy get() const { return h_; }
  tpmg_context context() const { return ctx_; }
  int finest_level() const { return levels_ - 1; }
  int depth() const { return levels_; }

 private:
  tpmg_context ctx_;
  tpmg_hierarchy h_ = nullptr;
  int levels_ = 0;
};

// Field (discretization.hpp:106-120), device resident.
class Field {
 public:
  Field(const Hierarchy& h, int level) : ctx_(h.context()) {
    check(tpmg_field_create(h.get(), level, &f_), ctx_);
    level_ = level;
  }
  ~Field() { tpmg_field_destroy(f_); }
  Field(const Field&) = delete;
  Field& operator=(const Field&) = delete;
  tpmg_field get() const { return f_; }
  int level() const { return level_; }
  void upload(const double* host, tpmg_layout layout = TPMG_LAYOUT_K_FASTEST) {
    check(tpmg_field_upload(f_, host, layout), ctx_);
  }
  void download(double* host, tpmg_layout layout = TPMG_LAYOUT_K_FASTEST) const {
    check(tpmg_field_download(f_, host, layout), ctx_);
  }
  void setZero() { check(tpmg_field_fill(f_, 0.0), ctx_); }

 private:
  tpmg_context ctx_;
  tpmg_field f_ = nullptr;
  int level_ = 0;
};

inline void apply_operator(const Hierarchy& h, const Field& u, Field& out) {
  check(tpmg_apply(h.get(), u.get(), out.get()), h.context());
}
inline void smooth(const Hierarchy& h, Field& u, const Field& f, int sweeps) {
  check(tpmg_smooth(h.get(), u.get(), f.get(), sweeps), h.context());
}
inline void restrict_field(const Hierarchy& h, const Field& fine, Field& coarse) {
  check(tpmg_restrict(h.get(), fine.get(), coarse.get()), h.context());
}
inline void prolongate_field(const Hierarchy& h, const Field& coarse, Field& fine) {
  check(tpmg_prolong(h.get(), coarse.get(), fine.get()), h.context());
}
inline void v_cycle(const Hierarchy& h, const Field& f, Field& u) {
  check(tpmg_vcycle(h.get(), f.get(), u.get()), h.context());
}
inline double measure_cycle_rate(const Hierarchy& h, const Field& f, int n_cycles) {
  double r = 0.0;
  check(tpmg_measure_cycle_rate(h.get(), f.get(), n_cycles, &r), h.context());
  return r;
}

struct ConvergenceHistory {  // SPEC.md:396-399 (res_norm column)
  std::vector<double> res_norm;
  int iterations = 0;
  int status = TPMG_OK;  // TPMG_OK / NOT_CONVERGED / BREAKDOWN / DIVERGED
};

inline ConvergenceHistory pcg_solve(const Hierarchy& h, const Field& f, Field& x, double tol,
                                    int max_iter) {
  ConvergenceHistory c;
  c.res_norm.assign(static_cast<size_t>(max_iter) + 1, 0.0);
  check(tpmg_pcg(h.get(), f.get(), x.get(), tol, max_iter, c.res_norm.data(), &c.iterations,
                 &c.status),
        h.context());
  c.res_norm.resize(static_cast<size_t>(c.iterations) + 1);
  return c;
}

// richardson_solve / bicgstab_solve with mu V-cycles per preconditioner
// application (SolverConfig::mu).
inline ConvergenceHistory richardson_solve(const Hierarchy& h, const Field& f, Field& x,
                                           double tol = 1e-5, int max_iter = 500, int mu = 1) {
  ConvergenceHistory c;
  c.res_norm.assign(static_cast<size_t>(max_iter) + 1, 0.0);
  check(tpmg_richardson(h.get(), f.get(), x.get(), tol, max_iter, mu, c.res_norm.data(),
                        &c.iterations, &c.status),
        h.context());
  c.res_norm.resize(static_cast<size_t>(c.iterations) + 1);
  return c;
}
inline ConvergenceHistory bicgstab_solve(const Hierarchy& h, const Field& f, Field& x,
                                         double tol = 1e-5, int max_iter = 500, int mu = 1) {
  ConvergenceHistory c;
  c.res_norm.assign(static_cast<size_t>(max_iter) + 1, 0.0);
  check(tpmg_bicgstab(h.get(), f.get(), x.get(), tol, max_iter, mu, c.res_norm.data(),
                      &c.iterations, &c.status),
        h.context());
  c.res_norm.resize(static_cast<size_t>(c.iterations) + 1);
  return c;
}

}  // namespace tpmg_b200
