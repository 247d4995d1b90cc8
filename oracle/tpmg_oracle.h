/*
 * tpmg_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference TPMG hot path (arXiv 1408.2981,
 * proj/include/tpmg/) used as the parity checker for the sm_100a path and
 * as the CPU baseline in bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline / --impl reference) may load it; the product library
 * (paper_1408_2981_b200/) never links, loads or calls it.
 *
 * The oracle works on explicit neighbour / edge / child tables exactly like the
 * reference's HorizontalGrid (geometry.hpp:41-71) and GridHierarchy
 * (geometry.hpp:75-91), so the same code runs
 *   - the doubly periodic Cartesian problem of BASELINE.json (tables generated
 *     here: 4 neighbours W,E,S,N, 4 children a+2b), and
 *   - arbitrary tables supplied by the caller (tpmgo_generic_create), e.g. the
 *     reference's own icosahedral hierarchy exported by oracle/_ref, which is
 *     how the restatement is pinned against the reference itself.
 * Field layout is the reference's: column-major n_r x n_cells, k fastest
 * (discretization.hpp:106-120).
 *
 * Parity status: see DESIGN.md "Oracle pinning".
 */
#ifndef TPMG_ORACLE_H
#define TPMG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tpmgo_hier_s* tpmgo_hier;

const char* tpmgo_last_error(void);

/* Cartesian doubly periodic problem: global nx*ny, cell widths hx, hy,
 * vertical faces z[0..nz], factorised profiles (profiles.hpp:196-210, same
 * array conventions as include/tpmg_b200.h), omega, multigrid config.
 * Returns 0 or a tpmg_status code. */
int tpmgo_cart_create(int64_t nx, int64_t ny, double hx, double hy, int64_t nz,
                      const double* z_faces, const double* beta_r, const double* alpha_s_r,
                      const double* alpha_r_r, const double* xi_r_r, const double* beta_s,
                      const double* alpha_r_s, const double* xi_r_s, const double* alpha_s_s,
                      double omega, double relax, int prolongation, int restriction, int nu_pre,
                      int nu_post, int depth, int threads, tpmgo_hier* out);

/* Partial (mode 1: dense alpha_r, MixedProfileSet) or full (mode 2: ProfileSet; the factorised
 * pointers may be NULL) coefficients on the same Cartesian problem.  Dense inputs in the
 * reference's Matrix order (k fastest): beta nz x ncells, alpha_s nz x 2 ncells (east, north),
 * alpha_r / xi_r (nz+1) x ncells (xi_r may be NULL). */
int tpmgo_cart_create_dense(int mode, const double* beta, const double* alpha_s,
                            const double* alpha_r, const double* xi_r, int64_t nx, int64_t ny,
                            double hx, double hy, int64_t nz, const double* z,
                            const double* beta_r, const double* alpha_s_r,
                            const double* alpha_r_r, const double* xi_r_r, const double* beta_s,
                            const double* alpha_r_s, const double* xi_r_s,
                            const double* alpha_s_s, double omega, double relax,
                            int prolongation, int restriction, int nu_pre, int nu_post,
                            int depth, int threads, tpmgo_hier* out);

/* Generic tables (one entry per level, coarsest first).  Per level l:
 * ncells[l], nedges[l]; nbr[l] / cedge[l]: ncells*nnb Index, entry T*nnb+d
 * (= Index3X neighbors(d,T) column-major); children[l] for l>=1: ncells[l-1]*nchild,
 * entry Tc*nchild+j = fine cell (GridHierarchy::child_of); colinear edge tables are not
 * needed (hatted coefficients are given directly).  prol_d1/prol_d2[j]: the two
 * neighbour directions blended into corner child j, or -1 for a centre child
 * (prolongate_field, multigrid.hpp:74-100).  Hatted coefficients per level
 * (separable, HattedComponent discretization.hpp:32-48): bv,sv (nz), av,xv (nz+1) shared
 * by all levels; bh,ah,xh[l] (ncells), sh[l] (nedges). */
int tpmgo_generic_create(int n_levels, int64_t nz, int nnb, int nchild, const int64_t* ncells,
                         const int64_t* nedges, const int64_t* const* nbr,
                         const int64_t* const* cedge, const int64_t* const* children,
                         const int* prol_d1, const int* prol_d2, const double* bv,
                         const double* sv, const double* av, const double* xv,
                         const double* const* bh, const double* const* ah,
                         const double* const* xh, const double* const* sh, double relax,
                         int prolongation, int restriction, int nu_pre, int nu_post, int threads,
                         tpmgo_hier* out);

void tpmgo_destroy(tpmgo_hier h);
int tpmgo_n_levels(tpmgo_hier h);
int64_t tpmgo_n_cells(tpmgo_hier h, int level);
int64_t tpmgo_nz(tpmgo_hier h);
int tpmgo_set_threads(tpmgo_hier h, int threads);
/* Reduction order of the PCG dots: -1 = the device's rule (default), 0 = plain, 1 = fused. */
int tpmgo_set_pcg_fused(tpmgo_hier h, int mode);
/* 1 (default): PCG dots in the device's reduction order (parity).  0: plain chunked dots and
 * element-wise updates on the worker threads (CPU-baseline timing). */
int tpmgo_set_device_order(tpmgo_hier h, int on);
/* Mirror of the device's TPMG_JACOBI_T4 switch (two-columns-per-thread smoother). */
int tpmgo_set_t4(tpmgo_hier h, int on);

/* Hatted coefficients of a level (assemble_hatted, discretization.hpp:144-184). */
int tpmgo_get_coefficients(tpmgo_hier h, int level, double* bh, double* ah, double* xh,
                           double* sh, double* bv, double* sv, double* av, double* xv);

/* Column blocks of one cell (build_column, discretization.hpp:235-251): diag, upper, lower
 * (nz each) and neighbor (nz*nnb, column d contiguous). */
int tpmgo_build_column(tpmgo_hier h, int level, int64_t cell, double* diag, double* upper,
                       double* lower, double* neighbor);

/* Thomas solve, relaxation.hpp:37-52 (in place on x). */
int tpmgo_thomas(int64_t n, const double* diag, const double* upper, const double* lower,
                 double* x);

/* apply_operator, discretization.hpp:262-278. */
int tpmgo_apply(tpmgo_hier h, int level, const double* u, double* y);
/* r = f - A u, multigrid.hpp:285-287. */
int tpmgo_residual(tpmgo_hier h, int level, const double* f, const double* u, double* r);
/* smooth (block_jacobi), relaxation.hpp:63-97. */
int tpmgo_smooth(tpmgo_hier h, int level, double* u, const double* f, int sweeps);
/* restrict_field / restrict_field_transpose (kind from the hierarchy), multigrid.hpp:29-69. */
int tpmgo_restrict(tpmgo_hier h, int coarse_level, const double* fine, double* coarse);
/* prolongate_field (kind from the hierarchy), multigrid.hpp:74-100. */
int tpmgo_prolong(tpmgo_hier h, int coarse_level, const double* coarse, double* fine);
/* v_cycle on `level`, multigrid.hpp:276-299. */
int tpmgo_vcycle(tpmgo_hier h, int level, const double* f, double* u);
/* measure_cycle_rate, multigrid.hpp:302-321. */
int tpmgo_measure_cycle_rate(tpmgo_hier h, const double* f, int n_cycles, double* rate);
/* PCG with one V-cycle preconditioner (SPEC.md:387-448 conventions). */
int tpmgo_pcg(tpmgo_hier h, const double* f, double* x, double tol, int max_iter,
              double* res_hist, int* iters, int* solve_status);
int tpmgo_pcg_timed(tpmgo_hier h, const double* f, double* x, double tol, int max_iter,
                    double* res_hist, double* seconds, int* iters, int* solve_status);
/* Preconditioned Richardson / right-preconditioned BiCGStab, mu V-cycles per
 * preconditioner application, x0 = 0; operation order of the device drivers. */
int tpmgo_richardson(tpmgo_hier h, const double* f, double* x, double tol, int max_iter, int mu,
                     double* res_hist, int* iters, int* solve_status);
int tpmgo_bicgstab(tpmgo_hier h, const double* f, double* x, double tol, int max_iter, int mu,
                   double* res_hist, int* iters, int* solve_status);
/* Deterministic dot product used by the oracle's PCG. */
double tpmgo_dot(int64_t n, const double* a, const double* b);

#ifdef __cplusplus
}
#endif
#endif
