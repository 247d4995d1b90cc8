/*
 * tpmg_b200.h -- C-ABI drop-in boundary of the B200-native tensor-product
 * multigrid (TPMG) hot path: matrix-free operator apply, vertical line
 * smoother, inter-grid transfers, V-cycle and the PCG driver, all fp64 and
 * device resident on sm_100a.
 *
 * The reference (arXiv 1408.2981, `proj/include/tpmg/`) is a header-only C++20
 * template library with no FFI of its own; every entry point below names the
 * reference function it replaces (path:line relative to the reference root).
 * Conventions carried over from the reference:
 *   - levels are numbered like MultigridHierarchy (multigrid.hpp:207-235):
 *     0 = coarsest ... n_levels-1 = finest;
 *   - the reference's exception taxonomy (types.hpp:24-58) becomes the
 *     tpmg_status return code, nothing is thrown across the ABI;
 *   - fields are one scalar per (column, level); on the host the caller picks
 *     the reference's k-fastest order (discretization.hpp:106-120, Field) or
 *     the device's x-fastest order [k][y][x]; conversion is a permutation;
 *   - horizontal grid: doubly periodic Cartesian nx*ny, cell (i,j) = j*nx+i,
 *     neighbour order W,E,S,N (the Cartesian restatement of the icosahedral
 *     neighbour tables, geometry.hpp:51-53); edge ids: east edge of cell c is
 *     c, north edge of cell c is nx*ny + c.
 * Ownership: handles are owned by the library; host buffers are only borrowed
 * for the duration of a call.  All calls are stream ordered on the context's
 * stream and synchronous at return.  A context is not shared across threads.
 */
#ifndef TPMG_B200_H
#define TPMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPMG_ABI_VERSION 2

typedef enum tpmg_status {
  TPMG_OK = 0,
  TPMG_E_CONFIG = 1,      /* config_error      types.hpp:24-28 */
  TPMG_E_SHAPE = 2,       /* shape_error       types.hpp:30-34 */
  TPMG_E_NONFINITE = 3,   /* nonfinite_error   types.hpp:36-40 */
  TPMG_E_FINGERPRINT = 4, /* fingerprint_error types.hpp:42-46 */
  TPMG_E_SINGULAR = 5,    /* singular_error    types.hpp:48-52 (zero Thomas pivot) */
  TPMG_E_CAP = 6,         /* cap_error         types.hpp:54-58 */
  TPMG_E_CUDA = 7,        /* CUDA runtime failure / extension missing */
  TPMG_E_NCCL = 8,        /* NCCL failure */
  TPMG_NOT_CONVERGED = 9, /* Krylov: max_iter reached */
  TPMG_BREAKDOWN = 10,    /* Krylov: p.q <= 0 / rho == 0 */
  TPMG_DIVERGED = 11      /* Krylov: |r|/|r0| > 1e4 */
} tpmg_status;

typedef enum tpmg_layout {
  TPMG_LAYOUT_K_FASTEST = 0, /* reference Field order: (k, column), k fastest */
  TPMG_LAYOUT_X_FASTEST = 1  /* device order [k][y][x] */
} tpmg_layout;

/* SmootherKind, relaxation.hpp:10. Only block_jacobi is data parallel; the
 * device rejects block_sor with TPMG_E_CONFIG (sequential by contract,
 * relaxation.hpp:13-16). */
typedef enum tpmg_smoother_kind {
  TPMG_SMOOTHER_BLOCK_JACOBI = 0,
  TPMG_SMOOTHER_BLOCK_SOR = 1
} tpmg_smoother_kind;

/* ProlongationKind / RestrictionKind, multigrid.hpp:10-11. */
typedef enum tpmg_prolongation_kind { TPMG_PROLONG_LINEAR = 0, TPMG_PROLONG_INJECTION = 1 } tpmg_prolongation_kind;
typedef enum tpmg_restriction_kind { TPMG_RESTRICT_SUMMATION = 0, TPMG_RESTRICT_TRANSPOSE = 1 } tpmg_restriction_kind;

typedef struct tpmg_context_s* tpmg_context;
typedef struct tpmg_hierarchy_s* tpmg_hierarchy;
typedef struct tpmg_field_s* tpmg_field;

/* One context per GPU / rank.  world_size == 1 needs no NCCL id. */
typedef struct tpmg_context_params {
  int device;          /* CUDA ordinal; -1 = keep the current device */
  int rank;            /* this process' rank */
  int world_size;      /* number of ranks (GPUs) */
  int px, py;          /* process grid, px*py == world_size; rank = ry*px + rx */
  const void* nccl_id; /* 128-byte ncclUniqueId produced by rank 0, or NULL */
} tpmg_context_params;

/* Horizontal (Cartesian, doubly periodic) x vertical grid.
 * VerticalGrid, geometry.hpp:98-111; flat analogue: faces z_0 < ... < z_nz,
 * volumes dz_k = z_{k+1} - z_k, Neumann masks on both boundary faces. */
typedef struct tpmg_grid_desc {
  int64_t nx, ny;        /* GLOBAL cell counts */
  double hx, hy;         /* cell widths (areas hx*hy; edge factors hy/hx, hx/hy) */
  int64_t nz;            /* vertical cells */
  const double* z_faces; /* nz+1 strictly increasing face heights */
} tpmg_grid_desc;

/* FactorizedProfileSet, profiles.hpp:196-210: four vertical vectors and four
 * horizontal scalar fields.  Horizontal arrays are GLOBAL (nx*ny / 2*nx*ny);
 * each rank extracts its tile. */
typedef struct tpmg_factorized_profiles {
  const double* beta_r;    /* nz   */
  const double* alpha_s_r; /* nz   */
  const double* alpha_r_r; /* nz+1 */
  const double* xi_r_r;    /* nz+1, NULL = no vertical advection */
  const double* beta_s;    /* nx*ny   */
  const double* alpha_r_s; /* nx*ny   */
  const double* xi_r_s;    /* nx*ny, NULL = no vertical advection */
  const double* alpha_s_s; /* 2*nx*ny: east edges, then north edges */
} tpmg_factorized_profiles;

/* Full (non-factorised) profiles, the reference's ProfileSet (profiles.hpp:182-192): dense
 * arrays in the reference's Matrix order (column-major, level k fastest).  GLOBAL, like the
 * factorised horizontal arrays. */
typedef struct tpmg_full_profiles {
  const double* beta;    /* nz x nx*ny                                    */
  const double* alpha_s; /* nz x 2*nx*ny: east edges, then north edges    */
  const double* alpha_r; /* (nz+1) x nx*ny                                */
  const double* xi_r;    /* (nz+1) x nx*ny, NULL = no vertical advection  */
} tpmg_full_profiles;

/* Coefficient storage of a hierarchy (HattedComponent, discretization.hpp:32-48). */
typedef enum tpmg_coef_mode {
  TPMG_COEF_FACTORIZED = 0, /* TPMG(tensor): every component vertical x horizontal      */
  TPMG_COEF_PARTIAL = 1,    /* TPMG(partial): alpha_r dense (MixedProfileSet)            */
  TPMG_COEF_FULL = 2        /* TPMG(full): every component dense (ProfileSet)            */
} tpmg_coef_mode;

/* Arguments of build_hierarchy_coefficients, multigrid.hpp:242-272. */
typedef struct tpmg_mg_config {
  int smoother;     /* tpmg_smoother_kind */
  double relax;     /* SmootherConfig::relax, must lie in (0,2) (relaxation.hpp:67-68) */
  int prolongation; /* tpmg_prolongation_kind */
  int restriction;  /* tpmg_restriction_kind */
  int nu_pre;       /* sweeps on refined levels; coarsest is forced to 1+0 (multigrid.hpp:269-270) */
  int nu_post;
  int depth;        /* number of levels; 0 = coarsen while every tile dim stays even and >= 2 */
  /* Coarse-grid agglomeration of a decomposed run (world > 1, or the loopback test mode): every
   * level whose GLOBAL grid has at most `agglomerate` columns is kept whole on every rank and
   * the bottom of the V-cycle is solved redundantly there -- the restricted right-hand side is
   * all-gathered once per V-cycle (NCCL all-gather, or each rank's tile stored straight into
   * every rank's copy through CUDA-IPC peer mappings) and each rank prolongates from its copy.
   * The levels are then those of the GLOBAL grid (depth 0: coarsen it while it stays even and
   * >= 4 per dimension), so the solve is bitwise the one-rank solve of the same problem and
   * the coarse grid does not grow with the rank count.  0 = off (every level decomposed, the
   * reference's one-coarse-cell-per-process layout).  Ignored on one rank. */
  int agglomerate;
} tpmg_mg_config;

/* ---- context ------------------------------------------------------------------------------ */
const char* tpmg_status_string(int status);
int tpmg_abi_version(void);
/* Fills 128 bytes with a fresh ncclUniqueId (rank 0 calls this, then broadcasts). */
int tpmg_nccl_unique_id(void* out128);
int tpmg_init(const tpmg_context_params* params, tpmg_context* out);
/* The same context with the CUDA-IPC transport instead of NCCL: the ranks of one node (on
 * distinct GPUs, or several processes sharing one GPU) write their halo faces straight into the
 * neighbours' receive buffers (cudaIpcMemHandle mappings, exchanged at hierarchy creation) and
 * reduce dot products in rank order through the POSIX shared-memory segment "/tpmg_<session>"
 * (rank 0 creates it; every rank passes the same session string; removed once all attached).
 * Each exchange and reduction is ordered by host barriers around stream synchronisations -- no
 * kernel waits on another rank -- so iterations are not captured into CUDA graphs.  Hierarchy
 * creation and destruction are collective.  world_size >= 2; nccl_id is ignored. */
int tpmg_init_ipc(const tpmg_context_params* params, const char* session, tpmg_context* out);
int tpmg_finalize(tpmg_context ctx);
const char* tpmg_last_error(tpmg_context ctx);
/* The cudaStream_t every call of this context is ordered on (for external CUDA-event timing). */
int tpmg_context_stream(tpmg_context ctx, void** stream);

/* ---- decomposition (pure host logic, no device needed) ------------------------------------ */
/* 2D horizontal block decomposition used by tpmg_hier_create: full columns per rank, tiles
 * aligned so the 2x2 children of every coarse cell stay on one rank.
 * Fills n_levels and, per level l (0 = coarsest, up to max_levels entries each):
 * local tile nx[l], ny[l], global offset x0[l], y0[l]; neighbour ranks nbr[0..3] = W,E,S,N
 * (a rank is its own neighbour along a dimension with one rank: periodic self wrap). */
int tpmg_plan_decomposition(int64_t nx, int64_t ny, int px, int py, int rank, int depth,
                            int max_levels, int* n_levels, int64_t* tile_nx, int64_t* tile_ny,
                            int64_t* x0, int64_t* y0, int* nbr);

/* ---- hierarchy: build_hierarchy_coefficients (multigrid.hpp:242-272) ---------------------- */
/* assemble_hatted (discretization.hpp:144-184) on every level after
 * restrict_profiles (multigrid.hpp:158-201); uploads the result, immutable. */
int tpmg_hier_create(tpmg_context ctx, const tpmg_grid_desc* grid,
                     const tpmg_factorized_profiles* profiles, double omega,
                     const tpmg_mg_config* cfg, tpmg_hierarchy* out);
/* build_hierarchy_coefficients with a MixedProfileSet (profiles.hpp:225-233,
 * build_partial_factorization :237-249): `profiles` supplies beta, alpha_s and xi_r (its
 * alpha_r parts are unused), `alpha_r` is the full (nz+1) x nx*ny field (k fastest). */
int tpmg_hier_create_partial(tpmg_context ctx, const tpmg_grid_desc* grid,
                             const tpmg_factorized_profiles* profiles, const double* alpha_r,
                             double omega, const tpmg_mg_config* cfg, tpmg_hierarchy* out);
/* build_hierarchy_coefficients with a full ProfileSet: every hatted component dense per
 * level (assemble_hatted, discretization.hpp:104-141; restrict_profiles multigrid.hpp:146-156).
 * The device reads +8 B/DOF (partial) or +48 B/DOF (+56 with xi) of coefficients per
 * operator row: alpha_s is stored per cell for its four edges, so no coefficient halo. */
int tpmg_hier_create_full(tpmg_context ctx, const tpmg_grid_desc* grid,
                          const tpmg_full_profiles* profiles, double omega,
                          const tpmg_mg_config* cfg, tpmg_hierarchy* out);
int tpmg_hier_coef_mode(tpmg_hierarchy h, int* mode);
/* build_hierarchy_coefficients' result on an arbitrary (indirect) grid hierarchy, e.g. the
 * reference's icosahedral GridHierarchy (geometry.hpp:41-91): per level (coarsest first)
 * ncells / nedges, neighbour and edge tables ncells x nnb (entry T*nnb + j = the reference's
 * Index3X neighbors(j, T) / cell_edges(j, T)), the child table of every level but the coarsest
 * (entry Tc*nchild + j on the next coarser level's cell Tc = GridHierarchy::child_of), the
 * prolongation's corner rule prol_d1/prol_d2 (-1 = centre child, multigrid.hpp:88-95), and the
 * separable hatted coefficients (vertical bv, sv nz; av, xv nz+1; horizontal bh, ah, xh per cell
 * and sh per edge, discretization.hpp:32-48).  One rank.  Fields of such a hierarchy are
 * [k][cell] on the device; nx = ncells, ny = 1 in tpmg_hier_level_shape. */
int tpmg_hier_create_generic(tpmg_context ctx, int n_levels, int nz, int nnb, int nchild,
                             const int64_t* ncells, const int64_t* nedges,
                             const int64_t* const* nbr, const int64_t* const* cedge,
                             const int64_t* const* children, const int* prol_d1,
                             const int* prol_d2, const double* bv, const double* sv,
                             const double* av, const double* xv, const double* const* bh,
                             const double* const* ah, const double* const* xh,
                             const double* const* sh, double relax, int prolongation,
                             int restriction, int nu_pre, int nu_post, tpmg_hierarchy* out);
int tpmg_hier_destroy(tpmg_hierarchy h);
int tpmg_hier_n_levels(tpmg_hierarchy h, int* n_levels);
/* Local tile shape and global offset of `level` on this rank. */
int tpmg_hier_level_shape(tpmg_hierarchy h, int level, int64_t* nx, int64_t* ny, int64_t* nz,
                          int64_t* x0, int64_t* y0);
/* Hatted coefficients of `level` (HattedCoefficients, discretization.hpp:53-67), tile local:
 * bh/ah/xh: nx*ny; sh: 2*nx*ny (east, north); bv/sv: nz; av/xv: nz+1.  Any pointer may be NULL. */
int tpmg_hier_get_coefficients(tpmg_hierarchy h, int level, double* bh, double* ah, double* xh,
                               double* sh, double* bv, double* sv, double* av, double* xv);

/* ---- fields: Field (discretization.hpp:106-120), device resident [k][y][x] ---------------- */
int tpmg_field_create(tpmg_hierarchy h, int level, tpmg_field* out);
int tpmg_field_destroy(tpmg_field f);
int tpmg_field_level(tpmg_field f, int* level);
int tpmg_field_upload(tpmg_field f, const double* host, int layout);
int tpmg_field_download(tpmg_field f, double* host, int layout);
int tpmg_field_fill(tpmg_field f, double value);
int tpmg_field_copy(tpmg_field dst, tpmg_field src);
/* Raw device pointer ([k][y][x], nx*ny*nz doubles) for zero-copy interop. */
int tpmg_field_device_ptr(tpmg_field f, double** out);

/* ---- hot path ------------------------------------------------------------------------------ */
/* apply_operator, discretization.hpp:262-278: y = A u on u's level. */
int tpmg_apply(tpmg_hierarchy h, tpmg_field u, tpmg_field y);
/* r = f - A u (multigrid.hpp:285-287). */
int tpmg_residual(tpmg_hierarchy h, tpmg_field f, tpmg_field u, tpmg_field r);
/* smooth, relaxation.hpp:63-97 (block_jacobi): `sweeps` line-Jacobi sweeps on u. */
int tpmg_smooth(tpmg_hierarchy h, tpmg_field u, tpmg_field f, int sweeps);
/* restrict_field / restrict_field_transpose, multigrid.hpp:29-69 (kind from the config). */
int tpmg_restrict(tpmg_hierarchy h, tpmg_field fine, tpmg_field coarse);
/* prolongate_field + `u +=`, multigrid.hpp:74-100, :294-295 (kind from the config). */
int tpmg_prolong_add(tpmg_hierarchy h, tpmg_field coarse, tpmg_field fine);
/* prolongate_field alone: fine = P coarse. */
int tpmg_prolong(tpmg_hierarchy h, tpmg_field coarse, tpmg_field fine);
/* The reference's transfer entry points with an explicit kind, independent of the hierarchy's
 * TransferConfig: restrict_field (TPMG_RESTRICT_SUMMATION, multigrid.hpp:29-43) /
 * restrict_field_transpose (TPMG_RESTRICT_TRANSPOSE, :46-69); prolongate_field(..., kind)
 * (:74-100), with add != 0 fine += P coarse. */
int tpmg_restrict_kind(tpmg_hierarchy h, tpmg_field fine, tpmg_field coarse, int restriction);
int tpmg_prolong_kind(tpmg_hierarchy h, tpmg_field coarse, tpmg_field fine, int prolongation,
                      int add);
/* v_cycle(m, finest, f, u), multigrid.hpp:276-299: one V-cycle, u updated in place. */
int tpmg_vcycle(tpmg_hierarchy h, tpmg_field f, tpmg_field u);
/* measure_cycle_rate, multigrid.hpp:302-321. */
int tpmg_measure_cycle_rate(tpmg_hierarchy h, tpmg_field f, int n_cycles, double* rate);
/* Global (all-reduced) dot product and Euclidean norm (Field::norm, discretization.hpp:27). */
int tpmg_dot(tpmg_hierarchy h, tpmg_field a, tpmg_field b, double* out);
int tpmg_norm(tpmg_hierarchy h, tpmg_field a, double* out);

/* PCG preconditioned by one V-cycle from a zero guess (SPEC.md:387-448 conventions):
 * x0 = 0 (x is overwritten), stop when |r_k|/|r_0| <= tol, divergence at > 1e4.
 * res_hist (may be NULL) receives |r_0| .. |r_iters| (max_iter+1 entries);
 * solve_status receives TPMG_OK / NOT_CONVERGED / BREAKDOWN / DIVERGED.
 * The return value is TPMG_OK unless the call itself failed. */
int tpmg_pcg(tpmg_hierarchy h, tpmg_field f, tpmg_field x, double tol, int max_iter,
             double* res_hist, int* iters, int* solve_status);

/* Preconditioned Richardson (richardson_solve):
 * x_{k+1} = x_k + M^{-1}(f - A x_k), M^{-1} = mu V-cycles on A e = r from e = 0, x_0 = 0.
 * Same history / status conventions as tpmg_pcg (divergence guard 1e4). */
int tpmg_richardson(tpmg_hierarchy h, tpmg_field f, tpmg_field x, double tol, int max_iter,
                    int mu, double* res_hist, int* iters, int* solve_status);

/* Right-preconditioned BiCGStab, classical single stabilisation (bicgstab_solve,
 * SPEC.md:412-420, design decisions :443-447): exactly two preconditioner and two operator
 * applications per full iteration; rho-breakdown (|r^.r| < 1e-30 |r_0|^2) -> TPMG_BREAKDOWN;
 * convergence is also tested on the intermediate residual s (half step). x_0 = 0. */
int tpmg_bicgstab(tpmg_hierarchy h, tpmg_field f, tpmg_field x, double tol, int max_iter,
                  int mu, double* res_hist, int* iters, int* solve_status);

/* Preconditioner and operator applications of the last tpmg_richardson / tpmg_bicgstab call
 * (the SPEC's per-iteration cost contract). */
int tpmg_solver_counts(tpmg_hierarchy h, int64_t* n_precond, int64_t* n_matvec);

/* End-to-end solve from host memory: upload f (layout), PCG, download x. */
int tpmg_pcg_host(tpmg_hierarchy h, const double* f_host, double* x_host, int layout, double tol,
                  int max_iter, double* res_hist, int* iters, int* solve_status);

/* End-to-end solves of `count` independent right-hand sides f_hosts[i] -> x_hosts[i] (layout),
 * the host<->device transfers overlapped with the solves: while right-hand side i is solved,
 * right-hand side i+1 is uploaded and solution i-1 downloaded on a copy stream (double-buffered
 * device fields; pinned host buffers for the copies to overlap).  Each solve is tpmg_pcg's, so
 * the results equal `count` tpmg_pcg_host calls bit for bit.  res_hist: count x (max_iter+1)
 * or NULL; iters, solve_status: count entries. */
int tpmg_pcg_host_batch(tpmg_hierarchy h, int count, const double* const* f_hosts,
                        double* const* x_hosts, int layout, double tol, int max_iter,
                        double* res_hist, int* iters, int* solve_status);

/* ---- profile files: save_profiles / load_profiles (profile_io.hpp:125-242) ------------------ */
/* The reference's JSON profile format, byte for byte as its writer (nlohmann dump(1): keys
 * sorted, shortest round-trip doubles, non-finite -> null): format_version 1, kind "factorized" |
 * "full", grid header {fingerprint, level, n_r, type}, arrays column-major with k fastest, as
 * decimal numbers or "base64-f64le".  Host-only, no context needed.
 * Arrays travel PACKED, back to back in this order (nc cells, ne edges):
 *   factorized: beta_r nz, alpha_s_r nz, alpha_r_r nz+1, xi_r_r nz+1,
 *               beta_s nc, alpha_r_s nc, xi_r_s nc, alpha_s_s ne
 *   full:       beta nz*nc, alpha_s nz*ne, alpha_r (nz+1)*nc, xi_r (nz+1)*nc
 * (each dense array k fastest, i.e. entry c*rows + k).  Load errors follow load_profiles, checked
 * in its order: unreadable file -> TPMG_E_CONFIG; wrong grid -> TPMG_E_FINGERPRINT; n_r, level,
 * kind, array length or malformed JSON -> TPMG_E_SHAPE; non-finite, null or non-numeric entry ->
 * TPMG_E_NONFINITE; output buffer too small -> TPMG_E_CAP. */
typedef enum tpmg_profile_kind { TPMG_PROFILE_FACTORIZED = 0, TPMG_PROFILE_FULL = 2 } tpmg_profile_kind;

/* The grid header a file is written for / validated against (detail::grid_header,
 * profile_io.hpp:114-121).  nx, ny > 0 are written as extra header keys (Cartesian grids). */
typedef struct tpmg_profile_grid {
  const char* type;     /* "icosahedral", "cartesian", ... */
  uint64_t fingerprint; /* grid_fingerprint, geometry.hpp:335-351 */
  int64_t level;
  int64_t n_r, n_cells, n_edges;
  int64_t nx, ny;       /* 0 = not written */
} tpmg_profile_grid;

/* grid_fingerprint (geometry.hpp:335-351): FNV-1a 64 over the bytes of the cell centres,
 * centers[3*c + i] (the reference's Matrix3X, column-major). */
uint64_t tpmg_grid_fingerprint(const double* centers, int64_t n_cells);
/* The Cartesian analogue: centres ((i+1/2) hx, (j+1/2) hy, 0) in cell order j*nx + i. */
uint64_t tpmg_grid_fingerprint_cartesian(const tpmg_grid_desc* grid);
int64_t tpmg_profile_packed_size(int kind, int64_t n_cells, int64_t n_edges, int64_t n_r);
/* Any grid (e.g. the reference's icosahedral levels, with tpmg_hier_create_generic). */
int tpmg_profile_save_grid(const char* path, const tpmg_profile_grid* grid, int kind,
                           const double* packed, int base64);
int tpmg_profile_load_grid(const char* path, const tpmg_profile_grid* grid, int* kind,
                           double* packed, int64_t capacity);
/* The Cartesian grid of tpmg_hier_create: type "cartesian", level 0, n_cells = nx*ny,
 * n_edges = 2*nx*ny (east edges, then north edges), fingerprint as above. */
int tpmg_profile_save(const char* path, const tpmg_grid_desc* grid, int kind, const double* packed,
                      int base64);
int tpmg_profile_load(const char* path, const tpmg_grid_desc* grid, int* kind, double* packed,
                      int64_t capacity);
/* Message of the last failed tpmg_profile_* call on this thread. */
const char* tpmg_profile_last_error(void);

/* (The reference's own icosahedral test problem is set up by test infrastructure,
 * oracle/icosa_setup.cpp, and reaches the device through tpmg_hier_create_generic.) */

/* ---- instrumentation ------------------------------------------------------------------------ */
/* Number of kernels this library launched on the context since creation. */
int tpmg_kernel_launch_count(tpmg_context ctx, int64_t* out);
/* NCCL API calls (sends, receives, collectives, group brackets; captured ones counted at capture)
 * this process has issued: 0 on a one-rank context, whose halos are periodic self views. */
int tpmg_nccl_call_count(int64_t* out);
/* Kernel ids for tpmg_time_kernel. */
typedef enum tpmg_kernel_id {
  TPMG_K_APPLY = 0,           /* y = A u                                  */
  TPMG_K_JACOBI = 1,          /* one line-Jacobi sweep, nonzero guess     */
  TPMG_K_JACOBI_ZERO = 2,     /* one line-Jacobi sweep from a zero guess  */
  TPMG_K_RESID_RESTRICT = 3,  /* coarse = R (f - A u) as used by the V-cycle */
  TPMG_K_PROLONG_ADD = 4,     /* fine += P coarse                         */
  TPMG_K_RESTRICT = 5,        /* coarse = R fine                          */
  TPMG_K_RESIDUAL = 6,        /* r = f - A u                              */
  TPMG_K_PCG_DIRECTION = 7,   /* fused PCG pass: x += a p; p = z + b p; A p and p.(A p) */
  TPMG_K_PCG_RUPDATE = 8,     /* fused PCG pre-sweep: r -= a A p, |r|^2, z = smoother(r) */
  TPMG_K_PCG_POSTSWEEP = 9,   /* fused PCG post-sweep: z = smoother(u) and the r.z partials */
  TPMG_K_REDUCE = 10          /* (probe only) fixed-order final sum of a dot's partials   */
} tpmg_kernel_id;
/* Average device time (CUDA events on the library's stream) of `reps` back-to-back launches
 * of one hot-path kernel on `level` (transfers: `level` is the fine level), on internal
 * scratch fields filled with deterministic data.  Instrumentation for bench.py. */
int tpmg_time_kernel(tpmg_hierarchy h, int kernel_id, int level, int reps, double* avg_ms);
/* Kernel probes: with `enable` != 0, every later tpmg_pcg solve brackets its finest-level
 * launches of TPMG_K_PCG_DIRECTION, _PCG_RUPDATE, _PCG_POSTSWEEP, _RESID_RESTRICT and
 * _PROLONG_ADD with CUDA events on the library stream (recorded into the iteration's CUDA
 * graph as external event nodes) and accumulates their device durations; enabling resets the
 * totals.  tpmg_kernel_probe_read returns the total milliseconds and the launch count of one
 * kernel id since then.  Instrumentation for bench.py (live durations inside the timed solves). */
int tpmg_kernel_probe(tpmg_hierarchy h, int enable);
int tpmg_kernel_probe_read(tpmg_hierarchy h, int kernel_id, double* total_ms, int64_t* launches);
/* Enable/disable CUDA-graph replay of the PCG iteration (default on). */
int tpmg_set_use_graphs(tpmg_hierarchy h, int enable);

#ifdef __cplusplus
}
#endif
#endif /* TPMG_B200_H */
