// tpmg_kernels.cuh -- device data views and kernel launchers of the sm_100a hot path.
//
// Device layout of every field: [k][y][x], x fastest (the transpose of the reference's
// k-fastest Field, discretization.hpp:106-120), so a warp covers 32 consecutive x columns
// and every load/store at fixed k is coalesced.  Coefficients are the separable hatted
// factors of discretization.hpp:32-67: four vertical vectors shared by all levels and six
// per-column horizontal scalars (bh, ah, xh and the four edge scalars W,E,S,N), i.e. 48 B
// per column, rebuilt into the column blocks on the fly (build_column, discretization.hpp:
// 235-251).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tpmg {

struct VertCoef {      // HattedComponent::vert of beta, alpha_s, alpha_r, xi_r
  const double* bv;    // nz
  const double* sv;    // nz
  const double* av;    // nz+1
  const double* xv;    // nz+1 (only read when the level has advection)
  // the same, interleaved for one bulk copy into shared memory: vr[k] = {bv_k, sv_k, av_k,
  // av_k+1}, vx[k] = {xv_k, xv_k+1} (nullptr: the kernels stage from the arrays above)
  const double* vr = nullptr;
  const double* vx = nullptr;
};

// Coefficient storage of a level (HattedComponent, discretization.hpp:32-48): factorised
// (TPMG-tensor-product: vertical x horizontal factors), partial (alpha_r hat dense, the rest
// factorised: MixedProfileSet, profiles.hpp:225-233), full (every component dense: ProfileSet).
enum CoefMode { CM_FACT = 0, CM_PARTIAL = 1, CM_FULL = 2,
                // kernel-side only (never a LevelCoef::cm): factorised coefficients whose four
                // edge scalars coincide on the level (LevelCoef::uni): the edge product of a row
                // is formed once instead of four times, same value
                CM_UNI = 3 };
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr bool cm_fact(int cm) { return cm == CM_FACT || cm == CM_UNI; }

struct LevelCoef {     // HattedComponent::horiz, per column of the local tile
  int nx, ny, nz;
  int64_t plane;       // nx*ny
  const double* bh;
  const double* ah;
  const double* xh;
  const double* sw;    // alpha_s hat of the W / E / S / N edge of each column
  const double* se;
  const double* ss;
  const double* sn;
  int cm = CM_FACT;
  // factorised levels: sw == se == ss == sn in every column (isotropic horizontal coefficient on
  // a square grid; then one value for the whole level, the edges being shared)
  bool uni = false;
  // dense components, [k][y][x] like the fields (HattedComponent::dense):
  const double* ard = nullptr;  // alpha_r hat, nz+1 planes (partial, full)
  const double* bd = nullptr;   // beta hat, nz planes (full)
  const double* xid = nullptr;  // xi_r hat, nz+1 planes (full, with advection)
  const double* swd = nullptr;  // alpha_s hat of the W / E / S / N edge of each cell (full)
  const double* sed = nullptr;
  const double* ssd = nullptr;
  const double* snd = nullptr;
  // indirect (unstructured) levels: the reference's HorizontalGrid tables (geometry.hpp:41-71);
  // nbr == nullptr on the Cartesian levels.  plane = number of cells, nx = plane, ny = 1.
  int nnb = 0;
  const int* nbr = nullptr;    // plane x nnb: neighbour j of cell T at nbr[T*nnb + j]
  const int* cedge = nullptr;  // plane x nnb: edge shared with that neighbour
  const double* shg = nullptr; // alpha_s hat horizontal factor per edge
  // coarse levels: the column blocks' Thomas factorisation, fixed for the hierarchy's life
  // (pivot_k and c'_k of thomas_solve_inplace, relaxation.hpp:42-48, [k][y][x]); nullptr: the
  // smoother forms it on the fly
  const double* piv = nullptr;
  const double* cpt = nullptr;
};

// Coarse-to-fine relation of an indirect hierarchy: children of the coarse cells
// (GridHierarchy::child_of) and the prolongation's corner rule (multigrid.hpp:88-95): child j
// blends the coarse neighbours in directions d1[j], d2[j]; d1[j] < 0 marks the centre child.
struct GenRule {
  int nchild;
  int d1[8], d2[8];
};

// Where the neighbour values across each tile face live.  For direction d
// (0=W,1=E,2=S,3=N) the value adjacent to boundary position t (t = y for W/E,
// x for S/N) at level k is p[d][k*sk[d] + t*st[d]].  Single GPU: strided views of
// the field itself (periodic wrap, no copy).  Multi GPU: NCCL-filled halo buffers.
struct Halo {
  const double* p[4];
  int64_t sk[4];
  int64_t st[4];
};

// Two-cell halo with corners (the fused residual + transpose restriction of a decomposed run
// reads u two cells beyond its tile).  Receive buffers, per level k:
//   p[0] W2 [k][j][c] = u(-2+c, j)     p[1] E2 [k][j][c] = u(nx+c, j)      (2*ny per level)
//   p[2] S2 [k][r][i] = u(i, -2+r)     p[3] N2 [k][r][i] = u(i, ny+r)      (2*nx per level)
//   p[4..7] corners SW, SE, NW, NE [k][r][c] = u(-2+c | nx+c, -2+r | ny+r)  (4 per level)
// xs / ys: 0 = that dimension has one rank (periodic wrap onto the tile itself, no buffers).
struct Halo2 {
  const double* p[8];
  int xs, ys;
};
// Where each packed halo piece lands (send buffer, a neighbour's receive buffer through a CUDA-IPC
// mapping, or this rank's own receive buffer in loopback); nullptr: the piece is not exchanged.
// Faces: W, E, S, N (1-cell, [k][j] / [k][i]).  Deep pieces: W, E, S, N, SW, SE, NW, NE in the
// Halo2 layouts of the receiving side (piece W = columns 0..1 -> the west rank's E2, ...).
struct FaceDst {
  double* p[4];
};
struct DeepDst {
  double* p[8];
};
// Ring of 1-cell coefficient scalars around the local tile (a decomposed run's fused residual +
// restriction forms residuals on it): 7 arrays (bh, ah, xh, sw, se, ss, sn) of 2*ny + 2*nx
// entries each, ring index W j, E ny+j, S 2ny+i, N 2ny+nx+i.
constexpr int kRingFields = 7;

enum ApplyMode { APPLY_AU = 0, APPLY_RESID = 1 };

// Deterministic reduction workspace: per-block partials, then one fixed-order pass.
constexpr int kMaxPartials = 8192;

struct Launch {
  cudaStream_t stream;
  int64_t* counter;  // incremented once per kernel launch (instrumentation)
};

// Thrown by a launcher when the launch itself fails (bad configuration); mapped to TPMG_E_CUDA.
struct LaunchError {
  cudaError_t err;
  const char* kernel;
};

Halo self_halo(const double* u, int nx, int ny, int64_t plane);

// y = A u  (apply_operator, discretization.hpp:262-278)  or  y = f - A u.
// If dot_partials != nullptr, per-block partial sums of y.u are written there (count returned
// through *nblocks) for a fused p.q in PCG.
void launch_apply(const Launch& L, const VertCoef& V, const LevelCoef& C, bool xi, int mode,
                  const double* u, const Halo& H, const double* f, double* y,
                  double* dot_partials, int* nblocks);

// PCG work fused into the finest-level line smoother (tiled TMEM path only).  Zero-guess
// sweep: f (== r) is replaced in place by r - alpha q (alpha = s[0]/s[1]) and per-tile |r|^2
// partials are written; nonzero-guess sweep: per-tile partials of f.out (r.z).
struct PcgFuse {
  const double* q = nullptr;
  double* r = nullptr;
  const double* s = nullptr;
  double* partials = nullptr;
  // zero-guess sweep only: q = A p formed in the sweep from a p patch (halo views in the
  // launch's Halo) instead of read from q (then q may be null)
  const double* p = nullptr;
};

// The V-cycle's prolongation fused into the first post-sweep (multigrid.hpp:294-295 then
// :296-297): the sweep's input is u + P ec with k_prolong_flat's linear values and addition
// order, formed on chip (u itself is not modified).  One rank (periodic wrap), linear
// prolongation, Cartesian levels; ec is the next coarser level's correction (cnx x cny x nz).
struct ProSrc {
  const double* ec = nullptr;
  int cnx = 0, cny = 0;
};

// One block-Jacobi line sweep (smooth, relaxation.hpp:77-97): out = u + relax * T^{-1}(f - A u);
// u == nullptr means a zero initial guess.  Zero pivots set bit 1 in *err.  pro: see ProSrc
// (only where jacobi_prolong_fusable holds).
// Thomas factorisation of every column block of a Cartesian level into piv / cpt (C.piv, C.cpt
// must point to nz*plane doubles each); *zero_pivot set when a pivot vanishes (the caller then
// keeps the on-the-fly smoother, which raises the singular error)
void launch_factor_columns(const Launch& L, const VertCoef& V, const LevelCoef& C, bool xi,
                           double* piv, double* cpt, int* zero_pivot);
// Device-side PCG loop state (tpmg_pcg's convergence logic run by k_pcg_check inside a CUDA
// graph while-node: no host round trip per iteration).  exit: 0 continue, 1 converged,
// 2 diverged, 3 breakdown (rho), 4 breakdown (p.q, x not finalised), 5 iteration cap.
struct PcgLoop {
  double r0, tol;
  int max_iter, it, iters, exit;
};
void launch_pcg_check(const Launch& L, const double* scal, double* hist, PcgLoop* st,
                      unsigned long long hw, unsigned long long hi, int use_hi);
// End of a PCG iteration (host loop, one rank): the scalars the convergence test reads and the
// zero-pivot flag written into mapped pinned host memory, then a sequence number behind a
// system-scope fence; the host polls the number instead of copying and synchronising.
struct PcgPublish {
  double s[4];
  int err;
  unsigned seq;
};
void launch_pcg_publish(const Launch& L, const double* scal, const int* err, unsigned* dseq,
                        PcgPublish* hp);
// levels whose sweeps take the pre-factorised warp-per-column path when factors exist
bool jacobi_wants_factors(const LevelCoef& C);
// one-time device constants (L2 cache policies); called at context creation, outside any
// graph capture
void init_device_constants(cudaStream_t st);
void launch_jacobi(const Launch& L, const VertCoef& V, const LevelCoef& C, bool xi,
                   const double* u, const Halo& H, const double* f, double* out, double relax,
                   int* err, const PcgFuse* fuse = nullptr, int* nblocks = nullptr,
                   const ProSrc* pro = nullptr);
// True when launch_jacobi takes the tiled TMEM path on this level (the fused PCG modes).
bool jacobi_fusable(const LevelCoef& C);
// True when a post-sweep on this level can take the prolongation (TMA tiled path, factorised
// coefficients; TPMG_FUSE_PRO=0 disables).
bool jacobi_prolong_fusable(const LevelCoef& C);

// x += alpha p_old; p = z + beta p_old   (alpha = s[0]/s[1], beta = s[3]/s[0])
void launch_pcg_px(const Launch& L, int64_t n, const double* s, const double* z, double* p,
                   double* x);
// x += alpha p   (alpha = s[0]/s[1])
// Fused x += alpha p_old; p_new = z + beta p_old; q = A p_new (+ per-tile p.q partials):
// k_pcg_px + launch_apply(DOT) in one pass (tiled levels, z/p_old halos as views).
bool pcg_ap_fusable(const LevelCoef& C);
void launch_pcg_ap(const Launch& L, const VertCoef& V, const LevelCoef& C, bool xi,
                   const double* z, const Halo& Hz, const double* pold, const Halo& Hp,
                   double* pnew, double* q, double* x, const double* s, double* partials,
                   int* nblocks);
// Richardson / BiCGStab element-wise updates (see k_vec_lin for the exact expressions).
enum VecLinOp { VL_P = 0, VL_AXMY = 1, VL_X2 = 2, VL_AXPY = 3, VL_ADD = 4 };
void launch_vec_lin(const Launch& L, int op, int64_t n, double* y, const double* a,
                    const double* b, double s1, double s2);
// Indirect levels (GenRule / LevelCoef::nbr): summation or transpose restriction from the fine
// level and linear / injection prolongation (+=) into it; Cc is the coarse level,
// `children` its child table on the fine level.
void launch_restrict_gen(const Launch& L, const LevelCoef& Cc, const int* children,
                         const GenRule& rule, int64_t fplane, const double* fine, double* coarse,
                         bool transpose);
void launch_prolong_gen(const Launch& L, const LevelCoef& Cc, const int* children,
                        const GenRule& rule, int64_t fplane, const double* coarse, double* fine,
                        bool linear, bool add);
void launch_pcg_xfinal(const Launch& L, int64_t n, const double* s, const double* p, double* x);

// coarse = R_sum(fine) (restrict_field, multigrid.hpp:29-43).
void launch_restrict_sum(const Launch& L, int cnx, int cny, int nz, const double* fine,
                         double* coarse);
// coarse = R_sum(f - A u) fused (multigrid.hpp:285-291), u on the fine level.
void launch_resid_restrict_sum(const Launch& L, const VertCoef& V, const LevelCoef& Cf, bool xi,
                               const double* u, const Halo& H, const double* f, double* coarse);
// coarse = P^T (f - A u) fused.  One rank: periodic wrap inside the kernel (hu.xs = hu.ys = 0,
// hf = self_halo(f), ringc = nullptr).  Decomposed (resid_restrict_T2_fusable levels, factorised
// coefficients): u's two-cell halo with corners in hu, f's face halo in hf, the coefficient ring
// in ringc.
bool resid_restrict_T_fusable(const LevelCoef& Cf);
bool resid_restrict_T2_fusable(const LevelCoef& Cf);
void launch_resid_restrict_T(const Launch& L, const VertCoef& V, const LevelCoef& Cf, bool xi,
                             const double* u, const Halo2& hu, const double* f, const Halo& hf,
                             const double* ringc, double* coarse);
// coarse = P^T fine (restrict_field_transpose, multigrid.hpp:46-69); Hf: fine face halo.
void launch_restrict_transpose(const Launch& L, int cnx, int cny, int nz, const double* fine,
                               const Halo& Hf, double* coarse);
// fine (+)= P coarse (prolongate_field, multigrid.hpp:74-100; +=, :294-295); Hc: coarse halo.
void launch_prolong(const Launch& L, int fnx, int fny, int nz, const double* coarse,
                    const Halo& Hc, double* fine, bool linear, bool add);

// PCG vector kernels (device scalars: s[0]=rho, s[1]=p.q, s[2]=r.r, s[3]=rho_new).
// x += alpha p; r -= alpha q; partial |r|^2.   alpha = s[0]/s[1].
void launch_pcg_xr(const Launch& L, int64_t n, const double* s, double* x, double* r,
                   const double* p, const double* q, double* partials, int* nblocks);
// p = z + beta p, beta = s[3]/s[0]; then s[0] = s[3] is done by the finaliser.
void launch_pcg_p(const Launch& L, int64_t n, const double* s, const double* z, double* p);
// partial dot a.b
void launch_dot(const Launch& L, int64_t n, const double* a, const double* b, double* partials,
                int* nblocks);
// out[slot] = sum(partials[0..nblocks)) in fixed order; if copy_from >= 0 also s[copy_to] = s[copy_from]
// first (used to roll rho_new -> rho).
void launch_reduce(const Launch& L, const double* partials, int nblocks, double* out);
// Tile-layout dot (32x4 columns per partial, the fused kernels' layout) on an nx x ny x nz
// field; dot_tiles_ok: the level tiles.  launch_reduce_tiles: k_reduce over px x py ranks' tile
// partials in the global tile order (bitwise the one-rank result).
bool dot_tiles_ok(int nx, int ny);
void launch_dot_tiles(const Launch& L, int nx, int ny, int nz, const double* a, const double* b,
                      double* partials, int* nblocks);
void launch_reduce_tiles(const Launch& L, const double* gathered, int64_t stride, int gxl,
                         int gyl, int px, int py, double* out);
void launch_copy_scalar(const Launch& L, double* s, int dst, int src);

// Layout permutations for upload/download: k-fastest (reference Field) <-> [k][y][x].
void launch_kfast_to_xfast(const Launch& L, int64_t ncol, int nz, const double* in, double* out);
void launch_xfast_to_kfast(const Launch& L, int64_t ncol, int nz, const double* in, double* out);
void launch_fill(const Launch& L, int64_t n, double* p, double v);
void launch_fill_hash(const Launch& L, int64_t n, double* p, double v, uint64_t seed);

// Multi-GPU halo packing: the face values of u ([k][j] W/E, [k][i] S/N) written to dst.
void launch_pack_faces(const Launch& L, int nx, int ny, int nz, const double* u, const FaceDst& dst);
// The two-cell faces and 2x2 corners of u (Halo2 layouts of the receiving ranks) written to dst.
void launch_pack_deep(const Launch& L, int nx, int ny, int nz, const double* u, const DeepDst& dst);

// ---- coarse-grid agglomeration (tpmg_mg_config::agglomerate) ---------------------------------
// A replicated level is held whole ([k][gny][gnx]) on every rank; the ranks' blocks of it are
// bnx x bny (rank r = ry*px + rx owns the block at (rx*bnx, ry*bny)).
constexpr int kMaxPeers = 64;
struct PeerDst {
  double* p[kMaxPeers];  // every rank's replicated copy (CUDA-IPC mappings; own copy included)
  int n;
};
// dst[k][y][x] = the blocks of all ranks, gathered [r][k][j][i] (NCCL all-gather; px = py = 1:
// one block, the loopback identity)
void launch_blocks_to_level(const Launch& L, const double* gathered, int px, int py, int bnx,
                            int bny, int nz, double* dst);
// this rank's block (bnx x bny at x0, y0) stored into every rank's replicated copy (NVLink peer
// stores): the all-gather of the CUDA-IPC transport
void launch_block_to_peers(const Launch& L, const double* blk, int bnx, int bny, int nz, int x0,
                           int y0, int gnx, int gny, const PeerDst& dst);
// blk[k][j][i] = src[k][y0+j][x0+i] of a replicated level (the rank's block, for the prolongation)
void launch_block_from_level(const Launch& L, const double* src, int gnx, int gny, int nz, int x0,
                             int y0, int bnx, int bny, double* blk);
// the face halo of the block at (x0, y0) as strided views into the replicated level (periodic)
Halo block_halo(const double* src, int gnx, int gny, int64_t gplane, int x0, int y0, int bnx,
                int bny);

}  // namespace tpmg
