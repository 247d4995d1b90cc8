// tpmg_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see tpmg_oracle.h).
//
// A line-by-line CPU restatement of the reference's hot path
// (/root/reference/proj/include/tpmg/{discretization,relaxation,multigrid,parallel}.hpp)
// on explicit neighbour tables.  Build with -ffp-contract=off so every
// expression rounds exactly like the reference's unfused Eigen expressions.
// Every function cites the reference lines it restates.
#include "tpmg_oracle.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using Index = int64_t;

// tpmg_status codes (include/tpmg_b200.h), mirroring types.hpp:24-58.
enum : int {
  OK = 0, E_CONFIG = 1, E_SHAPE = 2, E_NONFINITE = 3, E_SINGULAR = 5,
  NOT_CONVERGED = 9, BREAKDOWN = 10, DIVERGED = 11
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

thread_local std::string g_last_error;

// parallel.hpp:13-30: static block partition, one std::thread per worker,
// spawned and joined per call; threads <= 1 is the sequential reference mode.
template <typename Fn>
void parallel_for(Index n, int threads, Fn&& fn) {
  if (threads <= 1 || n < 2) {
    for (Index i = 0; i < n; ++i) fn(i);
    return;
  }
  const Index nw = std::min<Index>(threads, n);
  std::vector<std::thread> pool;
  pool.reserve(static_cast<size_t>(nw));
  for (Index w = 0; w < nw; ++w) {
    const Index lo = n * w / nw, hi = n * (w + 1) / nw;
    pool.emplace_back([lo, hi, &fn] {
      for (Index i = lo; i < hi; ++i) fn(i);
    });
  }
  for (auto& t : pool) t.join();
}

struct Level {
  Index ncells = 0, nedges = 0;
  std::vector<Index> nbr, cedge;  // T*nnb + d  (geometry.hpp:51-53)
  std::vector<Index> children;    // children of THIS level's cells on level+1: T*nchild + j
  // separable hatted horizontal factors (HattedComponent::horiz, discretization.hpp:32-48)
  std::vector<double> bh, ah, xh, sh;
  // dense hatted components (HattedComponent::dense) of the partial / full modes, [k][T]
  // (alpha_s: [k][e]); empty when unused
  std::vector<double> bd, ard, xid, sd;
};

struct Hier {
  int nnb = 4, nchild = 4;
  Index nz = 0;
  std::vector<Level> lv;  // coarsest .. finest (MultigridHierarchy::coefficients order)
  std::vector<int> prol_d1, prol_d2;
  std::vector<double> bv, sv, av, xv;  // HattedComponent::vert, shared by all levels
  double relax = 1.0;
  int prolongation = 0, restriction = 0;
  std::vector<int> nu_pre, nu_post;
  int threads = 1;
  Index cart_nx = 0, cart_ny = 0;  // finest Cartesian dims (0 for generic tables)
  int pcg_fused = -1;              // -1: device rule, 0/1: forced
  bool device_order = true;        // PCG dots in the device's reduction order (parity mode)
  int t4 = 0;                      // device smoother v4 enabled (TPMG_JACOBI_T4, opt-in)
  int cm = 0;                      // 0 factorised, 1 partial (alpha_r dense), 2 full
};

// ColumnMatrix, discretization.hpp:208-231.
struct Col {
  std::vector<double> diag, upper, lower, nb;  // nb: column d contiguous (neighbor(k,d))
  void resize(Index nz, int nnb) {
    diag.resize(nz); upper.resize(nz); lower.resize(nz); nb.resize(nz * nnb);
  }
};

// build_column, discretization.hpp:235-251 (HattedComponent::operator() = vert[k]*horiz[j],
// discretization.hpp:39-41).
// HattedComponent::operator()(k, j) (discretization.hpp:39-41): the separable product, or the
// dense entry for the components the partial / full modes store in full.
void build_column(const Hier& h, const Level& L, Index T, Col& c) {
  const Index nr = h.nz, nc = L.ncells;
  c.resize(nr, h.nnb);
  const double ahT = L.ah[T], xhT = L.xh[T], bhT = L.bh[T];
  auto alpha_r = [&](Index k) { return h.cm ? L.ard[k * nc + T] : h.av[k] * ahT; };
  auto xi_r = [&](Index k) { return h.cm == 2 ? (L.xid.empty() ? 0.0 : L.xid[k * nc + T]) : h.xv[k] * xhT; };
  for (Index k = 0; k < nr; ++k) {
    c.upper[k] = -alpha_r(k + 1) - xi_r(k + 1);
    c.lower[k] = -alpha_r(k) + xi_r(k);
  }
  for (int j = 0; j < h.nnb; ++j) {
    const Index e = L.cedge[T * h.nnb + j];
    for (Index k = 0; k < nr; ++k)
      c.nb[j * nr + k] = -(h.cm == 2 ? L.sd[k * L.nedges + e] : h.sv[k] * L.sh[e]);
  }
  for (Index k = 0; k < nr; ++k) {
    // Eigen row(k).sum() of the n_r x nnb neighbour block: ((n0 + n1) + n2) + ...
    double s = c.nb[k];
    for (int j = 1; j < h.nnb; ++j) s = s + c.nb[j * nr + k];
    const double beta = h.cm == 2 ? L.bd[k * nc + T] : h.bv[k] * bhT;
    c.diag[k] = beta - ((c.upper[k] + c.lower[k]) + s);
  }
}

// ColumnMatrix::apply_tridiag, discretization.hpp:220-230.
void apply_tridiag(const Col& c, Index n, const double* x, double* y) {
  for (Index k = 0; k < n; ++k) {
    double v = c.diag[k] * x[k];
    if (k + 1 < n) v += c.upper[k] * x[k + 1];
    if (k > 0) v += c.lower[k] * x[k - 1];
    y[k] = v;
  }
}

// thomas_solve_inplace, relaxation.hpp:37-52.
void thomas(Index n, const double* diag, const double* upper, const double* lower, double* x,
            double* scratch) {
  double pivot = diag[0];
  if (pivot == 0.0) throw Error(E_SINGULAR, "thomas_solve: zero pivot at row 0");
  x[0] /= pivot;
  for (Index k = 1; k < n; ++k) {
    scratch[k] = upper[k - 1] / pivot;
    pivot = diag[k] - lower[k] * scratch[k];
    if (pivot == 0.0)
      throw Error(E_SINGULAR, "thomas_solve: zero pivot at row " + std::to_string(k));
    x[k] = (x[k] - lower[k] * x[k - 1]) / pivot;
  }
  for (Index k = n - 2; k >= 0; --k) x[k] -= scratch[k + 1] * x[k + 1];
}

// thomas() plus the r.z column sum of the fused finest post-sweep (k_jacobi_t3 PCGF 2):
// r.z = sum_k r_k u_k + relax sum_k w_k d'_k, with d' the forward pass's values and
// w_k = r_k - c'_k w_{k-1} (w = U^-T r, U the unit upper factor; c'_0 = 0, w_{-1} = 0), both
// sums ascending in k and every recurrence a fused multiply-add (as the device kernel); equal to
// sum_k r_k (u_k + relax x_k) in exact arithmetic.
void thomas_rz(Index n, const double* diag, const double* upper, const double* lower, double* x,
               double* scratch, const double* r, const double* u, double relax, double* colsum) {
  double pivot = diag[0];
  if (pivot == 0.0) throw Error(E_SINGULAR, "thomas_solve: zero pivot at row 0");
  x[0] /= pivot;
  for (Index k = 1; k < n; ++k) {
    scratch[k] = upper[k - 1] / pivot;
    pivot = diag[k] - lower[k] * scratch[k];
    if (pivot == 0.0)
      throw Error(E_SINGULAR, "thomas_solve: zero pivot at row " + std::to_string(k));
    x[k] = (x[k] - lower[k] * x[k - 1]) / pivot;
  }
  double su = 0.0, sw = 0.0, w = 0.0;
  for (Index k = 0; k < n; ++k) {
    su = std::fma(r[k], u[k], su);
    w = std::fma(-(k == 0 ? 0.0 : scratch[k]), w, r[k]);
    sw = std::fma(w, x[k], sw);
  }
  *colsum = su + relax * sw;
  for (Index k = n - 2; k >= 0; --k) x[k] -= scratch[k + 1] * x[k + 1];
}

// apply_operator, discretization.hpp:262-278.
void apply(const Hier& h, int level, const double* u, double* y) {
  const Level& L = h.lv[level];
  const Index nr = h.nz;
  parallel_for(L.ncells, h.threads, [&](Index T) {
    thread_local Col col;
    build_column(h, L, T, col);
    double* yc = y + T * nr;
    apply_tridiag(col, nr, u + T * nr, yc);
    for (int j = 0; j < h.nnb; ++j) {
      const double* un = u + L.nbr[T * h.nnb + j] * nr;
      const double* nb = col.nb.data() + j * nr;
      for (Index k = 0; k < nr; ++k) yc[k] += nb[k] * un[k];
    }
  });
}

// smooth, relaxation.hpp:63-97 (block_jacobi branch; relax_cell :77-87).
// rz_col (the fused PCG's finest post-sweep): the last sweep also forms the per-column r.z sums
// of thomas_rz (f is r there)
void smooth(const Hier& h, int level, double* u, const double* f, int sweeps,
            double* rz_col = nullptr) {
  if (!(h.relax > 0.0 && h.relax < 2.0))
    throw Error(E_CONFIG, "smoother relaxation factor must lie in (0, 2)");
  const Level& L = h.lv[level];
  const Index nr = h.nz, ns = L.ncells;
  std::vector<double> snapshot;
  for (int s = 0; s < sweeps; ++s) {
    snapshot.assign(u, u + ns * nr);  // relaxation.hpp:92
    std::atomic<bool> failed{false};
    parallel_for(ns, h.threads, [&](Index T) {
      thread_local Col col;
      thread_local std::vector<double> res, scratch;
      build_column(h, L, T, col);
      res.resize(nr);
      scratch.resize(nr);
      const double* from = snapshot.data();
      apply_tridiag(col, nr, from + T * nr, res.data());
      for (int j = 0; j < h.nnb; ++j) {
        const double* un = from + L.nbr[T * h.nnb + j] * nr;
        const double* nb = col.nb.data() + j * nr;
        for (Index k = 0; k < nr; ++k) res[k] += nb[k] * un[k];
      }
      const double* fc = f + T * nr;
      for (Index k = 0; k < nr; ++k) res[k] = fc[k] - res[k];
      try {
        if (rz_col && s + 1 == sweeps)
          thomas_rz(nr, col.diag.data(), col.upper.data(), col.lower.data(), res.data(),
                    scratch.data(), fc, from + T * nr, h.relax, rz_col + T);
        else
          thomas(nr, col.diag.data(), col.upper.data(), col.lower.data(), res.data(),
                 scratch.data());
      } catch (const Error&) {
        failed = true;
        return;
      }
      double* into = u + T * nr;
      const double* fr = from + T * nr;
      for (Index k = 0; k < nr; ++k) into[k] = fr[k] + h.relax * res[k];
    });
    if (failed) throw Error(E_SINGULAR, "thomas_solve: zero pivot");
  }
}

// restrict_field (multigrid.hpp:29-43) / restrict_field_transpose (multigrid.hpp:46-69).
void restrict_(const Hier& h, int coarse_level, const double* fine, double* coarse) {
  const Level& C = h.lv[coarse_level];
  const Index nr = h.nz;
  const int nc = h.nchild;
  parallel_for(C.ncells, h.threads, [&](Index T) {
    double* acc = coarse + T * nr;
    const Index* ch = C.children.data() + T * nc;
    if (h.restriction == 0) {
      // ((c0 + c1) + c2) + c3, Eigen's left-to-right expression tree (multigrid.hpp:37-40)
      for (Index k = 0; k < nr; ++k) {
        double v = fine[ch[0] * nr + k];
        for (int j = 1; j < nc; ++j) v = v + fine[ch[j] * nr + k];
        acc[k] = v;
      }
      return;
    }
    // transpose: centre child weight 1 (if any), own corner children 1/2, the corner
    // children of each neighbour whose stencil touches T 1/4 (multigrid.hpp:54-66).
    int centre = -1;
    for (int j = 0; j < nc; ++j)
      if (h.prol_d1[j] < 0) centre = j;
    for (Index k = 0; k < nr; ++k) acc[k] = centre >= 0 ? fine[ch[centre] * nr + k] : 0.0;
    for (int j = 0; j < nc; ++j) {
      if (j == centre) continue;
      for (Index k = 0; k < nr; ++k) acc[k] += 0.5 * fine[ch[j] * nr + k];
    }
    for (int j = 0; j < h.nnb; ++j) {
      const Index Tn = C.nbr[T * h.nnb + j];
      for (int jj = 0; jj < nc; ++jj) {
        if (jj == centre) continue;
        const bool adjacent = C.nbr[Tn * h.nnb + h.prol_d1[jj]] == T ||
                              C.nbr[Tn * h.nnb + h.prol_d2[jj]] == T;
        if (!adjacent) continue;
        const double* fc = fine + C.children[Tn * nc + jj] * nr;
        for (Index k = 0; k < nr; ++k) acc[k] += 0.25 * fc[k];
      }
    }
  });
}

// prolongate_field, multigrid.hpp:74-100.
void prolong(const Hier& h, int coarse_level, const double* coarse, double* fine) {
  const Level& C = h.lv[coarse_level];
  const Index nr = h.nz;
  const int nc = h.nchild;
  parallel_for(C.ncells, h.threads, [&](Index T) {
    const double* cT = coarse + T * nr;
    for (int j = 0; j < nc; ++j) {
      double* child = fine + C.children[T * nc + j] * nr;
      if (h.prol_d1[j] < 0 || h.prolongation == 1) {
        for (Index k = 0; k < nr; ++k) child[k] = cT[k];
      } else {
        const double* n1 = coarse + C.nbr[T * h.nnb + h.prol_d1[j]] * nr;
        const double* n2 = coarse + C.nbr[T * h.nnb + h.prol_d2[j]] * nr;
        for (Index k = 0; k < nr; ++k) child[k] = (2.0 * cT[k] + n1[k] + n2[k]) / 4.0;
      }
    }
  });
}

// v_cycle, multigrid.hpp:276-299.
void vcycle(const Hier& h, int level, const double* f, double* u, double* rz_col = nullptr) {
  const Index nr = h.nz;
  smooth(h, level, u, f, h.nu_pre[level]);
  if (level > 0) {
    const Index n = h.lv[level].ncells * nr;
    std::vector<double> r(n);
    apply(h, level, u, r.data());
    for (Index i = 0; i < n; ++i) r[i] = f[i] - r[i];
    const Index nc = h.lv[level - 1].ncells * nr;
    std::vector<double> fc(nc), uc(nc, 0.0), pu(n);
    restrict_(h, level - 1, r.data(), fc.data());
    vcycle(h, level - 1, fc.data(), uc.data());
    prolong(h, level - 1, uc.data(), pu.data());
    for (Index i = 0; i < n; ++i) u[i] += pu[i];
  }
  smooth(h, level, u, f, h.nu_post[level], rz_col);
}

// Deterministic dot product: sequential sums over 4096-element chunks, then a
// pairwise tree over the chunk partials.  (Field::norm / Eigen's vectorised
// redux order, discretization.hpp:27, is not pinned by any reference test.)
double dot(Index n, const double* a, const double* b) {
  const Index chunk = 4096;
  const Index nch = (n + chunk - 1) / chunk;
  std::vector<double> part(static_cast<size_t>(std::max<Index>(nch, 1)), 0.0);
  for (Index c = 0; c < nch; ++c) {
    double s = 0.0;
    const Index lo = c * chunk, hi = std::min(n, lo + chunk);
    for (Index i = lo; i < hi; ++i) s += a[i] * b[i];
    part[c] = s;
  }
  Index m = nch;
  while (m > 1) {
    const Index half = (m + 1) / 2;
    for (Index i = 0; i + half < m; ++i) part[i] = part[i] + part[i + half];
    m = half;
  }
  return nch ? part[0] : 0.0;
}

// ---- device reduction order ------------------------------------------------------------
// The GPU path reduces dot products with a fixed tree (paper_1408_2981_b200/csrc/
// tpmg_kernels.cu: block_sum, k_dot, k_pcg_xr, k_reduce, k_apply[_tiled]).  The oracle's
// PCG uses the same tree so that the strict GPU build can be compared bitwise end to end;
// the reference's own summation order (Eigen's vectorised norm, discretization.hpp:27) is
// not pinned by any reference test.
double warp_tree(double* v) {  // __shfl_down_sync tree, result of lane 0
  for (int o = 16; o > 0; o >>= 1)
    for (int i = 0; i < o; ++i) v[i] = v[i] + v[i + o];
  return v[0];
}

double block_tree(const double* acc, int nthreads) {  // block_sum
  double part[32];
  const int nw = (nthreads + 31) / 32;
  for (int w = 0; w < nw; ++w) {
    double v[32];
    for (int l = 0; l < 32; ++l) v[l] = acc[w * 32 + l];
    part[w] = warp_tree(v);
  }
  double v[32];
  for (int l = 0; l < 32; ++l) v[l] = l < nw ? part[l] : 0.0;
  return warp_tree(v);
}

double reduce_partials(const std::vector<double>& p) {  // k_reduce<<<1,1024>>>
  std::vector<double> acc(1024, 0.0);
  for (int t = 0; t < 1024; ++t)
    for (size_t q = t; q < p.size(); q += 1024) acc[t] += p[q];
  return block_tree(acc.data(), 1024);
}

// Layout of the finest level on the device: [k][y][x]; element t <-> oracle (col, k).
struct DevOrder {
  Index nx = 0, ny = 0, nz = 0;
  Index plane() const { return nx * ny; }
  Index oidx(Index t) const { return (t % plane()) * nz + t / plane(); }
};

// k_dot / k_pcg_xr: grid-stride over the x-fastest index with vec_blocks(n) blocks of 256.
template <typename Val>
double gridstride_dot(const DevOrder& d, Val val) {
  const Index n = d.plane() * d.nz;
  Index B = (n + 255) / 256;
  if (B > 148 * 8) B = 148 * 8;
  if (B < 1) B = 1;
  const Index G = B * 256;
  std::vector<double> acc(G, 0.0);
  for (Index g = 0; g < G; ++g) {
    double a = 0.0;
    for (Index t = g; t < n; t += G) a += val(d.oidx(t));
    acc[g] = a;
  }
  std::vector<double> part(B);
  for (Index b = 0; b < B; ++b) part[b] = block_tree(acc.data() + b * 256, 256);
  return reduce_partials(part);
}

// fused p.q of the apply kernel: per-column sums over k, then per-CTA trees.
// descending: the per-column sum runs k = nz-1 .. 0 (sums formed in a back substitution)
// nc = 2: the two-columns-per-thread smoother (k_jacobi_t4): 64x4 tiles, thread t = (tx, ty)
// holds columns tx and tx+32 and adds its two column sums before the block tree.
double column_reduce(const DevOrder& d, const std::vector<double>& colsum, int nc);
double column_dot(const DevOrder& d, const double* y, const double* u, bool descending = false,
                  int nc = 1) {
  const Index plane = d.plane();
  std::vector<double> colsum(plane);
  for (Index c = 0; c < plane; ++c) {
    double a = 0.0;
    if (descending)
      for (Index k = d.nz - 1; k >= 0; --k) a += y[c * d.nz + k] * u[c * d.nz + k];
    else
      for (Index k = 0; k < d.nz; ++k) a += y[c * d.nz + k] * u[c * d.nz + k];
    colsum[c] = a;
  }
  return column_reduce(d, colsum, nc);
}

// the per-tile trees of the fused kernels over per-column sums, then k_reduce
double column_reduce(const DevOrder& d, const std::vector<double>& colsum, int nc) {
  const Index plane = d.plane();
  std::vector<double> part;
  if (nc == 2) {
    const Index gx = d.nx / 64, gy = d.ny / 4;
    part.resize(gx * gy);
    double acc[128];
    for (Index by = 0; by < gy; ++by)
      for (Index bx = 0; bx < gx; ++bx) {
        for (int t = 0; t < 128; ++t) {
          const Index c0 = (by * 4 + t / 32) * d.nx + bx * 64 + t % 32;
          acc[t] = colsum[c0] + colsum[c0 + 32];
        }
        part[by * gx + bx] = block_tree(acc, 128);
      }
  } else if (d.nx % 32 == 0 && d.ny % 4 == 0) {  // k_apply_t3: 32x4 tiles, order by*gx+bx
    const Index gx = d.nx / 32, gy = d.ny / 4;
    part.resize(gx * gy);
    double acc[128];
    for (Index by = 0; by < gy; ++by)
      for (Index bx = 0; bx < gx; ++bx) {
        for (int t = 0; t < 128; ++t) acc[t] = colsum[(by * 4 + t / 32) * d.nx + bx * 32 + t % 32];
        part[by * gx + bx] = block_tree(acc, 128);
      }
  } else {  // k_apply_small: 64 consecutive columns per block
    const Index B = (plane + 63) / 64;
    part.resize(B);
    double acc[64];
    for (Index b = 0; b < B; ++b) {
      for (int t = 0; t < 64; ++t) acc[t] = b * 64 + t < plane ? colsum[b * 64 + t] : 0.0;
      part[b] = block_tree(acc, 64);
    }
  }
  return reduce_partials(part);
}

// dot_into of the device (tpmg_host.cpp): k_dot_tiles on a level that tiles by 32x4 (per-thread
// column sums over k, per-tile block tree, k_reduce), k_dot's grid-stride tree otherwise
double tile_or_gridstride_dot(const DevOrder& d, const double* a, const double* b) {
  if (d.nx % 32 == 0 && d.ny % 4 == 0) return column_dot(d, a, b);
  return gridstride_dot(d, [&](Index i) { return a[i] * b[i]; });
}

void check_finite(const double* p, Index n, const char* what) {
  for (Index i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) throw Error(E_NONFINITE, std::string("non-finite values in ") + what);
}

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return E_CONFIG;
  }
}

void finalize_nu(Hier& h, int nu_pre, int nu_post) {
  const size_t d = h.lv.size();
  h.nu_pre.assign(d, nu_pre);
  h.nu_post.assign(d, nu_post);
  h.nu_pre[0] = 1;  // multigrid.hpp:269-270: coarsest does one sweep in total
  h.nu_post[0] = 0;
}

}  // namespace

struct tpmgo_hier_s {
  Hier h;
};

extern "C" {

const char* tpmgo_last_error(void) { return g_last_error.c_str(); }

namespace {
// cm: 0 factorised profiles; 1 partial (dense alpha_r `da`); 2 full (dense db, ds, da, dx; the
// factorised arguments may be null).  Dense inputs in the reference's Matrix order (k fastest).
int cart_create_impl(int cm, const double* db, const double* ds, const double* da,
                     const double* dx, int64_t nx, int64_t ny, double hx, double hy, int64_t nz,
                     const double* z, const double* beta_r, const double* alpha_s_r,
                     const double* alpha_r_r, const double* xi_r_r, const double* beta_s,
                     const double* alpha_r_s, const double* xi_r_s, const double* alpha_s_s,
                     double omega, double relax, int prolongation, int restriction, int nu_pre,
                     int nu_post, int depth, int threads, tpmgo_hier* out) {
  return guard([&] {
    if (nx < 1 || ny < 1 || nz < 1) throw Error(E_CONFIG, "grid dimensions must be positive");
    if (!(hx > 0.0) || !(hy > 0.0)) throw Error(E_CONFIG, "cell widths must be positive");
    for (Index k = 0; k < nz; ++k)
      if (!(z[k + 1] > z[k])) throw Error(E_CONFIG, "vertical faces must increase");
    if (!(relax > 0.0 && relax < 2.0))
      throw Error(E_CONFIG, "smoother relaxation factor must lie in (0, 2)");
    // depth: number of levels; 0 = coarsen while both dims stay even and >= 4.
    int levels = 1;
    {
      Index a = nx, b = ny;
      if (depth <= 0) {
        while (a % 2 == 0 && b % 2 == 0 && a / 2 >= 4 && b / 2 >= 4) {
          a /= 2; b /= 2; ++levels;
        }
      } else {
        for (int l = 1; l < depth; ++l) {
          if (a % 2 || b % 2) throw Error(E_CONFIG, "grid does not coarsen to the requested depth");
          a /= 2; b /= 2;
        }
        levels = depth;
      }
      // same rule as the product (tpmg_host.cpp plan_levels): with < 3 coarse cells per
      // dimension the W/E (S/N) neighbours coincide and the transpose stencil double counts
      if ((prolongation == 0 || restriction == 1) && levels > 1 && (a < 3 || b < 3))
        throw Error(E_CONFIG, "linear transfers need >= 3 coarse cells per dimension");
    }
    const Index ncf = nx * ny;
    check_finite(z, nz + 1, "z_faces");
    std::vector<double> zero_v(nz + 1, 0.0), zero_h(2 * ncf, 0.0);
    if (cm == 2) {  // full: the factorised parts are not used
      beta_r = alpha_s_r = alpha_r_r = zero_v.data();
      beta_s = alpha_r_s = alpha_s_s = zero_h.data();
      xi_r_r = xi_r_s = nullptr;
      check_finite(db, nz * ncf, "beta");
      check_finite(ds, nz * 2 * ncf, "alpha_s");
      check_finite(da, (nz + 1) * ncf, "alpha_r");
      if (dx) check_finite(dx, (nz + 1) * ncf, "xi_r");
    }
    if (cm == 1) check_finite(da, (nz + 1) * ncf, "alpha_r (full)");
    check_finite(beta_r, nz, "beta_r");
    check_finite(alpha_s_r, nz, "alpha_s_r");
    check_finite(alpha_r_r, nz + 1, "alpha_r_r");
    if (xi_r_r) check_finite(xi_r_r, nz + 1, "xi_r_r");
    check_finite(beta_s, ncf, "beta_s");
    check_finite(alpha_r_s, ncf, "alpha_r_s");
    if (xi_r_s) check_finite(xi_r_s, ncf, "xi_r_s");
    check_finite(alpha_s_s, 2 * ncf, "alpha_s_s");
    // dense profiles [k][global cell] (alpha_s: [k][edge])
    std::vector<double> Da, Db, Dx, Ds;
    auto to_kc = [&](const double* in, Index rows, Index cols, std::vector<double>& o) {
      o.resize(rows * cols);
      for (Index c = 0; c < cols; ++c)
        for (Index k = 0; k < rows; ++k) o[k * cols + c] = in[c * rows + k];
    };
    if (cm >= 1) to_kc(da, nz + 1, ncf, Da);
    if (cm == 2) {
      to_kc(db, nz, ncf, Db);
      to_kc(ds, nz, 2 * ncf, Ds);
      if (dx) to_kc(dx, nz + 1, ncf, Dx);
    }

    auto* H = new tpmgo_hier_s;
    Hier& h = H->h;
    h.nnb = 4;
    h.nchild = 4;
    h.nz = nz;
    h.relax = relax;
    h.prolongation = prolongation;
    h.restriction = restriction;
    h.threads = threads;
    h.cm = cm;
    // Cartesian corner child (a,b) = a + 2b blends the x-side and y-side coarse neighbours
    // (directions W=0, E=1, S=2, N=3) -- analogue of multigrid.hpp:91-95.
    h.cart_nx = nx;
    h.cart_ny = ny;
    h.prol_d1 = {0, 1, 0, 1};
    h.prol_d2 = {2, 2, 3, 3};

    // Flat vertical grid: volumes and face factors (discretization.hpp:72-87 with r_k^2 -> 1).
    std::vector<double> vol(nz), fdiff(nz + 1, 0.0), fadv(nz + 1, 0.0);
    for (Index k = 0; k < nz; ++k) vol[k] = z[k + 1] - z[k];
    for (Index k = 1; k < nz; ++k) {
      fdiff[k] = 2.0 / (z[k + 1] - z[k - 1]);
      fadv[k] = (z[k + 1] - z[k]) / (z[k + 1] - z[k - 1]);
    }
    // Vertical hatted vectors (discretization.hpp:165-181); shared by all levels.
    h.bv.resize(nz); h.sv.resize(nz); h.av.resize(nz + 1); h.xv.resize(nz + 1);
    for (Index k = 0; k < nz; ++k) {
      h.bv[k] = vol[k] * beta_r[k];
      h.sv[k] = (z[k + 1] - z[k]) * alpha_s_r[k];
    }
    for (Index k = 0; k <= nz; ++k) {
      h.av[k] = fdiff[k] * alpha_r_r[k];
      h.xv[k] = xi_r_r ? fadv[k] * xi_r_r[k] : 0.0;
    }
    const double w2 = omega * omega;

    h.lv.resize(levels);
    // Profiles on the current level (horizontal scalars only; profiles.hpp:196-210).
    std::vector<double> pb(beta_s, beta_s + ncf), pa(alpha_r_s, alpha_r_s + ncf),
        px(ncf, 0.0), ps(alpha_s_s, alpha_s_s + 2 * ncf);
    if (xi_r_s) px.assign(xi_r_s, xi_r_s + ncf);
    Index cx = nx, cy = ny;
    double chx = hx, chy = hy;
    for (int l = levels - 1; l >= 0; --l) {
      Level& L = h.lv[l];
      const Index nc = cx * cy;
      L.ncells = nc;
      L.nedges = 2 * nc;
      L.nbr.resize(nc * 4);
      L.cedge.resize(nc * 4);
      for (Index j = 0; j < cy; ++j)
        for (Index i = 0; i < cx; ++i) {
          const Index T = j * cx + i;
          const Index iw = (i + cx - 1) % cx, ie = (i + 1) % cx;
          const Index js = (j + cy - 1) % cy, jn = (j + 1) % cy;
          L.nbr[T * 4 + 0] = j * cx + iw;
          L.nbr[T * 4 + 1] = j * cx + ie;
          L.nbr[T * 4 + 2] = js * cx + i;
          L.nbr[T * 4 + 3] = jn * cx + i;
          L.cedge[T * 4 + 0] = j * cx + iw;       // east edge of the west neighbour
          L.cedge[T * 4 + 1] = T;                 // own east edge
          L.cedge[T * 4 + 2] = nc + js * cx + i;  // north edge of the south neighbour
          L.cedge[T * 4 + 3] = nc + T;            // own north edge
        }
      // assemble_hatted (factorised), discretization.hpp:144-184, flat Cartesian geometry:
      // |T| = hx*hy, edge factor |S| n.dc/|dc|^2 = hy/hx (east), hx/hy (north).
      const double area = chx * chy;
      const double ge_e = chy / chx, ge_n = chx / chy;
      L.bh.resize(nc); L.ah.resize(nc); L.xh.resize(nc); L.sh.resize(2 * nc);
      for (Index T = 0; T < nc; ++T) {
        L.bh[T] = area * pb[T];
        L.ah[T] = w2 * (area * pa[T]);
        L.xh[T] = w2 * (area * px[T]);
      }
      for (Index T = 0; T < nc; ++T) {
        L.sh[T] = w2 * ge_e * ps[T];
        L.sh[nc + T] = w2 * ge_n * ps[nc + T];
      }
      // assemble_hatted, dense components (discretization.hpp:122-140, 196-203)
      if (cm >= 1) {
        L.ard.resize((nz + 1) * nc);
        for (Index k = 0; k <= nz; ++k)
          for (Index T = 0; T < nc; ++T)
            L.ard[k * nc + T] = ((w2 * area) * fdiff[k]) * Da[k * nc + T];
      }
      if (cm == 2) {
        L.bd.resize(nz * nc);
        L.sd.resize(nz * 2 * nc);
        for (Index k = 0; k < nz; ++k)
          for (Index T = 0; T < nc; ++T) {
            L.bd[k * nc + T] = area * (vol[k] * Db[k * nc + T]);
            L.sd[k * 2 * nc + T] = ((w2 * (z[k + 1] - z[k])) * ge_e) * Ds[k * 2 * nc + T];
            L.sd[k * 2 * nc + nc + T] =
                ((w2 * (z[k + 1] - z[k])) * ge_n) * Ds[k * 2 * nc + nc + T];
          }
        if (!Dx.empty()) {
          L.xid.resize((nz + 1) * nc);
          for (Index k = 0; k <= nz; ++k)
            for (Index T = 0; T < nc; ++T)
              L.xid[k * nc + T] = ((w2 * area) * fadv[k]) * Dx[k * nc + T];
        }
      }
      if (l == 0) break;
      // restrict_profiles (factorised), multigrid.hpp:158-201 / :107-151.
      const Index ncx = cx / 2, ncy = cy / 2, ncc = ncx * ncy;
      Level& C = h.lv[l - 1];
      C.children.resize(ncc * 4);
      std::vector<double> qb(ncc), qa(ncc), qx(ncc), qs(2 * ncc);
      const double wf = chx * chy;  // fine areas
      for (Index J = 0; J < ncy; ++J)
        for (Index I = 0; I < ncx; ++I) {
          const Index Tc = J * ncx + I;
          Index ch[4];
          for (int b = 0; b < 2; ++b)
            for (int a = 0; a < 2; ++a) ch[a + 2 * b] = (2 * J + b) * cx + (2 * I + a);
          for (int j = 0; j < 4; ++j) C.children[Tc * 4 + j] = ch[j];
          // area-weighted mean (restrict_cell_profile, multigrid.hpp:108-124)
          auto cell_mean = [&](const std::vector<double>& p) {
            double acc = 0.0, wsum = 0.0;
            for (int j = 0; j < 4; ++j) {
              acc += wf * p[ch[j]];
              wsum += wf;
            }
            return acc / wsum;
          };
          qb[Tc] = cell_mean(pb);
          qa[Tc] = cell_mean(pa);
          qx[Tc] = cell_mean(px);
          // co-linear edge mean (restrict_edge_profile, multigrid.hpp:135-143): coarse east
          // edge = fine east edges of (2I+1,2J), (2I+1,2J+1); north = fine north edges of
          // (2I,2J+1), (2I+1,2J+1).
          qs[Tc] = (ps[(2 * J) * cx + 2 * I + 1] + ps[(2 * J + 1) * cx + 2 * I + 1]) / 2.0;
          qs[ncc + Tc] =
              (ps[nc + (2 * J + 1) * cx + 2 * I] + ps[nc + (2 * J + 1) * cx + 2 * I + 1]) / 2.0;
        }
      pb.swap(qb); pa.swap(qa); px.swap(qx); ps.swap(qs);
      // restrict_profiles, dense rows (multigrid.hpp:107-151): the same means per level k
      auto cell_rows = [&](std::vector<double>& D, Index rows) {
        std::vector<double> q(rows * ncc);
        for (Index k = 0; k < rows; ++k)
          for (Index Tc = 0; Tc < ncc; ++Tc) {
            const Index* chh = C.children.data() + Tc * 4;
            double acc = 0.0, wsum = 0.0;
            for (int j = 0; j < 4; ++j) {
              acc += wf * D[k * nc + chh[j]];
              wsum += wf;
            }
            q[k * ncc + Tc] = acc / wsum;
          }
        D.swap(q);
      };
      if (cm >= 1) cell_rows(Da, nz + 1);
      if (cm == 2) {
        cell_rows(Db, nz);
        if (!Dx.empty()) cell_rows(Dx, nz + 1);
        std::vector<double> q(nz * 2 * ncc);
        for (Index k = 0; k < nz; ++k)
          for (Index J = 0; J < ncy; ++J)
            for (Index I = 0; I < ncx; ++I) {
              const double* d = Ds.data() + k * 2 * nc;
              const Index Tc = J * ncx + I;
              q[k * 2 * ncc + Tc] = (d[(2 * J) * cx + 2 * I + 1] + d[(2 * J + 1) * cx + 2 * I + 1]) / 2.0;
              q[k * 2 * ncc + ncc + Tc] =
                  (d[nc + (2 * J + 1) * cx + 2 * I] + d[nc + (2 * J + 1) * cx + 2 * I + 1]) / 2.0;
            }
        Ds.swap(q);
      }
      cx = ncx; cy = ncy;
      chx *= 2.0; chy *= 2.0;
    }
    finalize_nu(h, nu_pre, nu_post);
    *out = H;
  });
}
}  // namespace

int tpmgo_cart_create(int64_t nx, int64_t ny, double hx, double hy, int64_t nz,
                      const double* z, const double* beta_r, const double* alpha_s_r,
                      const double* alpha_r_r, const double* xi_r_r, const double* beta_s,
                      const double* alpha_r_s, const double* xi_r_s, const double* alpha_s_s,
                      double omega, double relax, int prolongation, int restriction, int nu_pre,
                      int nu_post, int depth, int threads, tpmgo_hier* out) {
  return cart_create_impl(0, nullptr, nullptr, nullptr, nullptr, nx, ny, hx, hy, nz, z, beta_r,
                          alpha_s_r, alpha_r_r, xi_r_r, beta_s, alpha_r_s, xi_r_s, alpha_s_s,
                          omega, relax, prolongation, restriction, nu_pre, nu_post, depth,
                          threads, out);
}

int tpmgo_cart_create_dense(int mode, const double* beta, const double* alpha_s,
                            const double* alpha_r, const double* xi_r, int64_t nx, int64_t ny,
                            double hx, double hy, int64_t nz, const double* z,
                            const double* beta_r, const double* alpha_s_r,
                            const double* alpha_r_r, const double* xi_r_r, const double* beta_s,
                            const double* alpha_r_s, const double* xi_r_s,
                            const double* alpha_s_s, double omega, double relax,
                            int prolongation, int restriction, int nu_pre, int nu_post,
                            int depth, int threads, tpmgo_hier* out) {
  if (mode != 1 && mode != 2) {
    g_last_error = "mode must be 1 (partial) or 2 (full)";
    return E_CONFIG;
  }
  return cart_create_impl(mode, beta, alpha_s, alpha_r, xi_r, nx, ny, hx, hy, nz, z, beta_r,
                          alpha_s_r, alpha_r_r, xi_r_r, beta_s, alpha_r_s, xi_r_s, alpha_s_s,
                          omega, relax, prolongation, restriction, nu_pre, nu_post, depth,
                          threads, out);
}

int tpmgo_generic_create(int n_levels, int64_t nz, int nnb, int nchild, const int64_t* ncells,
                         const int64_t* nedges, const int64_t* const* nbr,
                         const int64_t* const* cedge, const int64_t* const* children,
                         const int* prol_d1, const int* prol_d2, const double* bv,
                         const double* sv, const double* av, const double* xv,
                         const double* const* bh, const double* const* ah,
                         const double* const* xh, const double* const* sh, double relax,
                         int prolongation, int restriction, int nu_pre, int nu_post, int threads,
                         tpmgo_hier* out) {
  return guard([&] {
    if (n_levels < 1 || nz < 1 || nnb < 1 || nchild < 1) throw Error(E_CONFIG, "bad sizes");
    auto* H = new tpmgo_hier_s;
    Hier& h = H->h;
    h.nnb = nnb;
    h.nchild = nchild;
    h.nz = nz;
    h.relax = relax;
    h.prolongation = prolongation;
    h.restriction = restriction;
    h.threads = threads;
    h.prol_d1.assign(prol_d1, prol_d1 + nchild);
    h.prol_d2.assign(prol_d2, prol_d2 + nchild);
    h.bv.assign(bv, bv + nz);
    h.sv.assign(sv, sv + nz);
    h.av.assign(av, av + nz + 1);
    h.xv = xv ? std::vector<double>(xv, xv + nz + 1) : std::vector<double>(nz + 1, 0.0);
    h.lv.resize(n_levels);
    for (int l = 0; l < n_levels; ++l) {
      Level& L = h.lv[l];
      L.ncells = ncells[l];
      L.nedges = nedges[l];
      L.nbr.assign(nbr[l], nbr[l] + L.ncells * nnb);
      L.cedge.assign(cedge[l], cedge[l] + L.ncells * nnb);
      L.bh.assign(bh[l], bh[l] + L.ncells);
      L.ah.assign(ah[l], ah[l] + L.ncells);
      L.xh = xh ? std::vector<double>(xh[l], xh[l] + L.ncells)
                : std::vector<double>(L.ncells, 0.0);
      L.sh.assign(sh[l], sh[l] + L.nedges);
      if (l >= 1) h.lv[l - 1].children.assign(children[l], children[l] + ncells[l - 1] * nchild);
    }
    finalize_nu(h, nu_pre, nu_post);
    *out = H;
  });
}

void tpmgo_destroy(tpmgo_hier h) { delete h; }
int tpmgo_n_levels(tpmgo_hier h) { return static_cast<int>(h->h.lv.size()); }
int64_t tpmgo_n_cells(tpmgo_hier h, int level) { return h->h.lv[level].ncells; }
int64_t tpmgo_nz(tpmgo_hier h) { return h->h.nz; }
int tpmgo_set_pcg_fused(tpmgo_hier h, int mode) {
  h->h.pcg_fused = mode;
  return OK;
}

int tpmgo_set_t4(tpmgo_hier h, int on) {
  h->h.t4 = on;
  return OK;
}

int tpmgo_set_device_order(tpmgo_hier h, int on) {
  h->h.device_order = on != 0;
  return OK;
}

int tpmgo_set_threads(tpmgo_hier h, int threads) {
  h->h.threads = threads;
  return OK;
}

static void check_level(const Hier& h, int level) {
  if (level < 0 || level >= static_cast<int>(h.lv.size()))
    throw Error(E_SHAPE, "level out of range");
}

int tpmgo_get_coefficients(tpmgo_hier H, int level, double* bh, double* ah, double* xh,
                           double* sh, double* bv, double* sv, double* av, double* xv) {
  return guard([&] {
    const Hier& h = H->h;
    check_level(h, level);
    const Level& L = h.lv[level];
    if (bh) std::memcpy(bh, L.bh.data(), L.ncells * 8);
    if (ah) std::memcpy(ah, L.ah.data(), L.ncells * 8);
    if (xh) std::memcpy(xh, L.xh.data(), L.ncells * 8);
    if (sh) std::memcpy(sh, L.sh.data(), L.nedges * 8);
    if (bv) std::memcpy(bv, h.bv.data(), h.nz * 8);
    if (sv) std::memcpy(sv, h.sv.data(), h.nz * 8);
    if (av) std::memcpy(av, h.av.data(), (h.nz + 1) * 8);
    if (xv) std::memcpy(xv, h.xv.data(), (h.nz + 1) * 8);
  });
}

int tpmgo_build_column(tpmgo_hier H, int level, int64_t cell, double* diag, double* upper,
                       double* lower, double* neighbor) {
  return guard([&] {
    const Hier& h = H->h;
    check_level(h, level);
    Col c;
    build_column(h, h.lv[level], cell, c);
    std::memcpy(diag, c.diag.data(), h.nz * 8);
    std::memcpy(upper, c.upper.data(), h.nz * 8);
    std::memcpy(lower, c.lower.data(), h.nz * 8);
    std::memcpy(neighbor, c.nb.data(), h.nz * h.nnb * 8);
  });
}

int tpmgo_thomas(int64_t n, const double* diag, const double* upper, const double* lower,
                 double* x) {
  return guard([&] {
    std::vector<double> scratch(n);
    thomas(n, diag, upper, lower, x, scratch.data());
  });
}

int tpmgo_apply(tpmgo_hier H, int level, const double* u, double* y) {
  return guard([&] {
    check_level(H->h, level);
    apply(H->h, level, u, y);
  });
}

int tpmgo_residual(tpmgo_hier H, int level, const double* f, const double* u, double* r) {
  return guard([&] {
    const Hier& h = H->h;
    check_level(h, level);
    apply(h, level, u, r);
    const Index n = h.lv[level].ncells * h.nz;
    for (Index i = 0; i < n; ++i) r[i] = f[i] - r[i];
  });
}

int tpmgo_smooth(tpmgo_hier H, int level, double* u, const double* f, int sweeps) {
  return guard([&] {
    check_level(H->h, level);
    smooth(H->h, level, u, f, sweeps);
  });
}

int tpmgo_restrict(tpmgo_hier H, int coarse_level, const double* fine, double* coarse) {
  return guard([&] {
    const Hier& h = H->h;
    if (coarse_level < 0 || coarse_level + 1 >= static_cast<int>(h.lv.size()))
      throw Error(E_SHAPE, "restrict_field: fine field is not one level above the target");
    restrict_(h, coarse_level, fine, coarse);
  });
}

int tpmgo_prolong(tpmgo_hier H, int coarse_level, const double* coarse, double* fine) {
  return guard([&] {
    const Hier& h = H->h;
    if (coarse_level < 0 || coarse_level + 1 >= static_cast<int>(h.lv.size()))
      throw Error(E_SHAPE, "prolongate_field: field level does not match");
    prolong(h, coarse_level, coarse, fine);
  });
}

int tpmgo_vcycle(tpmgo_hier H, int level, const double* f, double* u) {
  return guard([&] {
    check_level(H->h, level);
    vcycle(H->h, level, f, u);
  });
}

// measure_cycle_rate, multigrid.hpp:302-321.
int tpmgo_measure_cycle_rate(tpmgo_hier H, const double* f, int n_cycles, double* rate) {
  return guard([&] {
    const Hier& h = H->h;
    if (n_cycles < 2) throw Error(E_CONFIG, "measure_cycle_rate needs at least two cycles");
    const int L = static_cast<int>(h.lv.size()) - 1;
    const Index n = h.lv[L].ncells * h.nz;
    std::vector<double> u(n, 0.0), r(n);
    double first = 0, last = 0;
    for (int i = 1; i <= n_cycles; ++i) {
      vcycle(h, L, f, u.data());
      apply(h, L, u.data(), r.data());
      for (Index q = 0; q < n; ++q) r[q] = f[q] - r[q];
      const double nrm = std::sqrt(dot(n, r.data(), r.data()));
      if (i == 1) first = nrm;
      last = nrm;
    }
    const double fn = std::sqrt(dot(n, f, f));
    if (first <= 1e-300 || first <= std::numeric_limits<double>::epsilon() * fn) {
      *rate = 0.0;
      return;
    }
    *rate = std::pow(last / first, 1.0 / static_cast<double>(n_cycles - 1));
  });
}

// Preconditioned CG, right-hand side f, x0 = 0, preconditioner = one V-cycle from a zero
// guess on the residual.  Stop when |r_k|/|r_0| <= tol;
// divergence when > 1e4; breakdown when p.q <= 0 or r.z <= 0.
int tpmgo_pcg(tpmgo_hier H, const double* f, double* x, double tol, int max_iter,
              double* res_hist, int* iters, int* solve_status) {
  return tpmgo_pcg_timed(H, f, x, tol, max_iter, res_hist, nullptr, iters, solve_status);
}

// Same, with ConvergenceHistory's `seconds` column: wall time since the
// start of the solve at the end of each iteration (entry 0: after |r_0|).
int tpmgo_pcg_timed(tpmgo_hier H, const double* f, double* x, double tol, int max_iter,
                    double* res_hist, double* seconds, int* iters, int* solve_status) {
  const auto t0 = std::chrono::steady_clock::now();
  auto stamp = [&](int it) {
    if (seconds)
      seconds[it] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  return guard([&] {
    const Hier& h = H->h;
    const int L = static_cast<int>(h.lv.size()) - 1;
    const Index n = h.lv[L].ncells * h.nz;
    std::vector<double> r(f, f + n), z(n, 0.0), p(n), q(n);
    std::fill(x, x + n, 0.0);
    const bool dev = h.cart_nx > 0 && h.device_order;
    DevOrder d{h.cart_nx, h.cart_ny, h.nz};
    // Baseline mode (device_order off): plain chunked dots and element-wise updates spread over
    // the worker threads -- the fastest honest CPU schedule, used when timing the CPU port.
    const Index nchunk = (n + 65535) / 65536;
    auto par = [&](auto&& body) {
      parallel_for(nchunk, h.threads, [&](Index c) {
        const Index lo = c * 65536, hi = std::min(n, lo + 65536);
        body(lo, hi);
      });
    };
    auto pdot = [&](const double* a, const double* b) {
      std::vector<double> part(static_cast<size_t>(nchunk), 0.0);
      par([&](Index lo, Index hi) {
        double s = 0.0;
        for (Index i = lo; i < hi; ++i) s += a[i] * b[i];
        part[lo / 65536] = s;
      });
      double s = 0.0;
      for (double v : part) s += v;
      return s;
    };
    // the device's dot_into: tile-layout dot (k_dot_tiles) on a tiled level, else k_dot
    auto dotv = [&](const std::vector<double>& a, const std::vector<double>& b) {
      return dev ? tile_or_gridstride_dot(d, a.data(), b.data())
                 : (h.device_order ? dot(n, a.data(), b.data()) : pdot(a.data(), b.data()));
    };
    // k_pcg_xr (the unfused schedule's |r|^2): grid-stride partials
    auto gsdot = [&](const std::vector<double>& a) {
      return dev ? gridstride_dot(d, [&](Index i) { return a[i] * a[i]; })
                 : (h.device_order ? dot(n, a.data(), a.data()) : pdot(a.data(), a.data()));
    };
    // The device fuses |r|^2 into the first and r.z into the last finest-level sweep when the
    // finest level runs the tiled TMEM smoother (tpmg_host.cpp pcg_iteration); those partials
    // are per-column sums reduced per 32x4 tile.
    int cols = 32;
    while (cols < 2 * h.nz) cols <<= 1;
    const int Lf = static_cast<int>(h.lv.size()) - 1;
    const bool fused = dev && (h.pcg_fused >= 0 ? h.pcg_fused == 1
                                                : (h.cart_nx % 32 == 0 && h.cart_ny % 4 == 0 &&
                                                   h.nz % 4 == 0 && cols <= 512 && Lf > 0 &&
                                                   h.nu_pre[Lf] >= 1 && h.nu_post[Lf] >= 1));
    // ... and those sweeps run two columns per thread (64x4 tiles) when the device's
    // jacobi_uses_t4 rule holds (tpmg_kernels.cu): 64-wide tiles, even nz, 2 nz <= 256.
    int cols4 = 32;
    while (cols4 < 2 * h.nz) cols4 <<= 1;
    const int nc = (h.t4 != 0 && h.cart_nx > 0 && h.cart_nx % 64 == 0 && h.cart_ny % 4 == 0 &&
                    h.nz % 4 == 0 && cols4 <= 256) ? 2 : 1;
    const double r0 = std::sqrt(dotv(r, r));
    if (res_hist) res_hist[0] = r0;
    stamp(0);
    *iters = 0;
    *solve_status = OK;
    if (r0 == 0.0) return;
    vcycle(h, L, r.data(), z.data());
    p = z;
    double rho = dotv(r, z);
    if (!(rho > 0.0)) {
      *solve_status = BREAKDOWN;
      return;
    }
    for (int it = 1; it <= max_iter; ++it) {
      apply(h, L, p.data(), q.data());
      const double pq = dev ? column_dot(d, q.data(), p.data())
                            : (h.device_order ? dot(n, p.data(), q.data()) : pdot(p.data(), q.data()));
      if (!(pq > 0.0)) {
        *solve_status = BREAKDOWN;
        return;
      }
      const double alpha = rho / pq;
      par([&](Index lo, Index hi) {
        for (Index i = lo; i < hi; ++i) {
          x[i] += alpha * p[i];
          r[i] -= alpha * q[i];
        }
      });
      const double rn = std::sqrt(fused ? column_dot(d, r.data(), r.data(), false, nc) : gsdot(r));
      if (res_hist) res_hist[it] = rn;
      *iters = it;
      stamp(it);
      if (rn / r0 <= tol) return;
      if (rn / r0 > 1e4) {
        *solve_status = DIVERGED;
        return;
      }
      std::fill(z.begin(), z.end(), 0.0);
      // the fused post-sweep forms r.z in its forward pass (k_jacobi_t3 PCGF 2, thomas_rz); the
      // two-columns-per-thread kernel sums r_k z_k in its back substitution
      std::vector<double> rzc(fused && nc == 1 ? h.lv[L].ncells : 0);
      vcycle(h, L, r.data(), z.data(), rzc.empty() ? nullptr : rzc.data());
      const double rho_new = fused ? (nc == 1 ? column_reduce(d, rzc, 1)
                                              : column_dot(d, r.data(), z.data(), true, nc))
                                   : dotv(r, z);
      if (!(rho_new > 0.0)) {
        *solve_status = BREAKDOWN;
        return;
      }
      const double beta = rho_new / rho;
      rho = rho_new;
      par([&](Index lo, Index hi) {
        for (Index i = lo; i < hi; ++i) p[i] = z[i] + beta * p[i];
      });
    }
    *solve_status = NOT_CONVERGED;
  });
}

// Preconditioned Richardson and right-preconditioned BiCGStab (the krylov
// module the reference specifies but does not ship; design decisions :443-447).  Restated in the
// operation order of the device drivers (tpmg_host.cpp tpmg_richardson / tpmg_bicgstab) so the
// strict GPU build is comparable bit for bit: dots in the device's grid-stride tree (Cartesian
// problems), scalars in double on the host, element-wise updates as k_vec_lin writes them.
namespace {
struct Outer {
  const Hier& h;
  int L;
  Index n;
  bool dev;
  DevOrder d;
  explicit Outer(const Hier& hh)
      : h(hh), L(static_cast<int>(hh.lv.size()) - 1), n(hh.lv[L].ncells * hh.nz),
        dev(hh.cart_nx > 0 && hh.device_order), d{hh.cart_nx, hh.cart_ny, hh.nz} {}
  double dotv(const std::vector<double>& a, const std::vector<double>& b) const {
    return dev ? tile_or_gridstride_dot(d, a.data(), b.data()) : dot(n, a.data(), b.data());
  }
  // M^{-1} r: mu V-cycles on A e = r from e = 0
  void precond(int mu, const std::vector<double>& r, std::vector<double>& e) const {
    std::fill(e.begin(), e.end(), 0.0);
    for (int i = 0; i < mu; ++i) vcycle(h, L, r.data(), e.data());
  }
};
}  // namespace

int tpmgo_richardson(tpmgo_hier H, const double* f, double* x, double tol, int max_iter, int mu,
                     double* res_hist, int* iters, int* solve_status) {
  return guard([&] {
    if (max_iter < 0 || mu < 1) throw Error(E_CONFIG, "richardson: max_iter >= 0, mu >= 1");
    const Outer o(H->h);
    const Index n = o.n;
    std::vector<double> r(f, f + n), e(n), xv(n, 0.0), y(n);
    const double r0 = std::sqrt(o.dotv(r, r));
    if (res_hist) res_hist[0] = r0;
    *iters = 0;
    *solve_status = OK;
    std::copy(xv.begin(), xv.end(), x);
    if (r0 == 0.0) return;
    for (int it = 1; it <= max_iter; ++it) {
      o.precond(mu, r, e);
      for (Index i = 0; i < n; ++i) xv[i] = xv[i] + e[i];
      apply(o.h, o.L, xv.data(), y.data());
      for (Index i = 0; i < n; ++i) r[i] = f[i] - y[i];
      const double rn = std::sqrt(o.dotv(r, r));
      if (res_hist) res_hist[it] = rn;
      *iters = it;
      std::copy(xv.begin(), xv.end(), x);
      if (rn / r0 <= tol) return;
      if (!(rn / r0 <= 1e4)) {
        *solve_status = DIVERGED;
        return;
      }
    }
    *solve_status = NOT_CONVERGED;
  });
}

int tpmgo_bicgstab(tpmgo_hier H, const double* f, double* x, double tol, int max_iter, int mu,
                   double* res_hist, int* iters, int* solve_status) {
  return guard([&] {
    if (max_iter < 0 || mu < 1) throw Error(E_CONFIG, "bicgstab: max_iter >= 0, mu >= 1");
    const Outer o(H->h);
    const Index n = o.n;
    std::vector<double> r(f, f + n), rh(f, f + n), p(n, 0.0), v(n, 0.0), ph(n), s(n), sh(n),
        t(n), xv(n, 0.0);
    struct Out {  // x is written back on every exit
      double* x;
      const std::vector<double>& v;
      ~Out() { std::copy(v.begin(), v.end(), x); }
    } out{x, xv};
    const double r0 = std::sqrt(o.dotv(r, r));
    if (res_hist) res_hist[0] = r0;
    *iters = 0;
    *solve_status = OK;
    if (r0 == 0.0) return;
    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    for (int it = 1; it <= max_iter; ++it) {
      const double rho = o.dotv(rh, r);
      if (!(std::fabs(rho) >= 1e-30 * r0 * r0)) {
        *solve_status = BREAKDOWN;
        return;
      }
      const double beta = (rho / rho_prev) * (alpha / omega);
      for (Index i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
      o.precond(mu, p, ph);
      apply(o.h, o.L, ph.data(), v.data());
      const double rv = o.dotv(rh, v);
      if (!(rv != 0.0)) {
        *solve_status = BREAKDOWN;
        return;
      }
      alpha = rho / rv;
      for (Index i = 0; i < n; ++i) s[i] = r[i] - alpha * v[i];
      const double sn = std::sqrt(o.dotv(s, s));
      if (sn / r0 <= tol) {
        for (Index i = 0; i < n; ++i) xv[i] = xv[i] + alpha * ph[i];
        if (res_hist) res_hist[it] = sn;
        *iters = it;
        return;
      }
      o.precond(mu, s, sh);
      apply(o.h, o.L, sh.data(), t.data());
      const double tt = o.dotv(t, t);
      const double ts = o.dotv(t, s);
      if (!(tt != 0.0)) {
        *solve_status = BREAKDOWN;
        return;
      }
      omega = ts / tt;
      for (Index i = 0; i < n; ++i) xv[i] = (xv[i] + alpha * ph[i]) + omega * sh[i];
      for (Index i = 0; i < n; ++i) r[i] = s[i] - omega * t[i];
      const double rn = std::sqrt(o.dotv(r, r));
      if (res_hist) res_hist[it] = rn;
      *iters = it;
      if (rn / r0 <= tol) return;
      if (!(rn / r0 <= 1e4)) {
        *solve_status = DIVERGED;
        return;
      }
      if (!(omega != 0.0)) {
        *solve_status = BREAKDOWN;
        return;
      }
      rho_prev = rho;
    }
    *solve_status = NOT_CONVERGED;
  });
}

double tpmgo_dot(int64_t n, const double* a, const double* b) { return dot(n, a, b); }

}  // extern "C"
