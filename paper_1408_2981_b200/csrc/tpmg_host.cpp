#include <cstdio>
// tpmg_host.cpp -- C-ABI implementation (include/tpmg_b200.h): hierarchy setup, device
// resident fields, the V-cycle / PCG drivers and the NCCL halo + all-reduce plumbing.
//
// Setup restates the reference's hierarchy construction for the doubly periodic Cartesian
// grid (assemble_hatted, discretization.hpp:144-184; restrict_profiles, multigrid.hpp:158-201;
// build_hierarchy_coefficients, multigrid.hpp:242-272) on the host, once; every hot-path
// operation runs as sm_100a kernels (tpmg_kernels.cu) on the context's stream.  There is
// no CPU fallback: without a CUDA device every entry point returns TPMG_E_CUDA.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tpmg_b200.h"
#include "tpmg_kernels.cuh"

namespace {

using tpmg::Halo;
using tpmg::LevelCoef;
using tpmg::VertCoef;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

#define CUDA_CHECK(x)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw Error(TPMG_E_CUDA, std::string(#x ": ") + cudaGetErrorString(e_));          \
  } while (0)

// ---- NCCL, resolved lazily (single-GPU runs never load it) ------------------------------
struct Nccl {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // optional (NCCL >= 2.18): the second communicator of the side-stream halo exchanges
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;

  void load() {
    if (handle) return;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names)
      if ((handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!handle) throw Error(TPMG_E_NCCL, "cannot load libnccl.so.2");
    auto sym = [&](const char* s) {
      void* p = dlsym(handle, s);
      if (!p) throw Error(TPMG_E_NCCL, std::string("NCCL symbol missing: ") + s);
      return p;
    };
    GetUniqueId = (decltype(GetUniqueId))sym("ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))sym("ncclCommInitRank");
    CommDestroy = (decltype(CommDestroy))sym("ncclCommDestroy");
    Send = (decltype(Send))sym("ncclSend");
    Recv = (decltype(Recv))sym("ncclRecv");
    GroupStart = (decltype(GroupStart))sym("ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))sym("ncclGroupEnd");
    AllReduce = (decltype(AllReduce))sym("ncclAllReduce");
    AllGather = (decltype(AllGather))sym("ncclAllGather");
    GetErrorString = (decltype(GetErrorString))sym("ncclGetErrorString");
    CommSplit = (decltype(CommSplit))dlsym(handle, "ncclCommSplit");
  }
};
Nccl g_nccl;

std::atomic<int64_t> g_nccl_calls{0};  // NCCL API calls issued by this process (tpmg_nccl_call_count)
#define NCCL_CHECK(x)                                                                   \
  do {                                                                                  \
    g_nccl_calls.fetch_add(1, std::memory_order_relaxed);                               \
    ncclResult_t r_ = (x);                                                              \
    if (r_ != ncclSuccess)                                                              \
      throw Error(TPMG_E_NCCL, std::string(#x ": ") + g_nccl.GetErrorString(r_));       \
  } while (0)

thread_local std::string g_global_error;

// ---- CUDA-IPC transport (tpmg_init_ipc) ----------------------------------------------------
// Ranks of one node (any GPUs, or several processes sharing one GPU) exchange halos by writing
// straight into their neighbours' receive buffers (cudaIpcMemHandle mappings) and reduce their
// dot products through a POSIX shared-memory segment.  Every step is ordered by HOST barriers
// in that segment around stream synchronisations: no kernel ever waits on another rank.
constexpr int kIpcMaxRanks = 64, kIpcMaxLevels = 24;
constexpr int kIpcGatherMax = 32768;  // tile partials per rank (tiles up to 2048 x 2048 columns)
constexpr uint64_t kIpcMagic = 0x32637069676d7074ull;  // "tpmgipc2"
struct IpcShm {
  std::atomic<uint64_t> magic;
  std::atomic<uint32_t> count, gen, abort;
  int32_t world;
  double vals[2][kIpcMaxRanks];  // per-rank contributions, alternating phases
  double gather[2][kIpcMaxRanks][kIpcGatherMax];  // per-rank tile partials, alternating phases
  cudaIpcMemHandle_t handles[kIpcMaxRanks][kIpcMaxLevels][3];  // receive buffers per level / set
  cudaIpcMemHandle_t agg[kIpcMaxRanks];  // each rank's replicated copy of the agglomerated level's f
};
static_assert(std::atomic<uint32_t>::is_always_lock_free, "process-shared atomics");

}  // namespace

// ---- handles ------------------------------------------------------------------------------
struct tpmg_context_s {
  int device = 0;
  int rank = 0, world = 1, px = 1, py = 1, rx = 0, ry = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  // side stream of the halo exchanges that overlap compute (exchange_f_async), with its own
  // communicator so that its NCCL operations never interleave with the main stream's
  cudaStream_t side = nullptr;
  ncclComm_t comm2 = nullptr;
  // TPMG_LOOPBACK=2 at tpmg_init, one rank: a one-rank NCCL communicator, so that the loopback
  // halos and reductions go through the NCCL transport itself (send / receive to self)
  bool nccl_self = false;
  tpmg::Launch side_launch() { return tpmg::Launch{side, &launches}; }
  // CUDA-IPC transport (tpmg_init_ipc): shared segment, reduction phase, pinned staging
  IpcShm* ipc = nullptr;
  int ipc_phase = 0;
  double* ipc_host = nullptr;
  std::string last_error;
  int64_t launches = 0;
  tpmg::Launch launch() { return tpmg::Launch{stream, &launches}; }
  int rank_of(int x, int y) const {
    x = (x % px + px) % px;
    y = (y % py + py) % py;
    return y * px + x;
  }
};

namespace {

template <typename T>
struct DevBufT {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    n = count;
    CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  }
  void upload(const T* h, size_t count) {
    alloc(count);
    CUDA_CHECK(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice));
  }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBufT() {
    if (p) cudaFree(p);
  }
};
using DevBuf = DevBufT<double>;

struct Level {
  // replicated (coarse-grid agglomeration): the whole global level on every rank, solved
  // redundantly; nx/ny are the global dims and x0 = y0 = 0
  bool rep = false;
  int nx = 0, ny = 0;          // local tile
  int gnx = 0, gny = 0;        // global level dims
  int x0 = 0, y0 = 0;          // tile offset (global cell index)
  int64_t plane = 0;
  // host copies of the hatted horizontal factors (tile local)
  std::vector<double> bh, ah, xh, sh;  // sh: 2*plane (east, north)
  DevBuf d_bh, d_ah, d_xh, d_sw, d_se, d_ss, d_sn;
  // dense hatted components of the partial / full coefficient modes, [k][y][x]
  int cm = tpmg::CM_FACT;
  bool uni = false;  // one edge scalar on the whole (global) level: LevelCoef::uni
  DevBuf d_ard, d_bd, d_xid, d_swd, d_sed, d_ssd, d_snd;
  // indirect levels (tpmg_hier_create_generic): neighbour / edge tables, per-edge alpha_s hat,
  // and (coarse levels) the child table on the next finer level
  int nnb = 0;
  DevBufT<int> d_nbr, d_cedge, d_children;
  DevBuf d_shg;
  DevBuf u, t, f;              // V-cycle work: home iterate, ping-pong partner, rhs
  DevBuf send, recv;           // multi-GPU face buffers [W|E|S|N]
  DevBuf send2, recv2;         // finest level: a second set (z and p_old before the fused A p)
  DevBuf send3, recv3;         // two-cell halo with corners (tpmg::Halo2 layout, fused R(f - A u))
  DevBuf d_ringc;              // coefficient scalars on the 1-cell ring around the tile
  DevBuf sendF, recvF;         // face halo of f posted early on the side stream (exchange_f_async)
  bool f_pending = false;      // recvF is being filled for this level's next residual + restriction
  // IPC transport: where this rank's W / E / S / N faces land in the neighbours' receive
  // buffers (per halo set), and its deep pieces W, E, S, N, SW, SE, NW, NE
  double* peer[2][4] = {{nullptr, nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr, nullptr}};
  double* peer3[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  DevBuf d_piv, d_cpt;         // coarse levels: pre-factorised column blocks (LevelCoef::piv)
  LevelCoef coef(int nz) const {
    LevelCoef c;
    c.nx = nx; c.ny = ny; c.nz = nz; c.plane = plane;
    c.bh = d_bh.p; c.ah = d_ah.p; c.xh = d_xh.p;
    c.sw = d_sw.p; c.se = d_se.p; c.ss = d_ss.p; c.sn = d_sn.p;
    c.cm = cm;
    c.uni = uni && cm == tpmg::CM_FACT;
    c.ard = d_ard.p; c.bd = d_bd.p; c.xid = d_xid.p;
    c.swd = d_swd.p; c.sed = d_sed.p; c.ssd = d_ssd.p; c.snd = d_snd.p;
    c.nnb = nnb; c.nbr = d_nbr.p; c.cedge = d_cedge.p; c.shg = d_shg.p;
    c.piv = d_piv.p; c.cpt = d_cpt.p;
    return c;
  }
};

}  // namespace

struct tpmg_hierarchy_s {
  tpmg_context ctx = nullptr;
  int nz = 0;
  bool xi = false;
  int cm = 0;  // coefficient mode (tpmg::CoefMode)
  bool generic = false;     // indirect levels (tpmg_hier_create_generic)
  tpmg::GenRule rule{};
  double relax = 1.0;
  int prolongation = 0, restriction = 0;
  std::vector<int> nu_pre, nu_post;
  std::vector<Level> lv;  // coarsest .. finest
  std::vector<double> bv, sv, av, xv;
  DevBuf d_bv, d_sv, d_av, d_xv, d_vr, d_vx;
  // finest-level PCG / V-cycle work vectors
  DevBuf r, z, p, q, tmp;
  DevBuf p2;                // second search-direction buffer of the fused A p pass (ping-pong)
  int pcur = 0;             // which of p / p2 holds the current direction
  bool fused_ap = false;    // x += a p_old; p = z + b p_old; q = A p in one pass
  bool q_in_sweep = false;  // ... and q = A p re-formed in the r-update sweep (q not stored)
  // Richardson / BiCGStab work vectors (allocated on first use) and operation counts of the
  // last outer solve (2 preconditioner + 2 operator applications per BiCGStab step)
  DevBuf k_rh, k_p, k_v, k_ph, k_s, k_sh, k_t;
  int64_t n_precond = 0, n_matvec = 0;
  double* pbuf(int i) { return i == 0 ? p.p : p2.p; }
  DevBuf partials, scal;  // reduction partials; scalars s[0..7]
  DevBuf gathered;        // multi-rank: every rank's tile partials (gather_partials)
  // coarse-grid agglomeration: levels below agg_la are replicated; agg_tile holds this rank's
  // block of level agg_la-1 (restricted right-hand side on the way down, the prolongation's
  // coarse block on the way up), agg_gather every rank's block (NCCL all-gather), agg_peers
  // every rank's copy of level agg_la-1's f (CUDA-IPC)
  int agg_la = 0;
  DevBuf agg_tile, agg_gather;
  tpmg::PeerDst agg_peers{};
  int* d_err = nullptr;
  double* h_scal = nullptr;  // pinned
  // one-rank PCG host loop: per-iteration scalars published into mapped pinned memory by the
  // iteration's last kernel (k_pcg_publish); the host polls the sequence number
  tpmg::PcgPublish* h_pub = nullptr;  // host view (cudaHostAllocMapped)
  tpmg::PcgPublish* d_pub = nullptr;  // device alias
  unsigned* d_seq = nullptr;
  unsigned host_seq = 0;
  // tpmg_pcg_host_batch: double-buffered finest-level right-hand sides and iterates, staging
  // buffers of the layout permutations, the copy stream and its events (allocated on first use)
  struct Batch {
    DevBuf F[2], X[2], stage_in, stage_out;
    cudaStream_t copy = nullptr;
    cudaEvent_t up[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr},
                down[2] = {nullptr, nullptr};
  } bat;
  bool use_graphs = true;
  // Loopback halos (TPMG_LOOPBACK=1 at creation, one rank): every multi-rank device path —
  // face packing, the send -> recv transfer (here device copies onto this rank itself, the
  // periodic neighbour of a 1x1 process grid), kernels reading halos from the recv buffers, the
  // multi-rank schedule (no fused A p / residual+restriction / prolongation) — runs on one GPU,
  // so the GPU parity tests cover it (TPMG_LOOPBACK=2: with NCCL itself as the transport)
  bool loopback = false;
  bool multi() const;
  bool nccl_self() const;
  bool nccl_reduce() const;
  bool pcg_fused = false;  // PCG vector work fused into the finest-level smoother sweeps
  const double* f_first = nullptr;  // fused PCG: the right-hand side the first iteration reads
  bool fuse_rr = true;     // fused residual + transpose restriction (TPMG_FUSE_RR=0 disables)
  // Captured PCG work, one graph per key: the prologue (r_0 dot, V-cycle, rho dot) per
  // right-hand side, the first iteration per (right-hand side, iterate), the later iterations
  // per (iterate, direction parity).  probes: the probe pairs every launch records.
  struct GraphKey {
    int tag;
    const void* a;
    const void* b;
    bool operator==(const GraphKey& o) const { return tag == o.tag && a == o.a && b == o.b; }
  };
  struct GraphKeyHash {
    size_t operator()(const GraphKey& k) const {
      return std::hash<const void*>()(k.a) * 31u + std::hash<const void*>()(k.b) * 7u + (size_t)k.tag;
    }
  };
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
    uint32_t probes = 0;
  };
  std::unordered_map<GraphKey, Graph, GraphKeyHash> graphs;
  // device-side PCG loop (iterations 2..): one graph per iterate buffer, a while-node whose body
  // holds two iterations (both direction parities), the second behind an if-node
  std::unordered_map<const void*, cudaGraphExec_t> loop_graphs;
  int64_t loop_kernels_per_iter = 0;
  tpmg::PcgLoop* d_loop = nullptr;
  tpmg::PcgLoop* h_loop = nullptr;  // pinned
  DevBuf d_hist;                    // |r| per iteration, kLoopHist entries
  static constexpr int kLoopHist = 4096;
  // Kernel probes (tpmg_kernel_probe): a CUDA event pair around each probed finest-level PCG
  // launch, recorded as external event nodes when the iteration is captured into its graph, read
  // after every iteration's synchronisation: live per-launch durations inside a solve.
  struct Probe {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    double total_ms = 0.0;
    int64_t launches = 0;
  };
  static constexpr int kProbes = 16;
  bool probe_on = false;
  Probe probes[kProbes];
  uint32_t probe_pending = 0;  // pairs recorded by the work queued since the last collection
  std::vector<void*> ipc_mapped;  // neighbours' receive buffers opened through CUDA IPC
  // exchange_f_async: per level, f ready on the main stream / halo landed on the side stream
  std::vector<cudaEvent_t> ev_fsrc, ev_fdone;
  // which direction buffer's face halo set 1 (recv2) holds: the fused A p pass of a decomposed
  // run exchanges p_new once and both the r-update sweep and the next A p pass read it
  const double* p_halo_of = nullptr;
  int finest() const { return (int)lv.size() - 1; }
  VertCoef vcoef() const {
    VertCoef v{d_bv.p, d_sv.p, d_av.p, d_xv.p};
    v.vr = d_vr.p;
    v.vx = d_vx.p;
    return v;
  }
  // interleaved copies of the vertical vectors (VertCoef::vr / vx) for the kernels' bulk staging
  void upload_vertical_rows() {
    const size_t nzz = bv.size();
    std::vector<double> vr(4 * nzz), vx(2 * nzz);
    for (size_t k = 0; k < nzz; ++k) {
      vr[4 * k] = bv[k];
      vr[4 * k + 1] = sv[k];
      vr[4 * k + 2] = av[k];
      vr[4 * k + 3] = av[k + 1];
      vx[2 * k] = xv[k];
      vx[2 * k + 1] = xv[k + 1];
    }
    d_vr.upload(vr.data(), vr.size());
    d_vx.upload(vx.data(), vx.size());
  }
  ~tpmg_hierarchy_s() {
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t e : {bat.up[i], bat.done[i], bat.down[i]})
        if (e) cudaEventDestroy(e);
    if (bat.copy) cudaStreamDestroy(bat.copy);
    for (cudaEvent_t e : ev_fsrc) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_fdone) cudaEventDestroy(e);
    for (auto& pr : probes) {
      if (pr.e0) cudaEventDestroy(pr.e0);
      if (pr.e1) cudaEventDestroy(pr.e1);
    }
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    for (auto& kv : loop_graphs) cudaGraphExecDestroy(kv.second);
    if (d_loop) cudaFree(d_loop);
    if (h_loop) cudaFreeHost(h_loop);
    if (d_err) cudaFree(d_err);
    if (h_scal) cudaFreeHost(h_scal);
    if (h_pub) cudaFreeHost(h_pub);
    if (d_seq) cudaFree(d_seq);
  }
};

bool tpmg_hierarchy_s::multi() const { return ctx->world > 1 || loopback; }
// loopback halos carried by NCCL itself (a one-rank communicator): every send / receive of the
// NCCL transport, its all-gathers and all-reduces run on one GPU, inside the captured graphs too
bool tpmg_hierarchy_s::nccl_self() const { return loopback && ctx->nccl_self; }
// the rank's reductions go over NCCL
bool tpmg_hierarchy_s::nccl_reduce() const { return !ctx->ipc && (ctx->world > 1 || nccl_self()); }

namespace {
// level l is split over the ranks (halo exchanges); replicated levels behave like one rank
bool lmulti(tpmg_hierarchy h, int l) { return h->multi() && !h->lv[l].rep; }
}  // namespace

namespace {

// host barrier of the IPC ranks (sense by generation count); a rank that fails or times out
// raises the abort flag so the others fail instead of waiting forever
void ipc_barrier(tpmg_context ctx) {
  IpcShm* S = ctx->ipc;
  const uint32_t g = S->gen.load(std::memory_order_acquire);
  if (S->count.fetch_add(1, std::memory_order_acq_rel) + 1 == (uint32_t)ctx->world) {
    S->count.store(0, std::memory_order_relaxed);
    S->gen.fetch_add(1, std::memory_order_acq_rel);
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0; S->gen.load(std::memory_order_acquire) == g; ++spin) {
    if (S->abort.load(std::memory_order_relaxed))
      throw Error(TPMG_E_NCCL, "ipc transport: another rank failed");
    if (spin > 64) sched_yield();
    if ((spin & 1023) == 0 &&
        std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
      S->abort.store(1);
      throw Error(TPMG_E_NCCL, "ipc transport: barrier timeout (a rank is missing)");
    }
  }
}

// sum (or max) of one double over the ranks, in rank order 0..world-1 on every rank
double ipc_allreduce(tpmg_context ctx, double v, bool max_op) {
  IpcShm* S = ctx->ipc;
  const int ph = ctx->ipc_phase;
  ctx->ipc_phase ^= 1;
  S->vals[ph][ctx->rank] = v;
  ipc_barrier(ctx);
  double acc = S->vals[ph][0];
  for (int r = 1; r < ctx->world; ++r) {
    const double x = S->vals[ph][r];
    acc = max_op ? (x > acc ? x : acc) : acc + x;
  }
  return acc;
}

}  // namespace

struct tpmg_field_s {
  tpmg_hierarchy h = nullptr;
  int level = 0;
  DevBuf buf;
};

namespace {

template <typename Fn>
int guard(tpmg_context ctx, Fn&& fn) {
  try {
    fn();
    return TPMG_OK;
  } catch (const Error& e) {
    if (ctx) ctx->last_error = e.what();
    g_global_error = e.what();
    return e.code;
  } catch (const tpmg::LaunchError& e) {
    const std::string m = std::string("kernel launch failed in ") + e.kernel + ": " +
                          cudaGetErrorString(e.err);
    if (ctx) ctx->last_error = m;
    g_global_error = m;
    return TPMG_E_CUDA;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->last_error = "host allocation failed";
    return TPMG_E_CUDA;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_error = e.what();
    g_global_error = e.what();
    return TPMG_E_CONFIG;
  }
}

void check_finite(const double* p, size_t n, const char* what) {
  if (!p) throw Error(TPMG_E_CONFIG, std::string("missing array ") + what);
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i]))
      throw Error(TPMG_E_NONFINITE, std::string("non-finite values in ") + what);
}

// Number of levels of the horizontal hierarchy: tiles must stay even so the 2x2 children of
// a coarse cell share a rank; depth 0 coarsens while the global grid stays >= 4 per dimension.
int plan_levels(int64_t NX, int64_t NY, int px, int py, int depth, bool linear) {
  if (NX < 1 || NY < 1 || px < 1 || py < 1) throw Error(TPMG_E_CONFIG, "bad decomposition");
  if (NX % px || NY % py)
    throw Error(TPMG_E_CONFIG, "global grid does not split evenly over the process grid");
  int levels = 1;
  int64_t a = NX / px, b = NY / py, ga = NX, gb = NY;
  if (depth <= 0) {
    while (a % 2 == 0 && b % 2 == 0 && ga / 2 >= 4 && gb / 2 >= 4) {
      a /= 2; b /= 2; ga /= 2; gb /= 2; ++levels;
    }
  } else {
    for (int l = 1; l < depth; ++l) {
      if (a % 2 || b % 2) throw Error(TPMG_E_CONFIG, "tile does not coarsen to the requested depth");
      a /= 2; b /= 2; ga /= 2; gb /= 2;
    }
    levels = depth;
  }
  if (linear && levels > 1 && (ga < 3 || gb < 3))
    throw Error(TPMG_E_CONFIG, "linear transfers need >= 3 coarse cells per dimension");
  return levels;
}

// Coarse-grid agglomeration (tpmg_mg_config::agglomerate > 0 on a decomposed run): the levels
// are those of the GLOBAL grid; the finest level and every coarser one whose global grid has more
// than `agg` columns and splits evenly over the process grid stay decomposed, the rest (a prefix
// of coarse levels) are replicated.  The restriction into the finest replicated level forms
// each rank's block of it, so that level's dims must split evenly too.  Returns the number of
// levels; *la = the coarsest decomposed level (0: none replicated).
int plan_agg(int64_t NX, int64_t NY, int px, int py, int depth, bool linear, int64_t agg, int* la) {
  const int levels = plan_levels(NX, NY, 1, 1, depth, linear);
  auto splits = [&](int l) {
    const int sh = levels - 1 - l;
    return ((NX >> sh) % px) == 0 && ((NY >> sh) % py) == 0;
  };
  if (!splits(levels - 1))
    throw Error(TPMG_E_CONFIG, "global grid does not split evenly over the process grid");
  int a = levels - 1;
  while (a > 0) {
    const int c = a - 1, sh = levels - 1 - c;
    if ((NX >> sh) * (NY >> sh) <= agg || !splits(c)) break;
    a = c;
  }
  if (a > 0 && !splits(a - 1)) {
    if (a == levels - 1)
      throw Error(TPMG_E_CONFIG,
                  "agglomeration: the finest tile does not coarsen evenly onto its ranks' blocks");
    ++a;  // a is decomposed, so its tiles split: the gather lands one level higher
  }
  *la = a;
  return levels;
}

// ---- halos -----------------------------------------------------------------------------
// Exchange the 1-cell faces of u on level l with the 4 neighbouring ranks and return the
// view the kernels read across the tile faces.  Dimensions with a single rank wrap onto the
// tile itself (periodic) without any copy.
// The view of halo set `set` of level l as exchange() leaves it (receive buffers across the
// dimensions with several ranks, the periodic self views across the others).
Halo halo_view(tpmg_hierarchy h, int l, const double* u, int set) {
  tpmg_context ctx = h->ctx;
  Level& L = h->lv[l];
  Halo H = tpmg::self_halo(u, L.nx, L.ny, L.plane);
  if (!lmulti(h, l)) return H;
  const bool xs = ctx->px > 1 || h->loopback, ys = ctx->py > 1 || h->loopback;
  const int64_t nwe = (int64_t)L.ny * h->nz, nsn = (int64_t)L.nx * h->nz;
  double* rW = (set ? L.recv2 : L.recv).p;
  if (xs) {
    H.p[0] = rW; H.sk[0] = L.ny; H.st[0] = 1;
    H.p[1] = rW + nwe; H.sk[1] = L.ny; H.st[1] = 1;
  }
  if (ys) {
    H.p[2] = rW + 2 * nwe; H.sk[2] = L.nx; H.st[2] = 1;
    H.p[3] = rW + 2 * nwe + nsn; H.sk[3] = L.nx; H.st[3] = 1;
  }
  return H;
}

Halo exchange(tpmg_hierarchy h, int l, const double* u, int set = 0) {
  tpmg_context ctx = h->ctx;
  Level& L = h->lv[l];
  DevBuf& SB = set ? L.send2 : L.send;
  DevBuf& RB = set ? L.recv2 : L.recv;
  if (!lmulti(h, l)) return tpmg::self_halo(u, L.nx, L.ny, L.plane);
  const int nz = h->nz;
  const int64_t nwe = (int64_t)L.ny * nz, nsn = (int64_t)L.nx * nz;
  double* sW = SB.p;
  double* sE = sW + nwe;
  double* sS = sE + nwe;
  double* sN = sS + nsn;
  double* rW = RB.p;
  double* rE = rW + nwe;
  double* rS = rE + nwe;
  double* rN = rS + nsn;
  // each face is packed straight to where it lands: this rank's own receive buffer (loopback:
  // the periodic neighbour of a 1x1 process grid is the rank itself), the neighbour's receive
  // buffer (CUDA-IPC peer mapping), or the send buffer NCCL transfers
  if (ctx->ipc) {
    // the neighbours' kernels reading their receive buffers are done (barrier after each
    // rank's stream drained), then every rank writes its faces into them, then all land
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    ipc_barrier(ctx);
    tpmg::FaceDst dst{{ctx->px > 1 ? L.peer[set][0] : nullptr, ctx->px > 1 ? L.peer[set][1] : nullptr,
                       ctx->py > 1 ? L.peer[set][2] : nullptr, ctx->py > 1 ? L.peer[set][3] : nullptr}};
    tpmg::launch_pack_faces(ctx->launch(), L.nx, L.ny, nz, u, dst);
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    ipc_barrier(ctx);
  } else if (h->loopback && !h->nccl_self()) {  // this rank is its own neighbour on every side
    tpmg::launch_pack_faces(ctx->launch(), L.nx, L.ny, nz, u, tpmg::FaceDst{{rE, rW, rN, rS}});
  } else {
  const bool xs = ctx->px > 1 || h->loopback, ys = ctx->py > 1 || h->loopback;
  tpmg::launch_pack_faces(ctx->launch(), L.nx, L.ny, nz, u,
                          tpmg::FaceDst{{xs ? sW : nullptr, xs ? sE : nullptr,
                                         ys ? sS : nullptr, ys ? sN : nullptr}});
  NCCL_CHECK(g_nccl.GroupStart());
  if (xs) {
    const int west = ctx->rank_of(ctx->rx - 1, ctx->ry), east = ctx->rank_of(ctx->rx + 1, ctx->ry);
    NCCL_CHECK(g_nccl.Send(sW, nwe, ncclDouble, west, ctx->comm, ctx->stream));
    NCCL_CHECK(g_nccl.Send(sE, nwe, ncclDouble, east, ctx->comm, ctx->stream));
    NCCL_CHECK(g_nccl.Recv(rE, nwe, ncclDouble, east, ctx->comm, ctx->stream));
    NCCL_CHECK(g_nccl.Recv(rW, nwe, ncclDouble, west, ctx->comm, ctx->stream));
  }
  if (ys) {
    const int south = ctx->rank_of(ctx->rx, ctx->ry - 1), north = ctx->rank_of(ctx->rx, ctx->ry + 1);
    NCCL_CHECK(g_nccl.Send(sS, nsn, ncclDouble, south, ctx->comm, ctx->stream));
    NCCL_CHECK(g_nccl.Send(sN, nsn, ncclDouble, north, ctx->comm, ctx->stream));
    NCCL_CHECK(g_nccl.Recv(rN, nsn, ncclDouble, north, ctx->comm, ctx->stream));
    NCCL_CHECK(g_nccl.Recv(rS, nsn, ncclDouble, south, ctx->comm, ctx->stream));
  }
  NCCL_CHECK(g_nccl.GroupEnd());
  }
  return halo_view(h, l, u, set);
}

// ---- two-cell halo with corners (tpmg::Halo2) ---------------------------------------------
// Piece d of the deep exchange (d = W, E, S, N, SW, SE, NW, NE) goes to the neighbour in
// direction d and lands in its Halo2 slot kOpp[d]; offsets of the slots in a recv3 buffer.
constexpr int kDeepDx[8] = {-1, 1, 0, 0, -1, 1, -1, 1};
constexpr int kDeepDy[8] = {0, 0, -1, 1, -1, -1, 1, 1};
constexpr int kOpp[8] = {1, 0, 3, 2, 7, 6, 5, 4};
int64_t deep_size(const Level& L, int nz) {
  return (4 * (int64_t)L.ny + 4 * (int64_t)L.nx + 16) * nz;
}
void deep_offsets(const Level& L, int nz, int64_t off[8], int64_t cnt[8]) {
  const int64_t we = 2 * (int64_t)L.ny * nz, sn = 2 * (int64_t)L.nx * nz, c = 4 * (int64_t)nz;
  const int64_t o[8] = {0, we, 2 * we, 2 * we + sn, 2 * we + 2 * sn, 2 * we + 2 * sn + c,
                        2 * we + 2 * sn + 2 * c, 2 * we + 2 * sn + 3 * c};
  const int64_t n[8] = {we, we, sn, sn, c, c, c, c};
  for (int d = 0; d < 8; ++d) { off[d] = o[d]; cnt[d] = n[d]; }
}
// piece d is exchanged when its direction crosses a dimension with several ranks (loopback:
// every dimension); corners need both
bool deep_live(tpmg_hierarchy h, int d) {
  const bool xs = h->ctx->px > 1 || h->loopback, ys = h->ctx->py > 1 || h->loopback;
  return (kDeepDx[d] == 0 || xs) && (kDeepDy[d] == 0 || ys);
}

// Exchange u's two-cell faces and 2x2 corners on level l (the fused residual + transpose
// restriction of a decomposed run reads u two cells beyond its tile) and return the view.
tpmg::Halo2 exchange_deep(tpmg_hierarchy h, int l, const double* u) {
  tpmg_context ctx = h->ctx;
  Level& L = h->lv[l];
  tpmg::Halo2 H{};
  H.xs = lmulti(h, l) && (ctx->px > 1 || h->loopback);
  H.ys = lmulti(h, l) && (ctx->py > 1 || h->loopback);
  if (!lmulti(h, l)) return H;
  const int nz = h->nz;
  int64_t off[8], cnt[8];
  deep_offsets(L, nz, off, cnt);
  for (int d = 0; d < 8; ++d) H.p[d] = L.recv3.p + off[d];
  tpmg::DeepDst dst{};
  if (ctx->ipc) {
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    ipc_barrier(ctx);
    for (int d = 0; d < 8; ++d) dst.p[d] = deep_live(h, d) ? L.peer3[d] : nullptr;
    tpmg::launch_pack_deep(ctx->launch(), L.nx, L.ny, nz, u, dst);
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    ipc_barrier(ctx);
  } else if (h->loopback && !h->nccl_self()) {  // every neighbour is this rank: piece d lands in slot kOpp[d]
    for (int d = 0; d < 8; ++d) dst.p[d] = L.recv3.p + off[kOpp[d]];
    tpmg::launch_pack_deep(ctx->launch(), L.nx, L.ny, nz, u, dst);
  } else {
    for (int d = 0; d < 8; ++d) dst.p[d] = deep_live(h, d) ? L.send3.p + off[d] : nullptr;
    tpmg::launch_pack_deep(ctx->launch(), L.nx, L.ny, nz, u, dst);
    // every rank sends in the order d = 0..7 and receives slot kOpp[d] from the neighbour in
    // direction kOpp[d] in the same order, so that the pieces two ranks exchange in several
    // directions (px or py = 2) are matched in order
    NCCL_CHECK(g_nccl.GroupStart());
    for (int d = 0; d < 8; ++d) {
      if (!deep_live(h, d)) continue;
      NCCL_CHECK(g_nccl.Send(L.send3.p + off[d], cnt[d], ncclDouble,
                             ctx->rank_of(ctx->rx + kDeepDx[d], ctx->ry + kDeepDy[d]), ctx->comm,
                             ctx->stream));
      const int o = kOpp[d];
      NCCL_CHECK(g_nccl.Recv(L.recv3.p + off[o], cnt[o], ncclDouble,
                             ctx->rank_of(ctx->rx + kDeepDx[o], ctx->ry + kDeepDy[o]), ctx->comm,
                             ctx->stream));
    }
    NCCL_CHECK(g_nccl.GroupEnd());
  }
  return H;
}

// ---- halo exchanges that overlap compute ---------------------------------------------------
// A coarse level's right-hand side f_l is formed by the residual + restriction of level l+1
// and its face halo is next needed by level l's own residual + restriction, after its
// pre-sweeps (which read f_l only in their own columns).  The exchange is therefore posted on
// the side stream right away (its own buffers, its own NCCL communicator) and overlaps those
// sweeps; the main stream waits for it only at the residual + restriction.  Loopback and NCCL
// runs; the CUDA-IPC transport orders its exchanges by host barriers and keeps them in place.
bool f_async_ok(tpmg_hierarchy h) {
  tpmg_context ctx = h->ctx;
  if (!h->multi() || ctx->ipc || !ctx->side) return false;
  return (h->loopback && !h->nccl_self()) || ctx->comm2;
}

void exchange_f_async(tpmg_hierarchy h, int l, const double* f) {
  tpmg_context ctx = h->ctx;
  Level& L = h->lv[l];
  if (!f_async_ok(h) || !L.recvF.p) return;
  if (h->ev_fsrc.empty()) {
    h->ev_fsrc.assign(h->lv.size(), nullptr);
    h->ev_fdone.assign(h->lv.size(), nullptr);
    for (size_t i = 0; i < h->lv.size(); ++i) {
      CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_fsrc[i], cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_fdone[i], cudaEventDisableTiming));
    }
  }
  const int nz = h->nz;
  const int64_t nwe = (int64_t)L.ny * nz, nsn = (int64_t)L.nx * nz;
  double* sW = L.sendF.p;
  double* sE = sW + nwe;
  double* sS = sE + nwe;
  double* sN = sS + nsn;
  double* rW = L.recvF.p;
  double* rE = rW + nwe;
  double* rS = rE + nwe;
  double* rN = rS + nsn;
  CUDA_CHECK(cudaEventRecord(h->ev_fsrc[l], ctx->stream));
  CUDA_CHECK(cudaStreamWaitEvent(ctx->side, h->ev_fsrc[l], 0));
  if (h->loopback && !h->nccl_self()) {
    tpmg::launch_pack_faces(ctx->side_launch(), L.nx, L.ny, nz, f, tpmg::FaceDst{{rE, rW, rN, rS}});
  } else {
    const bool xs = ctx->px > 1 || h->loopback, ys = ctx->py > 1 || h->loopback;
    tpmg::launch_pack_faces(ctx->side_launch(), L.nx, L.ny, nz, f,
                            tpmg::FaceDst{{xs ? sW : nullptr, xs ? sE : nullptr,
                                           ys ? sS : nullptr, ys ? sN : nullptr}});
    NCCL_CHECK(g_nccl.GroupStart());
    if (xs) {
      const int west = ctx->rank_of(ctx->rx - 1, ctx->ry), east = ctx->rank_of(ctx->rx + 1, ctx->ry);
      NCCL_CHECK(g_nccl.Send(sW, nwe, ncclDouble, west, ctx->comm2, ctx->side));
      NCCL_CHECK(g_nccl.Send(sE, nwe, ncclDouble, east, ctx->comm2, ctx->side));
      NCCL_CHECK(g_nccl.Recv(rE, nwe, ncclDouble, east, ctx->comm2, ctx->side));
      NCCL_CHECK(g_nccl.Recv(rW, nwe, ncclDouble, west, ctx->comm2, ctx->side));
    }
    if (ys) {
      const int south = ctx->rank_of(ctx->rx, ctx->ry - 1), north = ctx->rank_of(ctx->rx, ctx->ry + 1);
      NCCL_CHECK(g_nccl.Send(sS, nsn, ncclDouble, south, ctx->comm2, ctx->side));
      NCCL_CHECK(g_nccl.Send(sN, nsn, ncclDouble, north, ctx->comm2, ctx->side));
      NCCL_CHECK(g_nccl.Recv(rN, nsn, ncclDouble, north, ctx->comm2, ctx->side));
      NCCL_CHECK(g_nccl.Recv(rS, nsn, ncclDouble, south, ctx->comm2, ctx->side));
    }
    NCCL_CHECK(g_nccl.GroupEnd());
  }
  CUDA_CHECK(cudaEventRecord(h->ev_fdone[l], ctx->side));
  L.f_pending = true;
}

// the main stream waits for level l's posted f halo; returns its view (exchange()'s layout)
Halo finish_f_async(tpmg_hierarchy h, int l, const double* f) {
  tpmg_context ctx = h->ctx;
  Level& L = h->lv[l];
  CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, h->ev_fdone[l], 0));
  L.f_pending = false;
  Halo H = tpmg::self_halo(f, L.nx, L.ny, L.plane);
  const bool xs = ctx->px > 1 || h->loopback, ys = ctx->py > 1 || h->loopback;
  const int64_t nwe = (int64_t)L.ny * h->nz, nsn = (int64_t)L.nx * h->nz;
  double* rW = L.recvF.p;
  if (xs) {
    H.p[0] = rW; H.sk[0] = L.ny; H.st[0] = 1;
    H.p[1] = rW + nwe; H.sk[1] = L.ny; H.st[1] = 1;
  }
  if (ys) {
    H.p[2] = rW + 2 * nwe; H.sk[2] = L.nx; H.st[2] = 1;
    H.p[3] = rW + 2 * nwe + nsn; H.sk[3] = L.nx; H.st[3] = 1;
  }
  return H;
}

// s[slot] = global sum of the per-block partials.
void probe_begin(tpmg_hierarchy h, int id);
void probe_end(tpmg_hierarchy h, int id);
// every rank's `nb` partials into h->gathered, rank r at r*nb
void gather_partials(tpmg_hierarchy h, int nb) {
  tpmg_context ctx = h->ctx;
  if ((int64_t)nb * ctx->world > (int64_t)h->gathered.n)
    throw Error(TPMG_E_CAP, "gather buffer too small");
  if (ctx->ipc) {  // through the shared segment (phase alternation as in ipc_allreduce)
    IpcShm* S = ctx->ipc;
    if (nb > kIpcGatherMax) throw Error(TPMG_E_CAP, "ipc transport: too many tile partials");
    const int ph = ctx->ipc_phase;
    ctx->ipc_phase ^= 1;
    CUDA_CHECK(cudaMemcpyAsync(S->gather[ph][ctx->rank], h->partials.p, (size_t)nb * 8,
                               cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    ipc_barrier(ctx);
    for (int r = 0; r < ctx->world; ++r)
      CUDA_CHECK(cudaMemcpyAsync(h->gathered.p + (int64_t)r * nb, S->gather[ph][r], (size_t)nb * 8,
                                 cudaMemcpyHostToDevice, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  } else {
    NCCL_CHECK(g_nccl.AllGather(h->partials.p, h->gathered.p, (size_t)nb, ncclDouble, ctx->comm,
                                ctx->stream));
  }
}
// s[slot] = global sum of the per-block partials.  `tile_level` >= 0: the partials are the
// 32x4-tile partials of that level (k_dot_tiles / the fused kernels).  A decomposed run then
// gathers every rank's tile partials and reduces them in the global tile order of a one-rank
// run: the dot products -- and with them the whole PCG solve -- are bitwise independent of the
// number of ranks.  Other layouts: local fixed-order sum, then a sum over the ranks.
void finish_dot(tpmg_hierarchy h, int nblocks, int slot, int tile_level = -1) {
  tpmg_context ctx = h->ctx;
  if ((ctx->world > 1 || h->nccl_self()) && tile_level >= 0) {
    const Level& L = h->lv[tile_level];
    if (tpmg::dot_tiles_ok(L.nx, L.ny) && nblocks == (L.nx / 32) * (L.ny / 4)) {
      gather_partials(h, nblocks);
      probe_begin(h, TPMG_K_REDUCE);
      tpmg::launch_reduce_tiles(ctx->launch(), h->gathered.p, nblocks, L.nx / 32,
                                L.ny / 4, ctx->px, ctx->py, h->scal.p + slot);
      probe_end(h, TPMG_K_REDUCE);
      return;
    }
  }
  probe_begin(h, TPMG_K_REDUCE);
  tpmg::launch_reduce(ctx->launch(), h->partials.p, nblocks, h->scal.p + slot);
  probe_end(h, TPMG_K_REDUCE);
  if (ctx->ipc) {
    CUDA_CHECK(cudaMemcpyAsync(ctx->ipc_host, h->scal.p + slot, sizeof(double),
                               cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    ctx->ipc_host[1] = ipc_allreduce(ctx, ctx->ipc_host[0], false);
    CUDA_CHECK(cudaMemcpyAsync(h->scal.p + slot, ctx->ipc_host + 1, sizeof(double),
                               cudaMemcpyHostToDevice, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  } else if (h->nccl_reduce()) {
    NCCL_CHECK(g_nccl.AllReduce(h->scal.p + slot, h->scal.p + slot, 1, ncclDouble, ncclSum,
                                ctx->comm, ctx->stream));
  }
}

// ---- kernel probes ----------------------------------------------------------------------
// an event record on the library stream; inside a stream capture an external event node of
// the graph (so the event is re-recorded by every launch of the graph)
void probe_record(tpmg_hierarchy h, cudaEvent_t e) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  CUDA_CHECK(cudaStreamIsCapturing(h->ctx->stream, &st));
  if (st == cudaStreamCaptureStatusActive)
    CUDA_CHECK(cudaEventRecordWithFlags(e, h->ctx->stream, cudaEventRecordExternal));
  else
    CUDA_CHECK(cudaEventRecord(e, h->ctx->stream));
}
void probe_begin(tpmg_hierarchy h, int id) {
  if (!h->probe_on) return;
  auto& pr = h->probes[id];
  if (!pr.e0) {
    CUDA_CHECK(cudaEventCreate(&pr.e0));
    CUDA_CHECK(cudaEventCreate(&pr.e1));
  }
  probe_record(h, pr.e0);
}
void probe_end(tpmg_hierarchy h, int id) {
  if (!h->probe_on) return;
  probe_record(h, h->probes[id].e1);
  h->probe_pending |= 1u << id;
}
// after a synchronisation: add the durations of the pairs recorded since the last one
void probe_collect(tpmg_hierarchy h) {
  for (int id = 0; id < tpmg_hierarchy_s::kProbes; ++id) {
    if (!(h->probe_pending & (1u << id))) continue;
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, h->probes[id].e0, h->probes[id].e1));
    h->probes[id].total_ms += ms;
    h->probes[id].launches += 1;
  }
  h->probe_pending = 0;
}

// a.b of two fields of level l: on a tiled Cartesian level in the fused kernels' tile layout
// (k_dot_tiles), so that every PCG dot of a decomposed run reduces to the one-rank bits
void dot_into(tpmg_hierarchy h, int l, const double* a, const double* b, int slot) {
  Level& L = h->lv[l];
  int nb = 0;
  const bool tiles = !h->generic && tpmg::dot_tiles_ok(L.nx, L.ny);
  if (tiles) tpmg::launch_dot_tiles(h->ctx->launch(), L.nx, L.ny, h->nz, a, b, h->partials.p, &nb);
  else tpmg::launch_dot(h->ctx->launch(), L.plane * h->nz, a, b, h->partials.p, &nb);
  if (L.rep) {  // a replicated level is whole on every rank: no sum over the ranks
    tpmg::launch_reduce(h->ctx->launch(), h->partials.p, nb, h->scal.p + slot);
    return;
  }
  finish_dot(h, nb, slot, tiles ? l : -1);
}

// ---- hot-path building blocks ------------------------------------------------------------
void apply_level(tpmg_hierarchy h, int l, int mode, const double* u, const double* f, double* y,
                 int dot_slot = -1, int set = 0) {
  Level& L = h->lv[l];
  const Halo H = exchange(h, l, u, set);
  int nb = 0;
  tpmg::launch_apply(h->ctx->launch(), h->vcoef(), L.coef(h->nz), h->xi, mode, u, H, f, y,
                     dot_slot >= 0 ? h->partials.p : nullptr, &nb);
  if (dot_slot >= 0) finish_dot(h, nb, dot_slot, l);
}

// One line-Jacobi sweep.  With `fz` the sweep also does fused PCG work (see PcgFuse) and its
// per-tile partials are reduced into scalar slot `slot`.
void sweep(tpmg_hierarchy h, int l, const double* u_in, const double* f, double* out,
           const tpmg::PcgFuse* fz = nullptr, int slot = -1, const tpmg::ProSrc* pro = nullptr,
           int probe = -1, const Halo* p_halo = nullptr) {
  Level& L = h->lv[l];
  // the haloed input: u, or p when the zero-guess sweep forms q = A p itself (p_halo: p's halo
  // already exchanged by the caller)
  Halo H = u_in ? exchange(h, l, u_in)
                : (fz && fz->p ? (p_halo ? *p_halo : exchange(h, l, fz->p))
                               : tpmg::self_halo(out, L.nx, L.ny, L.plane));
  int nb = 0;
  if (probe >= 0) probe_begin(h, probe);
  tpmg::launch_jacobi(h->ctx->launch(), h->vcoef(), L.coef(h->nz), h->xi, u_in, H, f, out,
                      h->relax, h->d_err, fz, &nb, pro);
  if (probe >= 0) probe_end(h, probe);
  if (fz) finish_dot(h, nb, slot, l);
}

// fine level lf -> coarse lf-1: coarse = R (f - A u).  `scratch` is a free fine-level buffer.
void restrict_plain(tpmg_hierarchy h, int lf, const double* fine, double* coarse, int kind);

// ---- coarse-grid agglomeration ---------------------------------------------------------------
// Every rank's block of the replicated level lc (this rank's in h->agg_tile, formed by the
// restriction from the decomposed level lc+1) into dst, the whole level, on every rank.
void agg_gather(tpmg_hierarchy h, int lc, double* dst) {
  tpmg_context ctx = h->ctx;
  const Level& F = h->lv[lc + 1];
  const Level& C = h->lv[lc];
  const int bnx = F.nx / 2, bny = F.ny / 2, nz = h->nz;
  const int64_t bn = (int64_t)bnx * bny * nz;
  if (ctx->ipc) {
    // the all-gather as NVLink peer stores: this rank's block goes straight into every rank's
    // copy (between barriers: every copy's readers are done, then every block has landed)
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    ipc_barrier(ctx);
    tpmg::launch_block_to_peers(ctx->launch(), h->agg_tile.p, bnx, bny, nz, F.x0 / 2, F.y0 / 2,
                                C.nx, C.ny, h->agg_peers);
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    ipc_barrier(ctx);
    if (dst != C.f.p)
      CUDA_CHECK(cudaMemcpyAsync(dst, C.f.p, (size_t)C.plane * nz * sizeof(double),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
  } else if (h->nccl_reduce()) {
    NCCL_CHECK(g_nccl.AllGather(h->agg_tile.p, h->agg_gather.p, (size_t)bn, ncclDouble, ctx->comm,
                                ctx->stream));
    tpmg::launch_blocks_to_level(ctx->launch(), h->agg_gather.p, ctx->px, ctx->py, bnx, bny, nz,
                                 dst);
  } else {  // loopback: the one block is the whole level
    tpmg::launch_blocks_to_level(ctx->launch(), h->agg_tile.p, 1, 1, bnx, bny, nz, dst);
  }
}
// crossing from a decomposed level lf to a replicated level lf-1
bool agg_boundary(tpmg_hierarchy h, int lf) { return h->lv[lf - 1].rep && !h->lv[lf].rep; }

void resid_restrict_impl(tpmg_hierarchy h, int lf, const double* u, const double* f,
                         double* coarse, double* scratch, bool probe);
// fine level lf -> coarse lf-1: coarse = R (f - A u); at the agglomeration boundary the rank's
// block is formed, then gathered into the replicated level on every rank
void resid_restrict(tpmg_hierarchy h, int lf, const double* u, const double* f, double* coarse,
                    double* scratch, bool probe = false) {
  if (!agg_boundary(h, lf)) return resid_restrict_impl(h, lf, u, f, coarse, scratch, probe);
  resid_restrict_impl(h, lf, u, f, h->agg_tile.p, scratch, probe);
  agg_gather(h, lf - 1, coarse);
}

void resid_restrict_impl(tpmg_hierarchy h, int lf, const double* u, const double* f,
                         double* coarse, double* scratch, bool probe) {
  Level& F = h->lv[lf];
  // f's face halo posted early by exchange_f_async (joined here whichever path runs)
  const bool f_posted = F.f_pending;
  const Halo hf_posted = f_posted ? finish_f_async(h, lf, f) : Halo{};
  if (h->generic) {
    apply_level(h, lf, tpmg::APPLY_RESID, u, f, scratch);
    restrict_plain(h, lf, scratch, coarse, -1);
    return;
  }
  if (h->restriction == TPMG_RESTRICT_SUMMATION) {
    const Halo H = exchange(h, lf, u);
    tpmg::launch_resid_restrict_sum(h->ctx->launch(), h->vcoef(), F.coef(h->nz), h->xi, u, H, f,
                                    coarse);
  } else if (h->fuse_rr && tpmg::resid_restrict_T_fusable(F.coef(h->nz)) &&
             (!lmulti(h, lf) || (F.d_ringc.p && tpmg::resid_restrict_T2_fusable(F.coef(h->nz))))) {
    // decomposed: u's two-cell halo with corners and f's face halo first (the ring residuals
    // the transpose stencil reaches outside the tile)
    const tpmg::Halo2 hu = exchange_deep(h, lf, u);
    const Halo hf = f_posted ? hf_posted : exchange(h, lf, f, 0);
    if (probe) probe_begin(h, TPMG_K_RESID_RESTRICT);
    tpmg::launch_resid_restrict_T(h->ctx->launch(), h->vcoef(), F.coef(h->nz), h->xi, u, hu, f,
                                  hf, F.d_ringc.p, coarse);
    if (probe) probe_end(h, TPMG_K_RESID_RESTRICT);
  } else {
    apply_level(h, lf, tpmg::APPLY_RESID, u, f, scratch);
    const Halo Hr = exchange(h, lf, scratch);
    tpmg::launch_restrict_transpose(h->ctx->launch(), F.nx / 2, F.ny / 2, h->nz, scratch, Hr,
                                    coarse);
  }
}

void restrict_plain(tpmg_hierarchy h, int lf, const double* fine, double* coarse, int kind = -1) {
  Level& C = h->lv[lf - 1];
  const Level& F = h->lv[lf];
  if (kind < 0) kind = h->restriction;
  if (h->generic) {
    tpmg::launch_restrict_gen(h->ctx->launch(), C.coef(h->nz), C.d_children.p, h->rule,
                              h->lv[lf].plane, fine, coarse, kind == TPMG_RESTRICT_TRANSPOSE);
    return;
  }
  // the coarse block of this rank's fine tile (at the agglomeration boundary: gathered after)
  const bool gather = agg_boundary(h, lf);
  double* dst = gather ? h->agg_tile.p : coarse;
  if (kind == TPMG_RESTRICT_SUMMATION) {
    tpmg::launch_restrict_sum(h->ctx->launch(), F.nx / 2, F.ny / 2, h->nz, fine, dst);
  } else {
    const Halo Hf = exchange(h, lf, fine);
    tpmg::launch_restrict_transpose(h->ctx->launch(), F.nx / 2, F.ny / 2, h->nz, fine, Hf, dst);
  }
  if (gather) agg_gather(h, lf - 1, coarse);
}

void prolong_level(tpmg_hierarchy h, int lc, const double* coarse, double* fine, bool add,
                   bool probe = false, int kind = -1) {
  Level& F = h->lv[lc + 1];
  const bool linear = (kind < 0 ? h->prolongation : kind) == TPMG_PROLONG_LINEAR;
  if (h->generic) {
    Level& C = h->lv[lc];
    tpmg::launch_prolong_gen(h->ctx->launch(), C.coef(h->nz), C.d_children.p, h->rule, F.plane,
                             coarse, fine, linear, add);
    return;
  }
  if (agg_boundary(h, lc + 1)) {
    // from this rank's block of the replicated coarse level; its halo is read straight from the
    // replicated copy (periodic views)
    const Level& C = h->lv[lc];
    const int bnx = F.nx / 2, bny = F.ny / 2, x0 = F.x0 / 2, y0 = F.y0 / 2;
    tpmg::launch_block_from_level(h->ctx->launch(), coarse, C.nx, C.ny, h->nz, x0, y0, bnx, bny,
                                  h->agg_tile.p);
    const Halo Hc = linear ? tpmg::block_halo(coarse, C.nx, C.ny, C.plane, x0, y0, bnx, bny)
                           : Halo{};
    if (probe) probe_begin(h, TPMG_K_PROLONG_ADD);
    tpmg::launch_prolong(h->ctx->launch(), F.nx, F.ny, h->nz, h->agg_tile.p, Hc, fine, linear, add);
    if (probe) probe_end(h, TPMG_K_PROLONG_ADD);
    return;
  }
  const Halo Hc = linear ? exchange(h, lc, coarse) : Halo{};
  if (probe) probe_begin(h, TPMG_K_PROLONG_ADD);
  tpmg::launch_prolong(h->ctx->launch(), F.nx, F.ny, h->nz, coarse, Hc, fine, linear, add);
  if (probe) probe_end(h, TPMG_K_PROLONG_ADD);
}

void fill(tpmg_hierarchy h, double* p, int64_t n, double v) {
  if (v == 0.0) CUDA_CHECK(cudaMemsetAsync(p, 0, n * sizeof(double), h->ctx->stream));
  else tpmg::launch_fill(h->ctx->launch(), n, p, v);
}

// v_cycle, multigrid.hpp:276-299.  On return the iterate is in A; B is scratch of the same
// level.  zero: A's content is ignored and treated as 0 (the preconditioner / coarse case).
//
// pcg_fuse (finest level of a fused PCG iteration, f == r): the first sweep from zero also does
// r -= alpha q and |r|^2 (slot 2); the last post-sweep also does r.z (slot 3).
// f_pre (fused PCG, first iteration): the zero-guess pre-sweep reads the right-hand side from
// f_pre and writes the updated r to fz.r == f, so r = f_0 never needs a device copy
void vcycle(tpmg_hierarchy h, int l, const double* f, double* A, double* B, bool zero,
            bool pcg_fuse = false, const double* p_dir = nullptr,
            const double* f_pre = nullptr, const Halo* p_halo = nullptr) {
  Level& L = h->lv[l];
  const int64_t n = L.plane * h->nz;
  const int npre = h->nu_pre[l], npost = h->nu_post[l], total = npre + npost;
  // an early-posted f halo (exchange_f_async) is consumed by the residual + restriction of the
  // same V-cycle; drop any left over by a V-cycle an error interrupted
  for (int m = 0; m < l; ++m) h->lv[m].f_pending = false;
  double* cur = A;
  auto other = [&](double* c) { return c == A ? B : A; };
  int s0 = 0;
  tpmg::PcgFuse fz;
  if (pcg_fuse) {
    // with p_dir the pre-sweep forms q = A p_dir itself and q is never stored
    fz.q = p_dir ? nullptr : h->q.p;
    fz.p = p_dir;
    fz.r = h->r.p;
    fz.s = h->scal.p;
    fz.partials = h->partials.p;
  }
  if (zero) {
    if (npre > 0) {
      // first sweep from zero writes where the last sweep must end in A
      cur = ((total - 1) % 2 == 0) ? A : B;
      sweep(h, l, nullptr, (pcg_fuse && f_pre) ? f_pre : f, cur, pcg_fuse ? &fz : nullptr, 2,
            nullptr, pcg_fuse ? TPMG_K_PCG_RUPDATE : -1, p_halo);
      s0 = 1;
    } else {
      cur = (npost % 2 == 0) ? A : B;
      fill(h, cur, n, 0.0);
    }
  }
  for (int s = s0; s < npre; ++s) {
    double* out = other(cur);
    sweep(h, l, cur, f, out);
    cur = out;
  }
  // the prolongation rides in the first post-sweep where that kernel can take it (one rank)
  tpmg::ProSrc pro;
  bool fuse_pro = false;
  if (l > 0) {
    Level& C = h->lv[l - 1];
    resid_restrict(h, l, cur, f, C.f.p, other(cur), pcg_fuse);
    // decomposed: f_{l-1}'s face halo travels while level l-1 pre-smooths
    if (l - 1 > 0 && C.recvF.p) exchange_f_async(h, l - 1, C.f.p);
    vcycle(h, l - 1, C.f.p, C.u.p, C.t.p, true);
    fuse_pro = npost > 0 && !h->multi() && !h->generic &&
               h->prolongation == TPMG_PROLONG_LINEAR && tpmg::jacobi_prolong_fusable(L.coef(h->nz));
    if (fuse_pro) {
      pro.ec = C.u.p;
      pro.cnx = (int)C.nx;
      pro.cny = (int)C.ny;
    } else {
      prolong_level(h, l - 1, C.u.p, cur, true, pcg_fuse);
    }
  }
  for (int s = 0; s < npost; ++s) {
    double* out = other(cur);
    const bool last = pcg_fuse && s + 1 == npost;
    sweep(h, l, cur, f, out, last ? &fz : nullptr, 3, s == 0 && fuse_pro ? &pro : nullptr,
          last ? TPMG_K_PCG_POSTSWEEP : -1);
    cur = out;
  }
  if (cur != A)
    CUDA_CHECK(cudaMemcpyAsync(A, cur, n * sizeof(double), cudaMemcpyDeviceToDevice,
                               h->ctx->stream));
}

// Synchronise and return the zero-pivot flag (all-reduced over the ranks) without acting on it.
int sync_err(tpmg_hierarchy h) {
  // the error flag rides behind the queued work into pinned memory: one synchronisation
  int* h_err = reinterpret_cast<int*>(h->h_scal + 7);
  // multi-rank: every rank must take the same exit decision, or the ranks that did not see a
  // zero pivot would enter the next iteration's collectives alone and hang
  if (h->ctx->ipc) {
    int e = 0;
    CUDA_CHECK(cudaMemcpyAsync(&e, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, h->ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(h->ctx->stream));
    const int any = (int)ipc_allreduce(h->ctx, (double)e, true);
    CUDA_CHECK(cudaMemcpyAsync(h->d_err, &any, sizeof(int), cudaMemcpyHostToDevice, h->ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(h->ctx->stream));
  } else if (h->nccl_reduce()) {
    NCCL_CHECK(g_nccl.AllReduce(h->d_err, h->d_err, 1, ncclInt32, ncclMax, h->ctx->comm,
                                h->ctx->stream));
  }
  CUDA_CHECK(cudaMemcpyAsync(h_err, h->d_err, sizeof(int), cudaMemcpyDeviceToHost,
                             h->ctx->stream));
  CUDA_CHECK(cudaStreamSynchronize(h->ctx->stream));
  return *h_err;
}

void clear_err(tpmg_hierarchy h) {
  CUDA_CHECK(cudaMemsetAsync(h->d_err, 0, sizeof(int), h->ctx->stream));
}

void sync_check(tpmg_hierarchy h) {
  if (sync_err(h)) {
    clear_err(h);
    throw Error(TPMG_E_SINGULAR, "thomas_solve: zero pivot");
  }
}

double read_scalar(tpmg_hierarchy h, int slot) {
  CUDA_CHECK(cudaMemcpyAsync(h->h_scal + slot, h->scal.p + slot, sizeof(double),
                             cudaMemcpyDeviceToHost, h->ctx->stream));
  sync_check(h);
  return h->h_scal[slot];
}

tpmg_field_s* field_of(tpmg_field f) {
  if (!f) throw Error(TPMG_E_CONFIG, "null field");
  return f;
}

void same_hier(tpmg_hierarchy h, tpmg_field f) {
  if (field_of(f)->h != h) throw Error(TPMG_E_SHAPE, "field belongs to another hierarchy");
}

// PCG iteration body (no host synchronisation).  Scalars: s[0]=rho, s[1]=p.q, s[2]=r.r,
// s[3]=rho_new.
// Fused schedule (h->pcg_fused): [x += a_prev p_old; p = z + b p_old; rho <- rho_new] (skipped
// on the first iteration, where p = z, x = 0); q = A p with p.q; V-cycle whose first finest
// sweep does r -= a q and r.r, and whose last finest sweep forms r.z.  The x update of the
// final iteration is applied after the loop (k_pcg_xfinal).  Every element is computed with
// the same operations as the plain schedule: q = A p, p.q; x += a p, r -= a q, r.r;
// z = V(r); r.z; p = z + b p.
// part (fused A p schedule): 0 the whole iteration; 1 only its head, the direction update + A p
// pass and its dot (run_iteration launches it eagerly, so that the launch of the graph holding
// the rest overlaps that 0.9 ms pass instead of idling the GPU); 2 only the rest
void pcg_iteration(tpmg_hierarchy h, double* x, bool first, int pc, int part = 0) {
  const int L = h->finest();
  const int64_t n = h->lv[L].plane * h->nz;
  tpmg_context ctx = h->ctx;
  if (h->pcg_fused) {
    if (!first && h->fused_ap) {
      // p_reuse: p_old's halo is already in set 1 (exchanged once, right after the pass that
      // formed it, for that iteration's r-update sweep)
      const bool p_reuse = h->multi() && h->q_in_sweep;
      if (part != 2) {
        // direction update and A p in one pass; p_new goes to the other buffer
        Level& F = h->lv[L];
        double* po = h->pbuf(pc);
        int nb = 0;
        // halos of z and p_old (single rank: the periodic self views, no copy)
        const Halo Hz = exchange(h, L, h->z.p, 0);
        const Halo Hp = p_reuse ? halo_view(h, L, po, 1) : exchange(h, L, po, 1);
        probe_begin(h, TPMG_K_PCG_DIRECTION);
        tpmg::launch_pcg_ap(ctx->launch(), h->vcoef(), F.coef(h->nz), h->xi, h->z.p, Hz, po, Hp,
                            h->pbuf(pc ^ 1),
                            h->q_in_sweep ? nullptr : h->q.p, x, h->scal.p, h->partials.p, &nb);
        probe_end(h, TPMG_K_PCG_DIRECTION);
        tpmg::launch_copy_scalar(ctx->launch(), h->scal.p, 0, 3);
        finish_dot(h, nb, 1, L);
      }
      if (part == 1) return;
      Halo Hpn;
      if (p_reuse) Hpn = exchange(h, L, h->pbuf(pc ^ 1), 1);
      vcycle(h, L, h->r.p, h->z.p, h->tmp.p, true, true,
             h->q_in_sweep ? h->pbuf(pc ^ 1) : nullptr, nullptr, p_reuse ? &Hpn : nullptr);
      return;
    } else {
      if (!first) {
        tpmg::launch_pcg_px(ctx->launch(), n, h->scal.p, h->z.p, h->pbuf(pc), x);
        tpmg::launch_copy_scalar(ctx->launch(), h->scal.p, 0, 3);
      }
      // decomposed fused A p schedule: p's halo goes to set 1, where the next A p pass reads
      // it as p_old's
      apply_level(h, L, tpmg::APPLY_AU, h->pbuf(pc), nullptr, h->q.p, 1,
                  h->multi() && h->q_in_sweep ? 1 : 0);
    }
    vcycle(h, L, h->r.p, h->z.p, h->tmp.p, true, true, nullptr, first ? h->f_first : nullptr);
    return;
  }
  apply_level(h, L, tpmg::APPLY_AU, h->p.p, nullptr, h->q.p, 1);
  int nb = 0;
  tpmg::launch_pcg_xr(ctx->launch(), n, h->scal.p, x, h->r.p, h->p.p, h->q.p, h->partials.p, &nb);
  finish_dot(h, nb, 2);
  vcycle(h, L, h->r.p, h->z.p, h->tmp.p, true);
  dot_into(h, L, h->r.p, h->z.p, 3);
  tpmg::launch_pcg_p(ctx->launch(), n, h->scal.p, h->z.p, h->p.p);
  tpmg::launch_copy_scalar(ctx->launch(), h->scal.p, 0, 3);
}

// Wait for the iteration's k_pcg_publish: poll the sequence number in mapped pinned memory
// (the host wakes as soon as it lands, no stream synchronisation); every few thousand polls ask
// the stream whether it failed.  Then the scalars go to h_scal and a zero pivot raises the
// reference's singular_error, as sync_check does.
int wait_publish_raw(tpmg_hierarchy h) {
  const unsigned want = ++h->host_seq;
  volatile unsigned* seq = &h->h_pub->seq;
  for (uint64_t spin = 0; *seq != want; ++spin) {
    if ((spin & 4095) == 4095) {
      const cudaError_t e = cudaStreamQuery(h->ctx->stream);
      if (e != cudaSuccess && e != cudaErrorNotReady) CUDA_CHECK(e);
      if (e == cudaSuccess && *seq != want)
        throw Error(TPMG_E_CUDA, "pcg: iteration scalars were not published");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  for (int i = 0; i < 4; ++i) h->h_scal[i] = h->h_pub->s[i];
  return h->h_pub->err;
}
void wait_publish(tpmg_hierarchy h) {
  if (wait_publish_raw(h)) {
    CUDA_CHECK(cudaMemsetAsync(h->d_err, 0, sizeof(int), h->ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(h->ctx->stream));
    throw Error(TPMG_E_SINGULAR, "thomas_solve: zero pivot");
  }
}

// the iteration's scalars to the host through k_pcg_publish (one rank; see wait_publish)
bool publish_ok(tpmg_hierarchy h) { return h->h_pub && !h->multi(); }
void publish(tpmg_hierarchy h) {
  if (publish_ok(h))
    tpmg::launch_pcg_publish(h->ctx->launch(), h->scal.p, h->d_err, h->d_seq, h->d_pub);
}

// Run fn() as the graph cached under key (captured on first use); fn() eagerly where graphs
// are off or the transport orders its exchanges on the host (IPC).
template <class Fn>
void run_graph(tpmg_hierarchy h, const tpmg_hierarchy_s::GraphKey& key, Fn&& fn) {
  tpmg_context ctx = h->ctx;
  if (!h->use_graphs || ctx->ipc) {
    fn();
    return;
  }
  auto it = h->graphs.find(key);
  if (it == h->graphs.end()) {
    cudaGraph_t g;
    const int64_t before = ctx->launches;
    const uint32_t eager_probes = h->probe_pending;  // recorded eagerly before the capture
    h->probe_pending = 0;
    CUDA_CHECK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    try {
      fn();
    } catch (...) {
      cudaStreamEndCapture(ctx->stream, &g);
      throw;
    }
    CUDA_CHECK(cudaStreamEndCapture(ctx->stream, &g));
    tpmg_hierarchy_s::Graph G;
    G.kernels = ctx->launches - before;
    ctx->launches = before;
    G.probes = h->probe_pending;  // recorded by every launch of this graph
    h->probe_pending = eager_probes;
    CUDA_CHECK(cudaGraphInstantiate(&G.exec, g, 0));
    cudaGraphDestroy(g);
    it = h->graphs.emplace(key, G).first;
  }
  CUDA_CHECK(cudaGraphLaunch(it->second.exec, ctx->stream));
  ctx->launches += it->second.kernels;
  h->probe_pending |= it->second.probes;
}

enum GraphTag { G_PROLOGUE = 1, G_FIRST = 2, G_ITER = 3 };

void run_iteration(tpmg_hierarchy h, double* x, bool first) {
  const int pc = h->pcur;
  // the fused A p pass moves the direction to the other buffer
  if (h->pcg_fused && h->fused_ap && !first) h->pcur ^= 1;
  if (first) {  // the fused schedule's first iteration reads the right-hand side f_first
    run_graph(h, {G_FIRST, x, h->pcg_fused ? h->f_first : nullptr}, [&] {
      pcg_iteration(h, x, true, pc);
      publish(h);
    });
    return;
  }
  // fused A p schedule: the head pass eagerly, the rest as the graph (whose launch then
  // overlaps the head instead of idling the GPU)
  const bool split = h->pcg_fused && h->fused_ap && h->use_graphs && !h->ctx->ipc;
  if (split) pcg_iteration(h, x, false, pc, 1);
  run_graph(h, {G_ITER, x, h->pbuf(pc)}, [&] {  // keyed by the direction parity
    pcg_iteration(h, x, false, pc, split ? 2 : 0);
    publish(h);
  });
}

// Opt-in (TPMG_DEVLOOP=1, read per solve): bench.py measures the same solve time either way
// (24.9 GDOF/s) once the host loop synchronises once per iteration, and ncu does not profile
// kernels inside conditional graph bodies, so the host loop stays the default.
bool device_loop_ok(tpmg_hierarchy h, int max_iter) {
  const char* e = getenv("TPMG_DEVLOOP");
  const int env = e ? atoi(e) : 0;
  return env != 0 && h->use_graphs && h->pcg_fused && !h->multi() &&
         max_iter < tpmg_hierarchy_s::kLoopHist;
}

cudaGraphExec_t loop_graph(tpmg_hierarchy h, double* x) {
  auto found = h->loop_graphs.find(x);
  if (found != h->loop_graphs.end()) return found->second;
  tpmg_context ctx = h->ctx;
  cudaStream_t s = ctx->stream;
  if (!h->d_loop) {
    CUDA_CHECK(cudaMalloc(&h->d_loop, sizeof(tpmg::PcgLoop)));
    CUDA_CHECK(cudaMallocHost(&h->h_loop, sizeof(tpmg::PcgLoop)));
    h->d_hist.alloc(tpmg_hierarchy_s::kLoopHist);
  }
  cudaGraph_t g;
  CUDA_CHECK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw, hi;
  CUDA_CHECK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp{};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wn;
  CUDA_CHECK(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  CUDA_CHECK(cudaGraphConditionalHandleCreate(&hi, body, 0, 0));
  const int64_t before = ctx->launches;
  // first half: direction parity 0, then the test (which also arms the second half)
  CUDA_CHECK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
  std::vector<cudaGraphNode_t> tail;
  try {
    pcg_iteration(h, x, false, 0);
    tpmg::launch_pcg_check(ctx->launch(), h->scal.p, h->d_hist.p, h->d_loop, hw, hi, 1);
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CUDA_CHECK(cudaStreamGetCaptureInfo(s, &cs, nullptr, nullptr, &deps, &nd));
    tail.assign(deps, deps + nd);
  } catch (...) {
    cudaStreamEndCapture(s, &body);
    cudaGraphDestroy(g);
    throw;
  }
  CUDA_CHECK(cudaStreamEndCapture(s, &body));
  const int64_t per_iter = ctx->launches - before;
  cudaGraphNodeParams ip{};
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = hi;
  ip.conditional.type = cudaGraphCondTypeIf;
  ip.conditional.size = 1;
  cudaGraphNode_t in;
  CUDA_CHECK(cudaGraphAddNode(&in, body, tail.data(), tail.size(), &ip));
  cudaGraph_t ibody = ip.conditional.phGraph_out[0];
  // second half: the other parity (the fused A p pass alternates the direction buffers)
  CUDA_CHECK(cudaStreamBeginCaptureToGraph(s, ibody, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
  try {
    pcg_iteration(h, x, false, h->fused_ap ? 1 : 0);
    tpmg::launch_pcg_check(ctx->launch(), h->scal.p, h->d_hist.p, h->d_loop, hw, hi, 0);
  } catch (...) {
    cudaStreamEndCapture(s, &ibody);
    cudaGraphDestroy(g);
    throw;
  }
  CUDA_CHECK(cudaStreamEndCapture(s, &ibody));
  ctx->launches = before;
  h->loop_kernels_per_iter = per_iter;
  cudaGraphExec_t ge;
  CUDA_CHECK(cudaGraphInstantiate(&ge, g, 0));
  cudaGraphDestroy(g);
  h->loop_graphs.emplace(x, ge);
  return ge;
}

}  // namespace

// =========================================================================================
extern "C" {

const char* tpmg_status_string(int s) {
  switch (s) {
    case TPMG_OK: return "ok";
    case TPMG_E_CONFIG: return "config_error";
    case TPMG_E_SHAPE: return "shape_error";
    case TPMG_E_NONFINITE: return "nonfinite_error";
    case TPMG_E_FINGERPRINT: return "fingerprint_error";
    case TPMG_E_SINGULAR: return "singular_error";
    case TPMG_E_CAP: return "cap_error";
    case TPMG_E_CUDA: return "cuda_error";
    case TPMG_E_NCCL: return "nccl_error";
    case TPMG_NOT_CONVERGED: return "not_converged";
    case TPMG_BREAKDOWN: return "breakdown";
    case TPMG_DIVERGED: return "diverged";
    default: return "unknown";
  }
}

int tpmg_abi_version(void) { return TPMG_ABI_VERSION; }

int tpmg_nccl_unique_id(void* out128) {
  return guard(nullptr, [&] {
    g_nccl.load();
    ncclUniqueId id;
    NCCL_CHECK(g_nccl.GetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int tpmg_init(const tpmg_context_params* prm, tpmg_context* out) {
  return guard(nullptr, [&] {
    if (!prm || !out) throw Error(TPMG_E_CONFIG, "null argument");
    if (prm->world_size < 1 || prm->rank < 0 || prm->rank >= prm->world_size)
      throw Error(TPMG_E_CONFIG, "bad rank / world_size");
    if (prm->px * prm->py != prm->world_size)
      throw Error(TPMG_E_CONFIG, "process grid px*py must equal world_size");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(TPMG_E_CUDA, "no CUDA device: the TPMG hot path has no CPU fallback");
    auto ctx = std::make_unique<tpmg_context_s>();
    if (prm->device >= 0) CUDA_CHECK(cudaSetDevice(prm->device));
    CUDA_CHECK(cudaGetDevice(&ctx->device));
    ctx->rank = prm->rank;
    ctx->world = prm->world_size;
    ctx->px = prm->px;
    ctx->py = prm->py;
    ctx->rx = prm->rank % prm->px;
    ctx->ry = prm->rank / prm->px;
    CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    tpmg::init_device_constants(ctx->stream);
    {
      const char* e = getenv("TPMG_LOOPBACK");
      ctx->nccl_self = ctx->world == 1 && e && atoi(e) == 2;
    }
    if (ctx->world > 1 || ctx->nccl_self) {
      if (!prm->nccl_id && !ctx->nccl_self)
        throw Error(TPMG_E_CONFIG, "world_size > 1 needs an ncclUniqueId");
      g_nccl.load();
      ncclUniqueId id;
      if (prm->nccl_id) std::memcpy(&id, prm->nccl_id, sizeof(id));
      else NCCL_CHECK(g_nccl.GetUniqueId(&id));
      NCCL_CHECK(g_nccl.CommInitRank(&ctx->comm, ctx->world, id, ctx->rank));
      // the side-stream communicator is an optimisation: without it (an NCCL that cannot split)
      // the early-posted halos fall back to the main stream
      if (g_nccl.CommSplit &&
          g_nccl.CommSplit(ctx->comm, 0, ctx->rank, &ctx->comm2, nullptr) != ncclSuccess)
        ctx->comm2 = nullptr;
    }
    CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    *out = ctx.release();
  });
}

int tpmg_init_ipc(const tpmg_context_params* prm, const char* session, tpmg_context* out) {
  return guard(nullptr, [&] {
    if (!prm || !out || !session || !*session) throw Error(TPMG_E_CONFIG, "null argument");
    if (prm->world_size < 2 || prm->world_size > kIpcMaxRanks || prm->rank < 0 ||
        prm->rank >= prm->world_size)
      throw Error(TPMG_E_CONFIG, "ipc transport: bad rank / world_size (2..64 ranks)");
    if (prm->px * prm->py != prm->world_size)
      throw Error(TPMG_E_CONFIG, "process grid px*py must equal world_size");
    for (const char* c = session; *c; ++c)
      if (*c == '/') throw Error(TPMG_E_CONFIG, "ipc transport: session name must not contain '/'");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(TPMG_E_CUDA, "no CUDA device: the TPMG hot path has no CPU fallback");
    auto ctx = std::make_unique<tpmg_context_s>();
    if (prm->device >= 0) CUDA_CHECK(cudaSetDevice(prm->device));
    CUDA_CHECK(cudaGetDevice(&ctx->device));
    ctx->rank = prm->rank;
    ctx->world = prm->world_size;
    ctx->px = prm->px;
    ctx->py = prm->py;
    ctx->rx = prm->rank % prm->px;
    ctx->ry = prm->rank / prm->px;
    CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    tpmg::init_device_constants(ctx->stream);
    CUDA_CHECK(cudaMallocHost(&ctx->ipc_host, 2 * sizeof(double)));
    const std::string name = std::string("/tpmg_") + session;
    const size_t bytes = sizeof(IpcShm);
    int fd = -1;
    if (ctx->rank == 0) {
      shm_unlink(name.c_str());
      fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0 || ftruncate(fd, (off_t)bytes) != 0)
        throw Error(TPMG_E_NCCL, "ipc transport: cannot create " + name);
    } else {
      const auto t0 = std::chrono::steady_clock::now();
      while ((fd = shm_open(name.c_str(), O_RDWR, 0600)) < 0) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
          throw Error(TPMG_E_NCCL, "ipc transport: rank 0 never created " + name);
        usleep(1000);
      }
      struct stat st {};
      while (fstat(fd, &st) == 0 && (size_t)st.st_size < bytes) usleep(1000);
    }
    void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) throw Error(TPMG_E_NCCL, "ipc transport: mmap failed");
    ctx->ipc = static_cast<IpcShm*>(m);
    if (ctx->rank == 0) {
      ctx->ipc->count.store(0);
      ctx->ipc->gen.store(0);
      ctx->ipc->abort.store(0);
      ctx->ipc->world = ctx->world;
      ctx->ipc->magic.store(kIpcMagic, std::memory_order_release);
    } else {
      const auto t0 = std::chrono::steady_clock::now();
      while (ctx->ipc->magic.load(std::memory_order_acquire) != kIpcMagic) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
          throw Error(TPMG_E_NCCL, "ipc transport: segment never initialised");
        usleep(1000);
      }
      if (ctx->ipc->world != ctx->world) throw Error(TPMG_E_CONFIG, "ipc transport: world mismatch");
    }
    ipc_barrier(ctx.get());                       // every rank has mapped the segment
    if (ctx->rank == 0) shm_unlink(name.c_str());  // nothing left behind in /dev/shm
    *out = ctx.release();
  });
}

int tpmg_finalize(tpmg_context ctx) {
  if (!ctx) return TPMG_OK;
  if (ctx->ipc) munmap(ctx->ipc, sizeof(IpcShm));
  if (ctx->ipc_host) cudaFreeHost(ctx->ipc_host);
  if (ctx->comm2) g_nccl.CommDestroy(ctx->comm2);
  if (ctx->comm) g_nccl.CommDestroy(ctx->comm);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return TPMG_OK;
}

const char* tpmg_last_error(tpmg_context ctx) {
  return ctx ? ctx->last_error.c_str() : g_global_error.c_str();
}

int tpmg_context_stream(tpmg_context ctx, void** stream) {
  if (!ctx || !stream) return TPMG_E_CONFIG;
  *stream = (void*)ctx->stream;
  return TPMG_OK;
}

int tpmg_plan_decomposition(int64_t nx, int64_t ny, int px, int py, int rank, int depth,
                            int max_levels, int* n_levels, int64_t* tile_nx, int64_t* tile_ny,
                            int64_t* x0, int64_t* y0, int* nbr) {
  return guard(nullptr, [&] {
    if (rank < 0 || rank >= px * py) throw Error(TPMG_E_CONFIG, "rank outside the process grid");
    const int levels = plan_levels(nx, ny, px, py, depth, false);
    *n_levels = levels;
    const int rx = rank % px, ry = rank / px;
    for (int l = 0; l < levels && l < max_levels; ++l) {
      const int64_t gx = nx >> (levels - 1 - l), gy = ny >> (levels - 1 - l);
      tile_nx[l] = gx / px;
      tile_ny[l] = gy / py;
      x0[l] = rx * tile_nx[l];
      y0[l] = ry * tile_ny[l];
    }
    auto rk = [&](int x, int y) { return ((y % py + py) % py) * px + ((x % px + px) % px); };
    nbr[0] = rk(rx - 1, ry);
    nbr[1] = rk(rx + 1, ry);
    nbr[2] = rk(rx, ry - 1);
    nbr[3] = rk(rx, ry + 1);
  });
}

namespace {
// IPC transport: publish this rank's receive buffers, map the neighbours' (every rank builds
// the same level structure, so the neighbour's buffers have this rank's shapes), and point
// each face at the segment it must land in (W face -> west's E segment, and so on).
void ipc_connect(tpmg_hierarchy h) {
  tpmg_context ctx = h->ctx;
  IpcShm* S = ctx->ipc;
  const int nl = (int)h->lv.size();
  if (nl > kIpcMaxLevels) throw Error(TPMG_E_CONFIG, "ipc transport: too many levels");
  for (int l = 0; l < nl; ++l)
    for (int set = 0; set < 3; ++set) {
      const double* b = set == 2 ? h->lv[l].recv3.p : (set ? h->lv[l].recv2.p : h->lv[l].recv.p);
      if (b) CUDA_CHECK(cudaIpcGetMemHandle(&S->handles[ctx->rank][l][set], (void*)b));
    }
  if (h->agg_la > 0)
    CUDA_CHECK(cudaIpcGetMemHandle(&S->agg[ctx->rank], (void*)h->lv[h->agg_la - 1].f.p));
  ipc_barrier(ctx);
  std::unordered_map<int64_t, double*> opened;
  auto base = [&](int r, int l, int set) {
    const int64_t key = ((int64_t)r * kIpcMaxLevels + l) * 3 + set;
    auto it = opened.find(key);
    if (it != opened.end()) return it->second;
    void* p = nullptr;
    CUDA_CHECK(cudaIpcOpenMemHandle(&p, S->handles[r][l][set], cudaIpcMemLazyEnablePeerAccess));
    h->ipc_mapped.push_back(p);
    return opened[key] = static_cast<double*>(p);
  };
  const int west = ctx->rank_of(ctx->rx - 1, ctx->ry), east = ctx->rank_of(ctx->rx + 1, ctx->ry);
  const int south = ctx->rank_of(ctx->rx, ctx->ry - 1), north = ctx->rank_of(ctx->rx, ctx->ry + 1);
  for (int l = 0; l < nl; ++l) {
    Level& L = h->lv[l];
    const int64_t nwe = (int64_t)L.ny * h->nz, nsn = (int64_t)L.nx * h->nz;
    for (int set = 0; set < 2; ++set) {
      if (!(set ? L.recv2.p : L.recv.p)) continue;
      if (ctx->px > 1) {
        L.peer[set][0] = base(west, l, set) + nwe;  // -> west's E segment
        L.peer[set][1] = base(east, l, set);        // -> east's W segment
      }
      if (ctx->py > 1) {
        L.peer[set][2] = base(south, l, set) + 2 * nwe + nsn;  // -> south's N segment
        L.peer[set][3] = base(north, l, set) + 2 * nwe;        // -> north's S segment
      }
    }
    if (L.rep) continue;
    if (L.recv3.p) {  // deep piece d -> slot kOpp[d] of the neighbour in direction d
      int64_t off[8], cnt[8];
      deep_offsets(L, h->nz, off, cnt);
      for (int d = 0; d < 8; ++d)
        if (deep_live(h, d))
          L.peer3[d] = base(ctx->rank_of(ctx->rx + kDeepDx[d], ctx->ry + kDeepDy[d]), l, 2) +
                       off[kOpp[d]];
    }
  }
  if (h->agg_la > 0) {  // every rank's copy of the finest replicated level's f (own included)
    h->agg_peers.n = ctx->world;
    for (int r = 0; r < ctx->world; ++r) {
      if (r == ctx->rank) {
        h->agg_peers.p[r] = h->lv[h->agg_la - 1].f.p;
        continue;
      }
      void* p = nullptr;
      CUDA_CHECK(cudaIpcOpenMemHandle(&p, S->agg[r], cudaIpcMemLazyEnablePeerAccess));
      h->ipc_mapped.push_back(p);
      h->agg_peers.p[r] = static_cast<double*>(p);
    }
  }
  ipc_barrier(ctx);
}

// build_hierarchy_coefficients (multigrid.hpp:242-272) for the three profile kinds of the
// reference's ProfileVariant (multigrid.hpp:102-103): factorised `p`; partial = `p` with
// alpha_r dense (`ar`, MixedProfileSet); full `fp` (ProfileSet).  Dense profiles are restricted
// level by level exactly like the factorised horizontal scalars (restrict_profiles,
// multigrid.hpp:146-201) and assembled per level (assemble_hatted, discretization.hpp:104-141,

// 187-204) into [k][y][x] device arrays.
int hier_create_impl(tpmg_context ctx, const tpmg_grid_desc* g, const tpmg_factorized_profiles* p,
                     const tpmg_full_profiles* fp, const double* ar, double omega,
                     const tpmg_mg_config* cfg, tpmg_hierarchy* out) {
  return guard(ctx, [&] {
    if (!ctx || !g || !(p || fp) || !cfg || !out) throw Error(TPMG_E_CONFIG, "null argument");
    const int cm = fp ? tpmg::CM_FULL : (ar ? tpmg::CM_PARTIAL : tpmg::CM_FACT);
    CUDA_CHECK(cudaSetDevice(ctx->device));
    const int64_t NX = g->nx, NY = g->ny, nz = g->nz;
    if (NX < 1 || NY < 1 || nz < 1) throw Error(TPMG_E_CONFIG, "grid dimensions must be positive");
    if (NX > (1 << 30) || NY > (1 << 30) || nz > (1 << 20))
      throw Error(TPMG_E_CONFIG, "grid dimensions too large");
    if (!(g->hx > 0.0) || !(g->hy > 0.0)) throw Error(TPMG_E_CONFIG, "cell widths must be positive");
    if (cfg->smoother != TPMG_SMOOTHER_BLOCK_JACOBI)
      throw Error(TPMG_E_CONFIG, "only the block_jacobi line smoother is data parallel");
    if (!(cfg->relax > 0.0 && cfg->relax < 2.0))
      throw Error(TPMG_E_CONFIG, "smoother relaxation factor must lie in (0, 2)");
    if (cfg->nu_pre < 0 || cfg->nu_post < 0) throw Error(TPMG_E_CONFIG, "negative sweep count");
    if (NX % ctx->px || NY % ctx->py)
      throw Error(TPMG_E_CONFIG, "global grid does not split evenly over the process grid");
    check_finite(g->z_faces, nz + 1, "z_faces");
    for (int64_t k = 0; k < nz; ++k)
      if (!(g->z_faces[k + 1] > g->z_faces[k]))
        throw Error(TPMG_E_CONFIG, "vertical faces must increase");
    const int64_t ncf = NX * NY;
    if (p) {
      check_finite(p->beta_r, nz, "beta_r");
      check_finite(p->alpha_s_r, nz, "alpha_s_r");
      check_finite(p->alpha_r_r, nz + 1, "alpha_r_r");
      if (p->xi_r_r) check_finite(p->xi_r_r, nz + 1, "xi_r_r");
      check_finite(p->beta_s, ncf, "beta_s");
      check_finite(p->alpha_r_s, ncf, "alpha_r_s");
      if (p->xi_r_s) check_finite(p->xi_r_s, ncf, "xi_r_s");
      check_finite(p->alpha_s_s, 2 * ncf, "alpha_s_s");
    }
    if (ar) check_finite(ar, (nz + 1) * ncf, "alpha_r (full)");
    if (fp) {
      if (!fp->beta || !fp->alpha_s || !fp->alpha_r)
        throw Error(TPMG_E_CONFIG, "full profiles: beta, alpha_s and alpha_r are required");
      check_finite(fp->beta, nz * ncf, "beta");
      check_finite(fp->alpha_s, nz * 2 * ncf, "alpha_s");
      check_finite(fp->alpha_r, (nz + 1) * ncf, "alpha_r");
      if (fp->xi_r) check_finite(fp->xi_r, (nz + 1) * ncf, "xi_r");
    }

    if (cfg->agglomerate < 0) throw Error(TPMG_E_CONFIG, "negative agglomeration threshold");
    const bool linear_tr = cfg->prolongation == TPMG_PROLONG_LINEAR ||
                           cfg->restriction == TPMG_RESTRICT_TRANSPOSE;
    auto h = std::make_unique<tpmg_hierarchy_s>();
    h->ctx = ctx;
    {
      const char* e = getenv("TPMG_LOOPBACK");
      h->loopback = ctx->world == 1 && e && atoi(e) != 0;
    }
    const bool agg = h->multi() && cfg->agglomerate > 0;
    if (agg && ctx->world > kIpcMaxRanks && ctx->ipc)
      throw Error(TPMG_E_CONFIG, "agglomeration: too many ranks for the IPC transport");
    const int levels =
        agg ? plan_agg(NX, NY, ctx->px, ctx->py, cfg->depth, linear_tr, cfg->agglomerate, &h->agg_la)
            : plan_levels(NX, NY, ctx->px, ctx->py, cfg->depth, linear_tr);
    h->nz = (int)nz;
    h->xi = fp ? fp->xi_r != nullptr : (p->xi_r_r != nullptr && p->xi_r_s != nullptr);
    h->cm = cm;
    h->relax = cfg->relax;
    h->prolongation = cfg->prolongation;
    h->restriction = cfg->restriction;
    h->lv.resize(levels);
    h->nu_pre.assign(levels, cfg->nu_pre);
    h->nu_post.assign(levels, cfg->nu_post);
    h->nu_pre[0] = 1;  // multigrid.hpp:269-270
    h->nu_post[0] = 0;

    // vertical hatted vectors (discretization.hpp:165-181, flat: volumes dz_k, r_k^2 -> 1)
    const double* z = g->z_faces;
    // face factors (discretization.hpp:72-87, flat: r_k^2 -> 1), zero on the boundary faces
    std::vector<double> fdiff(nz + 1, 0.0), fadv(nz + 1, 0.0);
    for (int64_t k = 1; k < nz; ++k) {
      fdiff[k] = 2.0 / (z[k + 1] - z[k - 1]);
      fadv[k] = (z[k + 1] - z[k]) / (z[k + 1] - z[k - 1]);
    }
    h->bv.assign(nz, 0.0); h->sv.assign(nz, 0.0); h->av.assign(nz + 1, 0.0); h->xv.assign(nz + 1, 0.0);
    if (p) {
      for (int64_t k = 0; k < nz; ++k) {
        h->bv[k] = (z[k + 1] - z[k]) * p->beta_r[k];
        h->sv[k] = (z[k + 1] - z[k]) * p->alpha_s_r[k];
      }
      for (int64_t k = 0; k <= nz; ++k) {
        const double fd = (k >= 1 && k < nz) ? 2.0 / (z[k + 1] - z[k - 1]) : 0.0;
        const double fa = (k >= 1 && k < nz) ? (z[k + 1] - z[k]) / (z[k + 1] - z[k - 1]) : 0.0;
        h->av[k] = fd * p->alpha_r_r[k];
        if (h->xi) h->xv[k] = fa * p->xi_r_r[k];
      }
    }
    const double w2 = omega * omega;

    // horizontal profiles on the current (global) level, restricted level by level
    std::vector<double> pb(ncf, 0.0), pa(ncf, 0.0), px(ncf, 0.0), ps(2 * ncf, 0.0);
    if (p) {
      pb.assign(p->beta_s, p->beta_s + ncf);
      pa.assign(p->alpha_r_s, p->alpha_r_s + ncf);
      ps.assign(p->alpha_s_s, p->alpha_s_s + 2 * ncf);
      if (h->xi) px.assign(p->xi_r_s, p->xi_r_s + ncf);
    }
    // dense profiles, [k][global cell] (input: the reference's column-major, k fastest)
    std::vector<double> Da, Db, Dx, Ds;
    auto to_kc = [&](const double* in, int64_t rows, int64_t cols, std::vector<double>& outv) {
      outv.resize(rows * cols);
      for (int64_t c = 0; c < cols; ++c)
        for (int64_t k = 0; k < rows; ++k) outv[k * cols + c] = in[c * rows + k];
    };
    if (ar) to_kc(ar, nz + 1, ncf, Da);
    if (fp) {
      to_kc(fp->alpha_r, nz + 1, ncf, Da);
      to_kc(fp->beta, nz, ncf, Db);
      to_kc(fp->alpha_s, nz, 2 * ncf, Ds);
      if (fp->xi_r) to_kc(fp->xi_r, nz + 1, ncf, Dx);
    }
    int64_t gx = NX, gy = NY;
    double hx = g->hx, hy = g->hy;
    for (int l = levels - 1; l >= 0; --l) {
      Level& L = h->lv[l];
      L.rep = l < h->agg_la;  // replicated: the whole global level on this rank
      const int lpx = L.rep ? 1 : ctx->px, lpy = L.rep ? 1 : ctx->py;
      L.gnx = (int)gx; L.gny = (int)gy;
      L.nx = (int)(gx / lpx); L.ny = (int)(gy / lpy);
      L.x0 = L.rep ? 0 : ctx->rx * L.nx; L.y0 = L.rep ? 0 : ctx->ry * L.ny;
      L.plane = (int64_t)L.nx * L.ny;
      const int64_t gnc = gx * gy;
      // assemble_hatted (factorised), discretization.hpp:256-274, flat Cartesian geometry
      const double area = hx * hy, ge_e = hy / hx, ge_n = hx / hy;
      L.bh.resize(L.plane); L.ah.resize(L.plane); L.xh.resize(L.plane); L.sh.resize(2 * L.plane);
      std::vector<double> sw(L.plane), se(L.plane), ss(L.plane), sn(L.plane);
      for (int j = 0; j < L.ny; ++j)
        for (int i = 0; i < L.nx; ++i) {
          const int64_t c = (int64_t)j * L.nx + i;
          const int64_t gi = L.x0 + i, gj = L.y0 + j, G = gj * gx + gi;
          L.bh[c] = area * pb[G];
          L.ah[c] = w2 * (area * pa[G]);
          L.xh[c] = w2 * (area * px[G]);
          const int64_t gw = gj * gx + (gi + gx - 1) % gx;
          const int64_t gs = ((gj + gy - 1) % gy) * gx + gi;
          L.sh[c] = w2 * ge_e * ps[G];
          L.sh[L.plane + c] = w2 * ge_n * ps[gnc + G];
          se[c] = L.sh[c];
          sn[c] = L.sh[L.plane + c];
          sw[c] = w2 * ge_e * ps[gw];
          ss[c] = w2 * ge_n * ps[gnc + gs];
        }
      {  // one edge scalar on the whole global level (every rank takes the same decision, and
         // the neighbours' ring columns of a decomposed run share it)
        const double S0 = w2 * ge_e * ps[0];
        bool uni = true;
        for (int64_t G = 0; G < gnc && uni; ++G)
          uni = (w2 * ge_e * ps[G] == S0) && (w2 * ge_n * ps[gnc + G] == S0);
        L.uni = uni;
      }
      L.d_bh.upload(L.bh.data(), L.plane);
      L.d_ah.upload(L.ah.data(), L.plane);
      L.d_xh.upload(L.xh.data(), L.plane);
      L.d_sw.upload(sw.data(), L.plane);
      L.d_se.upload(se.data(), L.plane);
      L.d_ss.upload(ss.data(), L.plane);
      L.d_sn.upload(sn.data(), L.plane);
      L.cm = cm;
      if (h->multi() && !L.rep && cm == tpmg::CM_FACT && l > 0) {
        // the same scalars on the 1-cell ring around the tile (tpmg::kRingFields layout), for the
        // ring residuals of the decomposed fused residual + transpose restriction
        const int64_t rn = 2 * (int64_t)L.ny + 2 * (int64_t)L.nx;
        std::vector<double> rc(tpmg::kRingFields * rn);
        auto put = [&](int64_t ri, int64_t gi, int64_t gj) {
          gi = (gi % gx + gx) % gx;
          gj = (gj % gy + gy) % gy;
          const int64_t G = gj * gx + gi;
          const int64_t gw = gj * gx + (gi + gx - 1) % gx;
          const int64_t gs = ((gj + gy - 1) % gy) * gx + gi;
          rc[ri] = area * pb[G];
          rc[rn + ri] = w2 * (area * pa[G]);
          rc[2 * rn + ri] = w2 * (area * px[G]);
          rc[3 * rn + ri] = w2 * ge_e * ps[gw];
          rc[4 * rn + ri] = w2 * ge_e * ps[G];
          rc[5 * rn + ri] = w2 * ge_n * ps[gnc + gs];
          rc[6 * rn + ri] = w2 * ge_n * ps[gnc + G];
        };
        for (int j = 0; j < L.ny; ++j) {
          put(j, L.x0 - 1, L.y0 + j);
          put(L.ny + j, L.x0 + L.nx, L.y0 + j);
        }
        for (int i = 0; i < L.nx; ++i) {
          put(2 * L.ny + i, L.x0 + i, L.y0 - 1);
          put(2 * L.ny + L.nx + i, L.x0 + i, L.y0 + L.ny);
        }
        L.d_ringc.upload(rc.data(), rc.size());
      }
      if (cm != tpmg::CM_FACT) {
        // assemble_hatted, dense components (discretization.hpp:122-140, 196-203):
        // alpha_r hat = ((w2 |T|) f_k) alpha_r; beta hat = |T| (dz_k beta);
        // alpha_s hat = ((w2 dz_k) g_e) alpha_s; xi_r hat = ((w2 |T|) fadv_k) xi_r
        const int64_t P = L.plane;
        std::vector<double> v((nz + 1) * P);
        auto tile = [&](int64_t rows, auto&& val, DevBuf& dst) {
          for (int64_t k = 0; k < rows; ++k)
            for (int j = 0; j < L.ny; ++j)
              for (int i = 0; i < L.nx; ++i) {
                const int64_t gi = L.x0 + i, gj = L.y0 + j;
                v[k * P + (int64_t)j * L.nx + i] = val(k, gi, gj);
              }
          dst.upload(v.data(), rows * P);
        };
        tile(nz + 1, [&](int64_t k, int64_t gi, int64_t gj) {
          return ((w2 * area) * fdiff[k]) * Da[k * gnc + gj * gx + gi];
        }, L.d_ard);
        if (cm == tpmg::CM_FULL) {
          tile(nz, [&](int64_t k, int64_t gi, int64_t gj) {
            return area * ((z[k + 1] - z[k]) * Db[k * gnc + gj * gx + gi]);
          }, L.d_bd);
          if (h->xi)
            tile(nz + 1, [&](int64_t k, int64_t gi, int64_t gj) {
              return ((w2 * area) * fadv[k]) * Dx[k * gnc + gj * gx + gi];
            }, L.d_xid);
          auto edge = [&](int64_t k, int64_t e, double ge) {
            return ((w2 * (z[k + 1] - z[k])) * ge) * Ds[k * 2 * gnc + e];
          };
          tile(nz, [&](int64_t k, int64_t gi, int64_t gj) {
            return edge(k, gj * gx + (gi + gx - 1) % gx, ge_e);  // east edge of the W cell
          }, L.d_swd);
          tile(nz, [&](int64_t k, int64_t gi, int64_t gj) { return edge(k, gj * gx + gi, ge_e); },
               L.d_sed);
          tile(nz, [&](int64_t k, int64_t gi, int64_t gj) {
            return edge(k, gnc + ((gj + gy - 1) % gy) * gx + gi, ge_n);  // north of the S cell
          }, L.d_ssd);
          tile(nz, [&](int64_t k, int64_t gi, int64_t gj) {
            return edge(k, gnc + gj * gx + gi, ge_n);
          }, L.d_snd);
        }
      }
      if (l == 0) break;
      if (cm != tpmg::CM_FACT) {
        // restrict_profiles, dense rows (multigrid.hpp:107-151, 146-156, 193-201)
        const int64_t cx = gx / 2, cy = gy / 2, cnc = cx * cy;
        const double wf = hx * hy;
        auto cell_rows = [&](std::vector<double>& D, int64_t rows) {
          std::vector<double> q(rows * cnc);
          for (int64_t k = 0; k < rows; ++k)
            for (int64_t J = 0; J < cy; ++J)
              for (int64_t I = 0; I < cx; ++I) {
                const int64_t c0 = (2 * J) * gx + 2 * I, c1 = c0 + 1, c2 = c0 + gx, c3 = c2 + 1;
                const double* d = D.data() + k * gnc;
                double acc = 0.0, ws = 0.0;
                acc += wf * d[c0]; ws += wf;
                acc += wf * d[c1]; ws += wf;
                acc += wf * d[c2]; ws += wf;
                acc += wf * d[c3]; ws += wf;
                q[k * cnc + J * cx + I] = acc / ws;
              }
          D.swap(q);
        };
        cell_rows(Da, nz + 1);
        if (cm == tpmg::CM_FULL) {
          cell_rows(Db, nz);
          if (h->xi) cell_rows(Dx, nz + 1);
          std::vector<double> q(nz * 2 * cnc);
          for (int64_t k = 0; k < nz; ++k)
            for (int64_t J = 0; J < cy; ++J)
              for (int64_t I = 0; I < cx; ++I) {
                const double* d = Ds.data() + k * 2 * gnc;
                const int64_t c0 = (2 * J) * gx + 2 * I, c1 = c0 + 1, c2 = c0 + gx, c3 = c2 + 1;
                q[k * 2 * cnc + J * cx + I] = (d[c1] + d[c3]) / 2.0;
                q[k * 2 * cnc + cnc + J * cx + I] = (d[gnc + c2] + d[gnc + c3]) / 2.0;
              }
          Ds.swap(q);
        }
      }
      // restrict_profiles (factorised), multigrid.hpp:158-201: area-weighted mean of the 4
      // children (:108-124), mean of the 2 co-linear child edges (:135-143)
      const int64_t cx = gx / 2, cy = gy / 2, cnc = cx * cy;
      std::vector<double> qb(cnc), qa(cnc), qx(cnc), qs(2 * cnc);
      const double wf = hx * hy;
      for (int64_t J = 0; J < cy; ++J)
        for (int64_t I = 0; I < cx; ++I) {
          const int64_t T = J * cx + I;
          const int64_t c0 = (2 * J) * gx + 2 * I, c1 = c0 + 1, c2 = c0 + gx, c3 = c2 + 1;
          auto mean4 = [&](const std::vector<double>& v) {
            double acc = 0.0, ws = 0.0;
            acc += wf * v[c0]; ws += wf;
            acc += wf * v[c1]; ws += wf;
            acc += wf * v[c2]; ws += wf;
            acc += wf * v[c3]; ws += wf;
            return acc / ws;
          };
          qb[T] = mean4(pb);
          qa[T] = mean4(pa);
          qx[T] = mean4(px);
          qs[T] = (ps[c1] + ps[c3]) / 2.0;
          qs[cnc + T] = (ps[gnc + c2] + ps[gnc + c3]) / 2.0;
        }
      pb.swap(qb); pa.swap(qa); px.swap(qx); ps.swap(qs);
      gx = cx; gy = cy;
      hx *= 2.0; hy *= 2.0;
    }
    h->d_bv.upload(h->bv.data(), nz);
    h->d_sv.upload(h->sv.data(), nz);
    h->d_av.upload(h->av.data(), nz + 1);
    h->d_xv.upload(h->xv.data(), nz + 1);
    h->upload_vertical_rows();

    // work buffers
    int64_t max_blocks = 1024;
    for (int l = 0; l < levels; ++l) {
      Level& L = h->lv[l];
      const int64_t n = L.plane * nz;
      if (l < levels - 1) {
        L.t.alloc(n);
        L.u.alloc(n);
        L.f.alloc(n);
      }
      if (h->multi() && !L.rep) {
        const int64_t faces = 2 * (int64_t)L.ny * nz + 2 * (int64_t)L.nx * nz;
        L.send.alloc(faces);
        L.recv.alloc(faces);
        // two-cell halo of the decomposed fused residual + transpose restriction
        if (L.d_ringc.p && tpmg::resid_restrict_T2_fusable(L.coef(nz))) {
          L.send3.alloc(deep_size(L, nz));
          L.recv3.alloc(deep_size(L, nz));
          if (l < levels - 1 && !ctx->ipc) {  // coarse levels: f's halo posted early
            L.sendF.alloc(faces);
            L.recvF.alloc(faces);
          }
        } else {
          L.d_ringc.reset();
        }
      }
      // one partial per 256-column block (k_apply) or per 32x4 tile (k_apply_tiled)
      max_blocks = std::max<int64_t>(max_blocks, (L.plane + 255) / 256 + 1);
      max_blocks = std::max<int64_t>(max_blocks, L.plane / 128 + 1);
    }
    if (h->agg_la > 0) {  // this rank's block of the finest replicated level (+ all ranks')
      const Level& A = h->lv[h->agg_la];
      const int64_t bn = (int64_t)(A.nx / 2) * (A.ny / 2) * nz;
      h->agg_tile.alloc(bn);
      if (h->nccl_reduce()) h->agg_gather.alloc((size_t)ctx->world * bn);
    }
    const int64_t nf = h->lv[levels - 1].plane * nz;
    h->r.alloc(nf); h->z.alloc(nf); h->p.alloc(nf); h->q.alloc(nf); h->tmp.alloc(nf);
    h->partials.alloc(std::max<int64_t>(max_blocks, 148 * 8));
    if (ctx->world > 1 || h->nccl_self())  // tile partials of the finest level, every rank's
      h->gathered.alloc((size_t)ctx->world * (h->lv[levels - 1].plane / 128 + 1));
    h->scal.alloc(8);
    CUDA_CHECK(cudaMemsetAsync(h->scal.p, 0, 8 * sizeof(double), h->ctx->stream));
    CUDA_CHECK(cudaMalloc(&h->d_err, sizeof(int)));
    CUDA_CHECK(cudaMemsetAsync(h->d_err, 0, sizeof(int), h->ctx->stream));
    CUDA_CHECK(cudaMallocHost(&h->h_scal, 8 * sizeof(double)));
    // Coarse levels (the warp-per-column regime, L2 resident): the column blocks' Thomas
    // factorisation is formed once here, so their sweeps only carry the right-hand side through
    // the recurrence (TPMG_PIV=0 disables); a level with a zero pivot keeps the on-the-fly
    // smoother (which raises the reference's singular_error when it is used)
    {
      const char* e = getenv("TPMG_PIV");
      const bool use = !(e && atoi(e) == 0);
      for (int l = 0; l < levels && use; ++l) {
        Level& L = h->lv[l];
        if (l == levels - 1 || !tpmg::jacobi_wants_factors(L.coef(nz))) continue;
        L.d_piv.alloc(L.plane * nz);
        L.d_cpt.alloc(L.plane * nz);
        CUDA_CHECK(cudaMemsetAsync(h->d_err, 0, sizeof(int), ctx->stream));
        LevelCoef c = L.coef(nz);
        c.piv = c.cpt = nullptr;
        tpmg::launch_factor_columns(ctx->launch(), h->vcoef(), c, h->xi, L.d_piv.p, L.d_cpt.p,
                                    h->d_err);
        int zero = 0;
        CUDA_CHECK(cudaMemcpyAsync(&zero, h->d_err, sizeof(int), cudaMemcpyDeviceToHost,
                                   ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (zero) {
          L.d_piv.reset();
          L.d_cpt.reset();
        }
      }
      CUDA_CHECK(cudaMemsetAsync(h->d_err, 0, sizeof(int), h->ctx->stream));
    }
    {
      const int L = levels - 1;
      const char* e = getenv("TPMG_PCG_FUSED");
      const bool allow = !(e && atoi(e) == 0);
      h->pcg_fused = allow && L > 0 && h->nu_pre[L] >= 1 && h->nu_post[L] >= 1 &&
                     tpmg::jacobi_fusable(h->lv[L].coef(h->nz));
      // fused residual + transpose restriction (TMA): 0.78 vs 0.83 ms split at config 3;
      // TPMG_FUSE_RR=0 selects the split apply + restrict pair (same bits)
      const char* e2 = getenv("TPMG_FUSE_RR");
      h->fuse_rr = !(e2 && atoi(e2) == 0);
      // fused direction update + A p (halos of z and p_old exchanged first; one rank: the
      // periodic self views); TPMG_FUSE_AP=0 selects k_pcg_px + the apply kernel
      const char* e3 = getenv("TPMG_FUSE_AP");
      h->fused_ap = h->pcg_fused && !(e3 && atoi(e3) == 0) &&
                    tpmg::pcg_ap_fusable(h->lv[L].coef(h->nz));
      if (h->fused_ap) h->p2.alloc(nf);
      if (h->fused_ap && h->multi()) {  // second halo set: z and p_old are exchanged together
        Level& F = h->lv[L];
        const int64_t faces = 2 * (int64_t)F.ny * nz + 2 * (int64_t)F.nx * nz;
        F.send2.alloc(faces);
        F.recv2.alloc(faces);
      }
      const char* e4 = getenv("TPMG_Q_IN_SWEEP");
      h->q_in_sweep = h->fused_ap && !(e4 && atoi(e4) == 0);
    }
    if (ctx->ipc) ipc_connect(h.get());
    *out = h.release();
  });
}
}  // namespace

int tpmg_hier_create(tpmg_context ctx, const tpmg_grid_desc* g,
                     const tpmg_factorized_profiles* p, double omega, const tpmg_mg_config* cfg,
                     tpmg_hierarchy* out) {
  if (!p) return hier_create_impl(ctx, nullptr, nullptr, nullptr, nullptr, omega, cfg, out);
  return hier_create_impl(ctx, g, p, nullptr, nullptr, omega, cfg, out);
}

int tpmg_hier_create_partial(tpmg_context ctx, const tpmg_grid_desc* g,
                             const tpmg_factorized_profiles* p, const double* alpha_r,
                             double omega, const tpmg_mg_config* cfg, tpmg_hierarchy* out) {
  if (!p || !alpha_r) return hier_create_impl(ctx, nullptr, nullptr, nullptr, nullptr, omega, cfg, out);
  return hier_create_impl(ctx, g, p, nullptr, alpha_r, omega, cfg, out);
}

int tpmg_hier_create_full(tpmg_context ctx, const tpmg_grid_desc* g, const tpmg_full_profiles* fp,
                          double omega, const tpmg_mg_config* cfg, tpmg_hierarchy* out) {
  if (!fp) return hier_create_impl(ctx, nullptr, nullptr, nullptr, nullptr, omega, cfg, out);
  return hier_create_impl(ctx, g, nullptr, fp, nullptr, omega, cfg, out);
}

int tpmg_hier_create_generic(tpmg_context ctx, int n_levels, int nz, int nnb, int nchild,
                             const int64_t* ncells, const int64_t* nedges,
                             const int64_t* const* nbr, const int64_t* const* cedge,
                             const int64_t* const* children, const int* prol_d1,
                             const int* prol_d2, const double* bv, const double* sv,
                             const double* av, const double* xv, const double* const* bh,
                             const double* const* ah, const double* const* xh,
                             const double* const* sh, double relax, int prolongation,
                             int restriction, int nu_pre, int nu_post, tpmg_hierarchy* out) {
  return guard(ctx, [&] {
    if (!ctx || !ncells || !nedges || !nbr || !cedge || !bv || !sv || !av || !xv || !bh || !ah ||
        !xh || !sh || !out)
      throw Error(TPMG_E_CONFIG, "null argument");
    if (ctx->world != 1) throw Error(TPMG_E_CONFIG, "indirect hierarchies run on one rank");
    if (n_levels < 1 || nz < 1 || nnb < 1 || nnb > 8 || nchild < 1 || nchild > 8)
      throw Error(TPMG_E_CONFIG, "bad table sizes (1 <= nnb, nchild <= 8)");
    if (!(relax > 0.0 && relax < 2.0))
      throw Error(TPMG_E_CONFIG, "smoother relaxation factor must lie in (0, 2)");
    if (n_levels > 1 && (!children || !prol_d1 || !prol_d2))
      throw Error(TPMG_E_CONFIG, "child tables and the prolongation rule are required");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    auto h = std::make_unique<tpmg_hierarchy_s>();
    h->ctx = ctx;
    h->nz = nz;
    h->xi = true;  // the reference's build_column always carries the xi terms
    h->generic = true;
    h->relax = relax;
    h->prolongation = prolongation;
    h->restriction = restriction;
    h->lv.resize(n_levels);
    h->nu_pre.assign(n_levels, nu_pre);
    h->nu_post.assign(n_levels, nu_post);
    h->nu_pre[0] = 1;  // multigrid.hpp:269-270
    h->nu_post[0] = 0;
    h->rule.nchild = nchild;
    for (int j = 0; j < nchild; ++j) {
      h->rule.d1[j] = prol_d1 ? prol_d1[j] : -1;
      h->rule.d2[j] = prol_d2 ? prol_d2[j] : -1;
      // d1 = -1: centre child (= parent); otherwise two neighbour slots of the parent
      if (n_levels > 1 && (h->rule.d1[j] < -1 || h->rule.d1[j] >= nnb ||
                           (h->rule.d1[j] >= 0 && (h->rule.d2[j] < 0 || h->rule.d2[j] >= nnb))))
        throw Error(TPMG_E_CONFIG, "prolongation rule out of range");
    }
    check_finite(bv, nz, "bv"); check_finite(sv, nz, "sv");
    check_finite(av, nz + 1, "av"); check_finite(xv, nz + 1, "xv");
    h->bv.assign(bv, bv + nz); h->sv.assign(sv, sv + nz);
    h->av.assign(av, av + nz + 1); h->xv.assign(xv, xv + nz + 1);
    auto to_int = [](const int64_t* a, int64_t n, int64_t bound, const char* what) {
      std::vector<int> v(n);
      for (int64_t i = 0; i < n; ++i) {
        if (a[i] < 0 || a[i] >= bound) throw Error(TPMG_E_SHAPE, std::string(what) + ": index out of range");
        v[i] = (int)a[i];
      }
      return v;
    };
    int64_t max_blocks = 1024;
    for (int l = 0; l < n_levels; ++l) {
      Level& L = h->lv[l];
      const int64_t nc = ncells[l], ne = nedges[l];
      if (nc < 1 || nc > (1 << 30) || ne < 1) throw Error(TPMG_E_SHAPE, "bad level size");
      L.nx = (int)nc; L.ny = 1; L.gnx = (int)nc; L.gny = 1; L.plane = nc;
      L.nnb = nnb;
      check_finite(bh[l], nc, "bh"); check_finite(ah[l], nc, "ah");
      check_finite(xh[l], nc, "xh"); check_finite(sh[l], ne, "sh");
      L.d_bh.upload(bh[l], nc); L.d_ah.upload(ah[l], nc); L.d_xh.upload(xh[l], nc);
      L.d_shg.upload(sh[l], ne);
      const auto vn = to_int(nbr[l], nc * nnb, nc, "neighbour table");
      const auto ve = to_int(cedge[l], nc * nnb, ne, "edge table");
      L.d_nbr.upload(vn.data(), vn.size());
      L.d_cedge.upload(ve.data(), ve.size());
      if (l + 1 < n_levels) {
        const auto vc = to_int(children[l + 1], nc * nchild, ncells[l + 1], "child table");
        L.d_children.upload(vc.data(), vc.size());
      }
      const int64_t n = nc * nz;
      if (l < n_levels - 1) {
        L.t.alloc(n); L.u.alloc(n); L.f.alloc(n);
      }
      max_blocks = std::max<int64_t>(max_blocks, (n + 255) / 256 + 1);
    }
    h->d_bv.upload(h->bv.data(), nz);
    h->d_sv.upload(h->sv.data(), nz);
    h->d_av.upload(h->av.data(), nz + 1);
    h->d_xv.upload(h->xv.data(), nz + 1);
    h->upload_vertical_rows();
    const int64_t nf = h->lv[n_levels - 1].plane * nz;
    h->r.alloc(nf); h->z.alloc(nf); h->p.alloc(nf); h->q.alloc(nf); h->tmp.alloc(nf);
    h->partials.alloc(std::max<int64_t>(max_blocks, 148 * 8));
    h->scal.alloc(8);
    CUDA_CHECK(cudaMemsetAsync(h->scal.p, 0, 8 * sizeof(double), h->ctx->stream));
    CUDA_CHECK(cudaMalloc(&h->d_err, sizeof(int)));
    CUDA_CHECK(cudaMemsetAsync(h->d_err, 0, sizeof(int), h->ctx->stream));
    CUDA_CHECK(cudaMallocHost(&h->h_scal, 8 * sizeof(double)));
    *out = h.release();
  });
}

int tpmg_hier_coef_mode(tpmg_hierarchy h, int* mode) {
  return guard(h ? h->ctx : nullptr, [&] { *mode = h->cm; });
}

int tpmg_hier_destroy(tpmg_hierarchy h) {
  if (!h) return TPMG_OK;
  cudaStreamSynchronize(h->ctx->stream);
  if (h->ctx->ipc) {  // collective: unmap the neighbours' buffers before anyone frees its own
    for (void* p : h->ipc_mapped) cudaIpcCloseMemHandle(p);
    try {
      ipc_barrier(h->ctx);
    } catch (const Error&) {
    }
  }
  delete h;
  return TPMG_OK;
}

int tpmg_hier_n_levels(tpmg_hierarchy h, int* n) {
  return guard(h ? h->ctx : nullptr, [&] { *n = (int)h->lv.size(); });
}

int tpmg_hier_level_shape(tpmg_hierarchy h, int level, int64_t* nx, int64_t* ny, int64_t* nz,
                          int64_t* x0, int64_t* y0) {
  return guard(h->ctx, [&] {
    if (level < 0 || level >= (int)h->lv.size()) throw Error(TPMG_E_SHAPE, "level out of range");
    const Level& L = h->lv[level];
    if (nx) *nx = L.nx;
    if (ny) *ny = L.ny;
    if (nz) *nz = h->nz;
    if (x0) *x0 = L.x0;
    if (y0) *y0 = L.y0;
  });
}

int tpmg_hier_get_coefficients(tpmg_hierarchy h, int level, double* bh, double* ah, double* xh,
                               double* sh, double* bv, double* sv, double* av, double* xv) {
  return guard(h->ctx, [&] {
    if (level < 0 || level >= (int)h->lv.size()) throw Error(TPMG_E_SHAPE, "level out of range");
    const Level& L = h->lv[level];
    const size_t np = L.plane * sizeof(double);
    if (bh) std::memcpy(bh, L.bh.data(), np);
    if (ah) std::memcpy(ah, L.ah.data(), np);
    if (xh) std::memcpy(xh, L.xh.data(), np);
    if (sh) std::memcpy(sh, L.sh.data(), 2 * np);
    if (bv) std::memcpy(bv, h->bv.data(), h->nz * sizeof(double));
    if (sv) std::memcpy(sv, h->sv.data(), h->nz * sizeof(double));
    if (av) std::memcpy(av, h->av.data(), (h->nz + 1) * sizeof(double));
    if (xv) std::memcpy(xv, h->xv.data(), (h->nz + 1) * sizeof(double));
  });
}

int tpmg_field_create(tpmg_hierarchy h, int level, tpmg_field* out) {
  return guard(h ? h->ctx : nullptr, [&] {
    if (level < 0 || level >= (int)h->lv.size()) throw Error(TPMG_E_SHAPE, "level out of range");
    auto f = std::make_unique<tpmg_field_s>();
    f->h = h;
    f->level = level;
    f->buf.alloc(h->lv[level].plane * h->nz);
    CUDA_CHECK(cudaMemsetAsync(f->buf.p, 0, f->buf.n * sizeof(double), h->ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(h->ctx->stream));
    *out = f.release();
  });
}

int tpmg_field_destroy(tpmg_field f) {
  if (f) {
    cudaStreamSynchronize(f->h->ctx->stream);
    delete f;
  }
  return TPMG_OK;
}

int tpmg_field_level(tpmg_field f, int* level) {
  *level = f->level;
  return TPMG_OK;
}

int tpmg_field_upload(tpmg_field f, const double* host, int layout) {
  return guard(f->h->ctx, [&] {
    tpmg_hierarchy h = f->h;
    const int64_t n = f->buf.n;
    cudaStream_t s = h->ctx->stream;
    if (layout == TPMG_LAYOUT_X_FASTEST) {
      CUDA_CHECK(cudaMemcpyAsync(f->buf.p, host, n * 8, cudaMemcpyHostToDevice, s));
    } else if (layout == TPMG_LAYOUT_K_FASTEST) {
      CUDA_CHECK(cudaMemcpyAsync(h->tmp.p, host, n * 8, cudaMemcpyHostToDevice, s));
      tpmg::launch_kfast_to_xfast(h->ctx->launch(), h->lv[f->level].plane, h->nz, h->tmp.p,
                                  f->buf.p);
    } else {
      throw Error(TPMG_E_CONFIG, "unknown layout");
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int tpmg_field_download(tpmg_field f, double* host, int layout) {
  return guard(f->h->ctx, [&] {
    tpmg_hierarchy h = f->h;
    const int64_t n = f->buf.n;
    cudaStream_t s = h->ctx->stream;
    if (layout == TPMG_LAYOUT_X_FASTEST) {
      CUDA_CHECK(cudaMemcpyAsync(host, f->buf.p, n * 8, cudaMemcpyDeviceToHost, s));
    } else if (layout == TPMG_LAYOUT_K_FASTEST) {
      tpmg::launch_xfast_to_kfast(h->ctx->launch(), h->lv[f->level].plane, h->nz, f->buf.p,
                                  h->tmp.p);
      CUDA_CHECK(cudaMemcpyAsync(host, h->tmp.p, n * 8, cudaMemcpyDeviceToHost, s));
    } else {
      throw Error(TPMG_E_CONFIG, "unknown layout");
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int tpmg_field_fill(tpmg_field f, double v) {
  return guard(f->h->ctx, [&] {
    fill(f->h, f->buf.p, f->buf.n, v);
    sync_check(f->h);
  });
}

int tpmg_field_copy(tpmg_field dst, tpmg_field src) {
  return guard(dst->h->ctx, [&] {
    if (dst->h != src->h || dst->level != src->level)
      throw Error(TPMG_E_SHAPE, "field_copy: shapes differ");
    CUDA_CHECK(cudaMemcpyAsync(dst->buf.p, src->buf.p, dst->buf.n * 8, cudaMemcpyDeviceToDevice,
                               dst->h->ctx->stream));
    sync_check(dst->h);
  });
}

int tpmg_field_device_ptr(tpmg_field f, double** out) {
  *out = f->buf.p;
  return TPMG_OK;
}

int tpmg_apply(tpmg_hierarchy h, tpmg_field u, tpmg_field y) {
  return guard(h->ctx, [&] {
    same_hier(h, u);
    same_hier(h, y);
    if (u->level != y->level || u == y)
      throw Error(TPMG_E_SHAPE, "apply_operator: field does not match the coefficients");
    apply_level(h, u->level, tpmg::APPLY_AU, u->buf.p, nullptr, y->buf.p);
    sync_check(h);
  });
}

int tpmg_residual(tpmg_hierarchy h, tpmg_field f, tpmg_field u, tpmg_field r) {
  return guard(h->ctx, [&] {
    same_hier(h, f); same_hier(h, u); same_hier(h, r);
    if (f->level != u->level || r->level != u->level || r == u)
      throw Error(TPMG_E_SHAPE, "residual: field shapes do not match");
    apply_level(h, u->level, tpmg::APPLY_RESID, u->buf.p, f->buf.p, r->buf.p);
    sync_check(h);
  });
}

int tpmg_smooth(tpmg_hierarchy h, tpmg_field u, tpmg_field f, int sweeps) {
  return guard(h->ctx, [&] {
    same_hier(h, u); same_hier(h, f);
    if (u->level != f->level) throw Error(TPMG_E_SHAPE, "smooth: field shapes do not match");
    if (!(h->relax > 0.0 && h->relax < 2.0))
      throw Error(TPMG_E_CONFIG, "smoother relaxation factor must lie in (0, 2)");
    const int l = u->level;
    Level& L = h->lv[l];
    double* A = u->buf.p;
    double* B = (l == h->finest()) ? h->tmp.p : L.t.p;  // level scratch
    double* cur = A;
    for (int s = 0; s < sweeps; ++s) {
      double* out = (cur == A) ? B : A;
      sweep(h, l, cur, f->buf.p, out);
      cur = out;
    }
    if (cur != A)
      CUDA_CHECK(cudaMemcpyAsync(A, cur, u->buf.n * 8, cudaMemcpyDeviceToDevice, h->ctx->stream));
    sync_check(h);
  });
}

int tpmg_restrict(tpmg_hierarchy h, tpmg_field fine, tpmg_field coarse) {
  return guard(h->ctx, [&] {
    same_hier(h, fine); same_hier(h, coarse);
    if (fine->level != coarse->level + 1)
      throw Error(TPMG_E_SHAPE, "restrict_field: fine field is not one level above the target");
    restrict_plain(h, fine->level, fine->buf.p, coarse->buf.p, -1);
    sync_check(h);
  });
}

static int prolong_impl(tpmg_hierarchy h, tpmg_field coarse, tpmg_field fine, bool add) {
  return guard(h->ctx, [&] {
    same_hier(h, fine); same_hier(h, coarse);
    if (fine->level != coarse->level + 1)
      throw Error(TPMG_E_SHAPE, "prolongate_field: field level does not match");
    prolong_level(h, coarse->level, coarse->buf.p, fine->buf.p, add);
    sync_check(h);
  });
}

int tpmg_restrict_kind(tpmg_hierarchy h, tpmg_field fine, tpmg_field coarse, int restriction) {
  return guard(h->ctx, [&] {
    same_hier(h, fine); same_hier(h, coarse);
    if (fine->level != coarse->level + 1)
      throw Error(TPMG_E_SHAPE, "restrict_field: fine field is not one level above the target");
    if (restriction != TPMG_RESTRICT_SUMMATION && restriction != TPMG_RESTRICT_TRANSPOSE)
      throw Error(TPMG_E_CONFIG, "unknown restriction kind");
    restrict_plain(h, fine->level, fine->buf.p, coarse->buf.p, restriction);
    sync_check(h);
  });
}

int tpmg_prolong_kind(tpmg_hierarchy h, tpmg_field coarse, tpmg_field fine, int prolongation,
                      int add) {
  return guard(h->ctx, [&] {
    same_hier(h, fine); same_hier(h, coarse);
    if (fine->level != coarse->level + 1)
      throw Error(TPMG_E_SHAPE, "prolongate_field: field level does not match");
    if (prolongation != TPMG_PROLONG_LINEAR && prolongation != TPMG_PROLONG_INJECTION)
      throw Error(TPMG_E_CONFIG, "unknown prolongation kind");
    prolong_level(h, coarse->level, coarse->buf.p, fine->buf.p, add != 0, false, prolongation);
    sync_check(h);
  });
}

int tpmg_prolong_add(tpmg_hierarchy h, tpmg_field coarse, tpmg_field fine) {
  return prolong_impl(h, coarse, fine, true);
}

int tpmg_prolong(tpmg_hierarchy h, tpmg_field coarse, tpmg_field fine) {
  return prolong_impl(h, coarse, fine, false);
}

int tpmg_vcycle(tpmg_hierarchy h, tpmg_field f, tpmg_field u) {
  return guard(h->ctx, [&] {
    same_hier(h, f); same_hier(h, u);
    const int L = h->finest();
    if (f->level != L || u->level != L) throw Error(TPMG_E_SHAPE, "v_cycle: fields must be finest");
    vcycle(h, L, f->buf.p, u->buf.p, h->tmp.p, false);
    sync_check(h);
  });
}

int tpmg_dot(tpmg_hierarchy h, tpmg_field a, tpmg_field b, double* out) {
  return guard(h->ctx, [&] {
    same_hier(h, a); same_hier(h, b);
    if (a->level != b->level) throw Error(TPMG_E_SHAPE, "dot: shapes differ");
    dot_into(h, a->level, a->buf.p, b->buf.p, 4);
    *out = read_scalar(h, 4);
  });
}

int tpmg_norm(tpmg_hierarchy h, tpmg_field a, double* out) {
  double d = 0.0;
  const int rc = tpmg_dot(h, a, a, &d);
  if (rc == TPMG_OK) *out = std::sqrt(d);
  return rc;
}

int tpmg_measure_cycle_rate(tpmg_hierarchy h, tpmg_field f, int n_cycles, double* rate) {
  return guard(h->ctx, [&] {
    same_hier(h, f);
    const int L = h->finest();
    if (f->level != L) throw Error(TPMG_E_SHAPE, "measure_cycle_rate: f must be finest");
    if (n_cycles < 2) throw Error(TPMG_E_CONFIG, "measure_cycle_rate needs at least two cycles");
    const int64_t n = f->buf.n;
    double* u = h->z.p;
    double* r = h->r.p;
    fill(h, u, n, 0.0);
    double first = 0.0, last = 0.0;
    for (int i = 1; i <= n_cycles; ++i) {
      vcycle(h, L, f->buf.p, u, h->tmp.p, i == 1);
      apply_level(h, L, tpmg::APPLY_RESID, u, f->buf.p, r);
      dot_into(h, L, r, r, 5);
      const double nrm = std::sqrt(read_scalar(h, 5));
      if (i == 1) first = nrm;
      last = nrm;
    }
    dot_into(h, L, f->buf.p, f->buf.p, 5);
    const double fn = std::sqrt(read_scalar(h, 5));
    if (first <= 1e-300 || first <= 2.220446049250313e-16 * fn) {
      *rate = 0.0;
      return;
    }
    *rate = std::pow(last / first, 1.0 / (double)(n_cycles - 1));
  });
}

namespace {
// The PCG solve of tpmg_pcg on raw finest-level device buffers f (read) and x (written).
void pcg_impl(tpmg_hierarchy h, const double* fp, double* xp, int64_t n, double tol, int max_iter,
              double* res_hist, int* iters, int* solve_status) {
    const int L = h->finest();
    tpmg_context ctx = h->ctx;
    cudaStream_t s = ctx->stream;
    if (!h->h_pub && !h->multi()) {  // before any iteration graph is captured
      CUDA_CHECK(cudaHostAlloc(&h->h_pub, sizeof(tpmg::PcgPublish), cudaHostAllocMapped));
      std::memset(h->h_pub, 0, sizeof(tpmg::PcgPublish));
      CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->d_pub), h->h_pub, 0));
      CUDA_CHECK(cudaMalloc(&h->d_seq, sizeof(unsigned)));
      CUDA_CHECK(cudaMemsetAsync(h->d_seq, 0, sizeof(unsigned), s));
      h->host_seq = 0;
    }
    CUDA_CHECK(cudaMemsetAsync(xp, 0, n * 8, s));
    // r_0 = f.  The fused schedule never copies it: the prologue reads f, and the first
    // iteration's pre-sweep reads f and writes r_1 = f - alpha q into r (vcycle f_pre)
    const double* r0p = h->pcg_fused ? fp : h->r.p;
    if (h->pcg_fused) h->f_first = fp;
    // prologue, one graph per right-hand side: |r_0|^2; z_0 = M r_0 straight into the direction
    // buffer (p_1 = z_0; the first iteration's V-cycle writes z itself: no 1 GB device copy);
    // rho_0 = r_0.z_0 -- then one synchronisation reads both scalars
    run_graph(h, {G_PROLOGUE, fp, nullptr}, [&] {
      if (!h->pcg_fused)
        CUDA_CHECK(cudaMemcpyAsync(h->r.p, fp, n * 8, cudaMemcpyDeviceToDevice, s));
      dot_into(h, L, r0p, r0p, 2);
      vcycle(h, L, r0p, h->p.p, h->tmp.p, true);
      dot_into(h, L, r0p, h->p.p, 0);
    });
    h->pcur = 0;
    // (published through mapped memory where possible: a copy-engine readback would queue
    // behind the large device-to-host copies of tpmg_pcg_host_batch)
    int err0 = 0;
    if (publish_ok(h)) {
      publish(h);
      err0 = wait_publish_raw(h);
    } else {
      CUDA_CHECK(cudaMemcpyAsync(h->h_scal, h->scal.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
      err0 = sync_err(h);
    }
    const double r0 = std::sqrt(h->h_scal[2]);
    if (res_hist) res_hist[0] = r0;
    *iters = 0;
    *solve_status = TPMG_OK;
    if (r0 == 0.0) {  // x = 0 is the solution; the V-cycle of a zero right-hand side is moot
      if (err0) clear_err(h);
      return;
    }
    if (err0) {
      clear_err(h);
      throw Error(TPMG_E_SINGULAR, "thomas_solve: zero pivot");
    }
    if (!(h->h_scal[0] > 0.0)) {
      *solve_status = TPMG_BREAKDOWN;
      return;
    }
    // fused schedule: the last iteration's x += alpha p is still pending when the loop ends
    auto finish_x = [&] {
      if (h->pcg_fused && *iters > 0) {  // max_iter = 0: no pending update, x stays 0
        tpmg::launch_pcg_xfinal(ctx->launch(), n, h->scal.p, h->pbuf(h->pcur), xp);
        if (publish_ok(h)) {
          publish(h);
          wait_publish(h);
        } else {
          sync_check(h);
        }
      }
    };
    static const bool debug_timing = [] {
      const char* e = getenv("TPMG_DEBUG_TIMING");
      return e && atoi(e) != 0;
    }();
    for (int it = 1; it <= max_iter; ++it) {
      if (it == 2 && device_loop_ok(h, max_iter)) {
        // iterations 2.. as one graph launch: the convergence test runs on the device
        cudaGraphExec_t ge = loop_graph(h, xp);
        *h->h_loop = tpmg::PcgLoop{r0, tol, max_iter, 1, 1, 0};
        CUDA_CHECK(cudaMemcpyAsync(h->d_loop, h->h_loop, sizeof(tpmg::PcgLoop),
                                   cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaGraphLaunch(ge, s));
        CUDA_CHECK(cudaMemcpyAsync(h->h_loop, h->d_loop, sizeof(tpmg::PcgLoop),
                                   cudaMemcpyDeviceToHost, s));
        sync_check(h);
        const tpmg::PcgLoop st = *h->h_loop;
        const int ran = st.it - 1;  // iterations executed by the graph
        ctx->launches += (int64_t)ran * h->loop_kernels_per_iter;
        if (h->fused_ap && (ran & 1)) h->pcur ^= 1;
        if (res_hist && st.iters >= 2)
          CUDA_CHECK(cudaMemcpy(res_hist + 2, h->d_hist.p + 2, (st.iters - 1) * sizeof(double),
                                cudaMemcpyDeviceToHost));
        *iters = st.iters;
        switch (st.exit) {
          case 1: finish_x(); return;
          case 2: *solve_status = TPMG_DIVERGED; finish_x(); return;
          case 3: *solve_status = TPMG_BREAKDOWN; finish_x(); return;
          case 4: *solve_status = TPMG_BREAKDOWN; return;
          default: *solve_status = TPMG_NOT_CONVERGED; finish_x(); return;
        }
      }
      const auto t_a = std::chrono::steady_clock::now();
      run_iteration(h, xp, it == 1);
      const auto t_b = std::chrono::steady_clock::now();
      if (publish_ok(h)) {
        wait_publish(h);
      } else {
        CUDA_CHECK(cudaMemcpyAsync(h->h_scal, h->scal.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
        sync_check(h);
      }
      probe_collect(h);
      if (debug_timing) {  // TPMG_DEBUG_TIMING=1: host time to queue / wait for each iteration
        const auto t_c = std::chrono::steady_clock::now();
        fprintf(stderr, "[tpmg] it %d queue %.1f us wait %.1f us\n", it,
                std::chrono::duration<double, std::micro>(t_b - t_a).count(),
                std::chrono::duration<double, std::micro>(t_c - t_b).count());
      }
      const double pq = h->h_scal[1], rr = h->h_scal[2], rho_new = h->h_scal[3];
      if (!(pq > 0.0)) {
        *solve_status = TPMG_BREAKDOWN;
        return;
      }
      const double rn = std::sqrt(rr);
      if (res_hist) res_hist[it] = rn;
      *iters = it;
      if (rn / r0 <= tol) {
        finish_x();
        return;
      }
      if (rn / r0 > 1e4) {
        *solve_status = TPMG_DIVERGED;
        finish_x();
        return;
      }
      if (!(rho_new > 0.0)) {
        *solve_status = TPMG_BREAKDOWN;
        finish_x();
        return;
      }
    }
    *solve_status = TPMG_NOT_CONVERGED;
    finish_x();
}
}  // namespace

int tpmg_pcg(tpmg_hierarchy h, tpmg_field f, tpmg_field x, double tol, int max_iter,
             double* res_hist, int* iters, int* solve_status) {
  return guard(h->ctx, [&] {
    same_hier(h, f); same_hier(h, x);
    const int L = h->finest();
    if (f->level != L || x->level != L) throw Error(TPMG_E_SHAPE, "pcg: fields must be finest");
    if (max_iter < 0) throw Error(TPMG_E_CONFIG, "max_iter must be >= 0");
    pcg_impl(h, f->buf.p, x->buf.p, f->buf.n, tol, max_iter, res_hist, iters, solve_status);
  });
}

// Solves `count` independent right-hand sides from host memory, the transfers overlapped with
// the solves: while right-hand side i is solved on the library stream, the copy stream uploads
// (and permutes) right-hand side i+1 into the other device buffer and permutes and downloads
// solution i-1.  Each solve is tpmg_pcg's, so every solution, history and status is bitwise
// the one-at-a-time result.  Host buffers should be pinned for the copies to overlap.
int tpmg_pcg_host_batch(tpmg_hierarchy h, int count, const double* const* f_hosts,
                        double* const* x_hosts, int layout, double tol, int max_iter,
                        double* res_hist, int* iters, int* solve_status) {
  return guard(h->ctx, [&] {
    if (count < 0 || max_iter < 0) throw Error(TPMG_E_CONFIG, "count and max_iter must be >= 0");
    if (count > 0 && (!f_hosts || !x_hosts || !iters || !solve_status))
      throw Error(TPMG_E_CONFIG, "null argument");
    if (layout != TPMG_LAYOUT_X_FASTEST && layout != TPMG_LAYOUT_K_FASTEST)
      throw Error(TPMG_E_CONFIG, "unknown layout");
    tpmg_context ctx = h->ctx;
    const int L = h->finest();
    const int64_t n = h->lv[L].plane * h->nz;
    auto& B = h->bat;
    if (!B.copy) {
      CUDA_CHECK(cudaStreamCreateWithFlags(&B.copy, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        B.F[i].alloc(n);
        B.X[i].alloc(n);
        CUDA_CHECK(cudaEventCreateWithFlags(&B.up[i], cudaEventDisableTiming));
        CUDA_CHECK(cudaEventCreateWithFlags(&B.done[i], cudaEventDisableTiming));
        CUDA_CHECK(cudaEventCreateWithFlags(&B.down[i], cudaEventDisableTiming));
      }
      B.stage_in.alloc(n);
      B.stage_out.alloc(n);
    }
    const tpmg::Launch cl{B.copy, &ctx->launches};
    const bool kf = layout == TPMG_LAYOUT_K_FASTEST;
    // the copy stream's first work may not overtake anything queued on the library stream
    CUDA_CHECK(cudaEventRecord(B.done[0], ctx->stream));
    CUDA_CHECK(cudaEventRecord(B.done[1], ctx->stream));
    CUDA_CHECK(cudaEventRecord(B.down[0], ctx->stream));
    CUDA_CHECK(cudaEventRecord(B.down[1], ctx->stream));
    auto upload = [&](int i) {  // f_i -> F[i % 2], after the solve that last read F[i % 2]
      const int b = i % 2;
      CUDA_CHECK(cudaStreamWaitEvent(B.copy, B.done[b], 0));
      if (kf) {
        CUDA_CHECK(cudaMemcpyAsync(B.stage_in.p, f_hosts[i], n * 8, cudaMemcpyHostToDevice, B.copy));
        tpmg::launch_kfast_to_xfast(cl, h->lv[L].plane, h->nz, B.stage_in.p, B.F[b].p);
      } else {
        CUDA_CHECK(cudaMemcpyAsync(B.F[b].p, f_hosts[i], n * 8, cudaMemcpyHostToDevice, B.copy));
      }
      CUDA_CHECK(cudaEventRecord(B.up[b], B.copy));
    };
    auto download = [&](int i) {  // X[i % 2] -> x_i, after solve i
      const int b = i % 2;
      CUDA_CHECK(cudaStreamWaitEvent(B.copy, B.done[b], 0));
      if (kf) {
        tpmg::launch_xfast_to_kfast(cl, h->lv[L].plane, h->nz, B.X[b].p, B.stage_out.p);
        CUDA_CHECK(cudaMemcpyAsync(x_hosts[i], B.stage_out.p, n * 8, cudaMemcpyDeviceToHost, B.copy));
      } else {
        CUDA_CHECK(cudaMemcpyAsync(x_hosts[i], B.X[b].p, n * 8, cudaMemcpyDeviceToHost, B.copy));
      }
      CUDA_CHECK(cudaEventRecord(B.down[b], B.copy));
    };
    try {
      if (count > 0) upload(0);
      for (int i = 0; i < count; ++i) {
        const int b = i % 2;
        if (i + 1 < count) upload(i + 1);  // overlaps solve i
        CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, B.up[b], 0));
        CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, B.down[b], 0));  // solution i-2 left X[b]
        pcg_impl(h, B.F[b].p, B.X[b].p, n, tol, max_iter,
                 res_hist ? res_hist + (int64_t)i * (max_iter + 1) : nullptr, iters + i,
                 solve_status + i);
        CUDA_CHECK(cudaEventRecord(B.done[b], ctx->stream));
        download(i);  // overlaps solve i+1
      }
    } catch (...) {
      // no copy may still touch the caller's host buffers once the error is returned
      cudaStreamSynchronize(B.copy);
      throw;
    }
    CUDA_CHECK(cudaStreamSynchronize(B.copy));
  });
}

int tpmg_pcg_host(tpmg_hierarchy h, const double* f_host, double* x_host, int layout, double tol,
                  int max_iter, double* res_hist, int* iters, int* solve_status) {
  tpmg_field f = nullptr, x = nullptr;
  int rc = tpmg_field_create(h, h->finest(), &f);
  if (rc == TPMG_OK) rc = tpmg_field_create(h, h->finest(), &x);
  if (rc == TPMG_OK) rc = tpmg_field_upload(f, f_host, layout);
  if (rc == TPMG_OK) rc = tpmg_pcg(h, f, x, tol, max_iter, res_hist, iters, solve_status);
  if (rc == TPMG_OK) rc = tpmg_field_download(x, x_host, layout);
  tpmg_field_destroy(f);
  tpmg_field_destroy(x);
  return rc;
}

// ---- Richardson and right-preconditioned BiCGStab -------------------------
// Preconditioner M^{-1}: mu V-cycles on A e = r from e = 0; the finest-level
// operator and V-cycle are the PCG ones.  Dot products are the deterministic device dots, the
// scalars are formed on the host in IEEE double, element-wise updates in a fixed order
// (k_vec_lin), so the CPU restatement (tpmgo_richardson / tpmgo_bicgstab) is bitwise equal.
namespace {
void precondition(tpmg_hierarchy h, int mu, const double* r, double* e) {
  const int L = h->finest();
  for (int i = 0; i < mu; ++i) vcycle(h, L, r, e, h->tmp.p, i == 0);
  ++h->n_precond;
}
double dot_now(tpmg_hierarchy h, int64_t n, const double* a, const double* b) {
  (void)n;  // finest-level fields
  dot_into(h, h->finest(), a, b, 4);
  return read_scalar(h, 4);
}
}  // namespace

int tpmg_richardson(tpmg_hierarchy h, tpmg_field f, tpmg_field x, double tol, int max_iter,
                    int mu, double* res_hist, int* iters, int* solve_status) {
  return guard(h->ctx, [&] {
    same_hier(h, f); same_hier(h, x);
    const int L = h->finest();
    if (f->level != L || x->level != L) throw Error(TPMG_E_SHAPE, "richardson: fields must be finest");
    if (max_iter < 0 || mu < 1) throw Error(TPMG_E_CONFIG, "richardson: max_iter >= 0, mu >= 1");
    tpmg_context ctx = h->ctx;
    const int64_t n = f->buf.n;
    cudaStream_t st = ctx->stream;
    h->n_precond = h->n_matvec = 0;
    if (!h->k_rh.p) h->k_rh.alloc(n);
    double* e = h->k_rh.p;
    CUDA_CHECK(cudaMemsetAsync(x->buf.p, 0, n * 8, st));
    CUDA_CHECK(cudaMemcpyAsync(h->r.p, f->buf.p, n * 8, cudaMemcpyDeviceToDevice, st));
    const double r0 = std::sqrt(dot_now(h, n, h->r.p, h->r.p));
    if (res_hist) res_hist[0] = r0;
    *iters = 0;
    *solve_status = TPMG_OK;
    if (r0 == 0.0) return;
    for (int it = 1; it <= max_iter; ++it) {
      precondition(h, mu, h->r.p, e);                                   // e = M^{-1} r
      tpmg::launch_vec_lin(ctx->launch(), tpmg::VL_ADD, n, x->buf.p, e, nullptr, 0.0, 0.0);
      apply_level(h, L, tpmg::APPLY_RESID, x->buf.p, f->buf.p, h->r.p); // r = f - A x
      ++h->n_matvec;
      const double rn = std::sqrt(dot_now(h, n, h->r.p, h->r.p));
      if (res_hist) res_hist[it] = rn;
      *iters = it;
      if (rn / r0 <= tol) return;
      if (!(rn / r0 <= 1e4)) {
        *solve_status = TPMG_DIVERGED;
        return;
      }
    }
    *solve_status = TPMG_NOT_CONVERGED;
  });
}

int tpmg_bicgstab(tpmg_hierarchy h, tpmg_field f, tpmg_field x, double tol, int max_iter,
                  int mu, double* res_hist, int* iters, int* solve_status) {
  return guard(h->ctx, [&] {
    same_hier(h, f); same_hier(h, x);
    const int L = h->finest();
    if (f->level != L || x->level != L) throw Error(TPMG_E_SHAPE, "bicgstab: fields must be finest");
    if (max_iter < 0 || mu < 1) throw Error(TPMG_E_CONFIG, "bicgstab: max_iter >= 0, mu >= 1");
    tpmg_context ctx = h->ctx;
    const int64_t n = f->buf.n;
    cudaStream_t st = ctx->stream;
    h->n_precond = h->n_matvec = 0;
    for (DevBuf* b : {&h->k_rh, &h->k_p, &h->k_v, &h->k_ph, &h->k_s, &h->k_sh, &h->k_t})
      if (!b->p) b->alloc(n);
    double *r = h->r.p, *rh = h->k_rh.p, *p = h->k_p.p, *v = h->k_v.p, *ph = h->k_ph.p;
    double *sv = h->k_s.p, *sh = h->k_sh.p, *t = h->k_t.p, *xp = x->buf.p;
    CUDA_CHECK(cudaMemsetAsync(xp, 0, n * 8, st));
    CUDA_CHECK(cudaMemcpyAsync(r, f->buf.p, n * 8, cudaMemcpyDeviceToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(rh, f->buf.p, n * 8, cudaMemcpyDeviceToDevice, st));  // r^ = r_0
    CUDA_CHECK(cudaMemsetAsync(p, 0, n * 8, st));
    CUDA_CHECK(cudaMemsetAsync(v, 0, n * 8, st));
    const double r0 = std::sqrt(dot_now(h, n, r, r));
    if (res_hist) res_hist[0] = r0;
    *iters = 0;
    *solve_status = TPMG_OK;
    if (r0 == 0.0) return;
    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    const auto lin = [&](int op, double* y, const double* a, const double* b, double s1, double s2) {
      tpmg::launch_vec_lin(ctx->launch(), op, n, y, a, b, s1, s2);
    };
    for (int it = 1; it <= max_iter; ++it) {
      const double rho = dot_now(h, n, rh, r);
      if (!(std::fabs(rho) >= 1e-30 * r0 * r0)) {  // rho-breakdown
        *solve_status = TPMG_BREAKDOWN;
        return;
      }
      const double beta = (rho / rho_prev) * (alpha / omega);
      lin(tpmg::VL_P, p, r, v, beta, omega);                   // p = r + beta (p - omega v)
      CUDA_CHECK(cudaMemsetAsync(ph, 0, n * 8, st));
      precondition(h, mu, p, ph);                              // p^ = M^{-1} p
      apply_level(h, L, tpmg::APPLY_AU, ph, nullptr, v);      // v = A p^
      ++h->n_matvec;
      const double rv = dot_now(h, n, rh, v);
      if (!(rv != 0.0)) {
        *solve_status = TPMG_BREAKDOWN;
        return;
      }
      alpha = rho / rv;
      lin(tpmg::VL_AXMY, sv, r, v, alpha, 0.0);               // s = r - alpha v
      const double sn = std::sqrt(dot_now(h, n, sv, sv));
      if (sn / r0 <= tol) {                                    // converged at the half step
        lin(tpmg::VL_AXPY, xp, ph, nullptr, alpha, 0.0);       // x = x + alpha p^
        if (res_hist) res_hist[it] = sn;
        *iters = it;
        return;
      }
      CUDA_CHECK(cudaMemsetAsync(sh, 0, n * 8, st));
      precondition(h, mu, sv, sh);                             // s^ = M^{-1} s
      apply_level(h, L, tpmg::APPLY_AU, sh, nullptr, t);      // t = A s^
      ++h->n_matvec;
      const double tt = dot_now(h, n, t, t);
      const double ts = dot_now(h, n, t, sv);
      if (!(tt != 0.0)) {
        *solve_status = TPMG_BREAKDOWN;
        return;
      }
      omega = ts / tt;
      lin(tpmg::VL_X2, xp, ph, sh, alpha, omega);              // x = (x + alpha p^) + omega s^
      lin(tpmg::VL_AXMY, r, sv, t, omega, 0.0);                // r = s - omega t
      const double rn = std::sqrt(dot_now(h, n, r, r));
      if (res_hist) res_hist[it] = rn;
      *iters = it;
      if (rn / r0 <= tol) return;
      if (!(rn / r0 <= 1e4)) {
        *solve_status = TPMG_DIVERGED;
        return;
      }
      if (!(omega != 0.0)) {
        *solve_status = TPMG_BREAKDOWN;
        return;
      }
      rho_prev = rho;
    }
    *solve_status = TPMG_NOT_CONVERGED;
  });
}

int tpmg_solver_counts(tpmg_hierarchy h, int64_t* n_precond, int64_t* n_matvec) {
  *n_precond = h->n_precond;
  *n_matvec = h->n_matvec;
  return TPMG_OK;
}

int tpmg_nccl_call_count(int64_t* out) {
  if (!out) return TPMG_E_CONFIG;
  *out = g_nccl_calls.load(std::memory_order_relaxed);
  return TPMG_OK;
}

int tpmg_kernel_launch_count(tpmg_context ctx, int64_t* out) {
  *out = ctx->launches;
  return TPMG_OK;
}

int tpmg_time_kernel(tpmg_hierarchy h, int kernel_id, int level, int reps, double* avg_ms) {
  return guard(h->ctx, [&] {
    if (level < 0 || level >= (int)h->lv.size()) throw Error(TPMG_E_SHAPE, "level out of range");
    if (reps < 1) throw Error(TPMG_E_CONFIG, "reps must be >= 1");
    const bool transfer = kernel_id == TPMG_K_RESID_RESTRICT || kernel_id == TPMG_K_PROLONG_ADD ||
                          kernel_id == TPMG_K_RESTRICT;
    if (transfer && level < 1) throw Error(TPMG_E_SHAPE, "transfers need a fine level >= 1");
    for (Level& Lm : h->lv) Lm.f_pending = false;  // no early-posted halo belongs to these calls
    Level& L = h->lv[level];
    const int64_t n = L.plane * h->nz;
    const bool pcg_kernel = kernel_id == TPMG_K_PCG_DIRECTION || kernel_id == TPMG_K_PCG_RUPDATE ||
                            kernel_id == TPMG_K_PCG_POSTSWEEP;
    if (pcg_kernel && !(tpmg::jacobi_fusable(h->lv[level].coef(h->nz)) &&
                        tpmg::pcg_ap_fusable(h->lv[level].coef(h->nz))))
      throw Error(TPMG_E_SHAPE, "the fused PCG kernels need a tiled level");
    DevBuf a, b, c, d, cc;
    a.alloc(n); b.alloc(n); c.alloc(n);
    if (pcg_kernel) d.alloc(n);
    const int64_t ncoarse = transfer ? h->lv[level - 1].plane * h->nz : 1;
    cc.alloc(ncoarse);
    // seeded pseudo-random operands (constant fields make A u vanish in places, which would
    // time the smoother's exact-division fallback instead of its hot path)
    tpmg::launch_fill_hash(h->ctx->launch(), n, a.p, 1.0, 1);
    tpmg::launch_fill_hash(h->ctx->launch(), n, b.p, 1.0, 2);
    tpmg::launch_fill_hash(h->ctx->launch(), ncoarse, cc.p, 1.0, 3);
    if (pcg_kernel) {
      tpmg::launch_fill_hash(h->ctx->launch(), n, d.p, 1.0, 4);
      // PCG scalars rho = 1, p.q = 2, rho_new = 0.5 (alpha = 0.5, beta = 0.5); the r-update
      // kernel rewrites r in place, so its timing reps start from slightly different r
      const double sc[4] = {1.0, 2.0, 0.0, 0.5};
      CUDA_CHECK(cudaMemcpyAsync(h->scal.p, sc, sizeof(sc), cudaMemcpyHostToDevice,
                                 h->ctx->stream));
    }
    auto once = [&] {
      switch (kernel_id) {
        case TPMG_K_APPLY: apply_level(h, level, tpmg::APPLY_AU, a.p, nullptr, c.p); break;
        case TPMG_K_RESIDUAL: apply_level(h, level, tpmg::APPLY_RESID, a.p, b.p, c.p); break;
        case TPMG_K_JACOBI: sweep(h, level, a.p, b.p, c.p); break;
        case TPMG_K_JACOBI_ZERO: sweep(h, level, nullptr, b.p, c.p); break;
        case TPMG_K_RESID_RESTRICT: resid_restrict(h, level, a.p, b.p, cc.p, c.p); break;
        case TPMG_K_PROLONG_ADD: prolong_level(h, level - 1, cc.p, c.p, true); break;
        case TPMG_K_RESTRICT: restrict_plain(h, level, a.p, cc.p); break;
        case TPMG_K_PCG_DIRECTION: {  // z = a, p_old = b, p_new = c, x = d (finest, tiled)
          Level& F = h->lv[level];
          int nb = 0;
          tpmg::launch_pcg_ap(h->ctx->launch(), h->vcoef(), F.coef(h->nz), h->xi, a.p,
                              tpmg::self_halo(a.p, F.nx, F.ny, F.plane), b.p,
                              tpmg::self_halo(b.p, F.nx, F.ny, F.plane), c.p, nullptr, d.p,
                              h->scal.p, h->partials.p, &nb);
          break;
        }
        case TPMG_K_PCG_RUPDATE: {  // r = a (updated in place), p = b, z = c
          tpmg::PcgFuse fz;
          fz.r = a.p;
          fz.p = b.p;
          fz.s = h->scal.p;
          fz.partials = h->partials.p;
          sweep(h, level, nullptr, a.p, c.p, &fz, 2);
          break;
        }
        case TPMG_K_PCG_POSTSWEEP: {  // u = a, r = b (the sweep's f), z = c; r.z partials
          tpmg::PcgFuse fz;
          fz.r = b.p;
          fz.s = h->scal.p;
          fz.partials = h->partials.p;
          sweep(h, level, a.p, b.p, c.p, &fz, 3);
          break;
        }
        default: throw Error(TPMG_E_CONFIG, "unknown kernel id");
      }
    };
    once();  // warm-up
    cudaEvent_t e0, e1;
    CUDA_CHECK(cudaEventCreate(&e0));
    CUDA_CHECK(cudaEventCreate(&e1));
    CUDA_CHECK(cudaEventRecord(e0, h->ctx->stream));
    for (int r = 0; r < reps; ++r) once();
    CUDA_CHECK(cudaEventRecord(e1, h->ctx->stream));
    CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    sync_check(h);
    *avg_ms = ms / reps;
  });
}

int tpmg_kernel_probe(tpmg_hierarchy h, int enable) {
  return guard(h->ctx, [&] {
    if ((enable != 0) != h->probe_on) {  // cached iteration graphs carry (or lack) the probes
      CUDA_CHECK(cudaStreamSynchronize(h->ctx->stream));
      for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second.exec);
      h->graphs.clear();
      for (auto& kv : h->loop_graphs) cudaGraphExecDestroy(kv.second);
      h->loop_graphs.clear();
    }
    h->probe_on = enable != 0;
    h->probe_pending = 0;
    for (auto& pr : h->probes) {
      pr.total_ms = 0.0;
      pr.launches = 0;
    }
  });
}

int tpmg_kernel_probe_read(tpmg_hierarchy h, int kernel_id, double* total_ms, int64_t* launches) {
  return guard(h->ctx, [&] {
    if (kernel_id < 0 || kernel_id >= tpmg_hierarchy_s::kProbes)
      throw Error(TPMG_E_CONFIG, "unknown kernel id");
    if (total_ms) *total_ms = h->probes[kernel_id].total_ms;
    if (launches) *launches = h->probes[kernel_id].launches;
  });
}

int tpmg_set_use_graphs(tpmg_hierarchy h, int enable) {
  h->use_graphs = enable != 0;
  return TPMG_OK;
}

}  // extern "C"
