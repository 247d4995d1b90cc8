"""Host-side mirror of the reference's operator / smoother / transfer / solver interface.

Function names and argument meaning follow the reference (proj/include/tpmg/):
``apply_operator`` (discretization.hpp:262-287), ``smooth`` (relaxation.hpp:63-108),
``restrict_field`` / ``restrict_field_transpose`` (multigrid.hpp:29-69),
``prolongate_field`` (multigrid.hpp:74-100), ``build_hierarchy_coefficients``
(multigrid.hpp:242-272), ``v_cycle`` (multigrid.hpp:276-299), ``measure_cycle_rate``
(multigrid.hpp:302-321) plus the PCG driver of BASELINE.json.  Errors are raised as the
reference's exception types (types.hpp:24-58).  Every call goes through the C-ABI of
``libtpmg_b200.so`` into hand-written sm_100a kernels; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
import sys
import time

import numpy as np

from . import _capi
from ._capi import ContextParams, FactorizedProfiles, FullProfiles, GridDesc, MGConfig

K_FASTEST, X_FASTEST = 0, 1
(K_APPLY, K_JACOBI, K_JACOBI_ZERO, K_RESID_RESTRICT, K_PROLONG_ADD, K_RESTRICT, K_RESIDUAL,
 K_PCG_DIRECTION, K_PCG_RUPDATE, K_PCG_POSTSWEEP, K_REDUCE) = range(11)
LINEAR, INJECTION = 0, 1
SUMMATION, TRANSPOSE = 0, 1
OK, E_CONFIG, E_SHAPE, E_NONFINITE, E_FINGERPRINT, E_SINGULAR, E_CAP, E_CUDA, E_NCCL = range(9)
NOT_CONVERGED, BREAKDOWN, DIVERGED = 9, 10, 11


class TpmgError(RuntimeError):
    code = -1


class config_error(TpmgError):
    code = E_CONFIG


class shape_error(TpmgError):
    code = E_SHAPE


class nonfinite_error(TpmgError):
    code = E_NONFINITE


class fingerprint_error(TpmgError):
    code = E_FINGERPRINT


class singular_error(TpmgError):
    code = E_SINGULAR


class cap_error(TpmgError):
    code = E_CAP


class cuda_error(TpmgError):
    code = E_CUDA


class nccl_error(TpmgError):
    code = E_NCCL


_ERRORS = {c.code: c for c in (config_error, shape_error, nonfinite_error, fingerprint_error,
                                singular_error, cap_error, cuda_error, nccl_error)}


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Context:
    """One GPU (rank) -- tpmg_init / tpmg_finalize."""

    def __init__(self, device: int = 0, rank: int = 0, world_size: int = 1, px: int = 1,
                 py: int = 1, nccl_id: bytes | None = None, variant: str = "exact",
                 ipc_session: str | None = None):
        """One rank.  world_size > 1: NCCL transport (nccl_id from rank 0), or with
        `ipc_session` the CUDA-IPC transport (tpmg_init_ipc; every rank passes the same
        session string)."""
        self.lib = _capi.load(variant)
        self._idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        prm = ContextParams(device, rank, world_size, px, py,
                            C.cast(self._idbuf, C.c_void_p) if self._idbuf else None)
        h = C.c_void_p()
        self._h = None
        if ipc_session:
            self._check(self.lib.tpmg_init_ipc(C.byref(prm), ipc_session.encode(), C.byref(h)))
        else:
            self._check(self.lib.tpmg_init(C.byref(prm), C.byref(h)))
        self._h = h
        self.rank, self.world_size, self.px, self.py = rank, world_size, px, py

    def _check(self, rc: int):
        if rc != OK:
            msg = self.lib.tpmg_last_error(self._h if self._h else None)
            raise _ERRORS.get(rc, TpmgError)(f"{self.lib.tpmg_status_string(rc).decode()}: "
                                             f"{msg.decode() if msg else ''}")

    @staticmethod
    def nccl_unique_id(variant: str = "exact") -> bytes:
        lib = _capi.load(variant)
        buf = C.create_string_buffer(128)
        rc = lib.tpmg_nccl_unique_id(buf)
        if rc != OK:
            raise nccl_error(lib.tpmg_last_error(None).decode())
        return buf.raw

    def stream_handle(self) -> int:
        """cudaStream_t (as int) the library orders all work on."""
        s = C.c_void_p()
        self._check(self.lib.tpmg_context_stream(self._h, C.byref(s)))
        return s.value or 0

    def kernel_launches(self) -> int:
        n = C.c_int64()
        self.lib.tpmg_kernel_launch_count(self._h, C.byref(n))
        return n.value

    def nccl_calls(self) -> int:
        """NCCL API calls issued by this process so far (0 unless a transport uses NCCL)."""
        n = C.c_int64()
        self.lib.tpmg_nccl_call_count(C.byref(n))
        return n.value

    # Handles are freed parent-last whatever order the garbage collector finalises them in
    # (objects in a reference cycle, e.g. held by a traceback, are finalised in arbitrary
    # order): a parent closed while children are alive only marks itself, and the last child
    # to close frees it.
    _live_children = 0
    _pending_close = False

    def _child_closed(self):
        self._live_children -= 1
        if self._pending_close and self._live_children == 0:
            self.close()

    def close(self):
        if self._live_children > 0:
            self._pending_close = True
            return
        if self._h is not None:
            self.lib.tpmg_finalize(self._h)
            self._h = None

    def __del__(self):
        # at interpreter shutdown the destruction order of handles is arbitrary: leave the
        # device memory to the driver instead of freeing through possibly-dead parents
        if sys.is_finalizing():
            return
        try:
            self.close()
        except Exception:
            pass


class Field:
    """Device-resident Field (discretization.hpp:106-120) of one level, stored [k][y][x]."""

    def __init__(self, hier: "Hierarchy", level: int):
        self.hier, self.level = hier, level
        h = C.c_void_p()
        hier.ctx._check(hier.lib.tpmg_field_create(hier._h, level, C.byref(h)))
        self._h = h
        hier._live_children += 1
        self.nx, self.ny, self.nz = hier.level_shape(level)[:3]

    @property
    def size(self) -> int:
        return self.nx * self.ny * self.nz

    def upload(self, a: np.ndarray, layout: int = X_FASTEST) -> "Field":
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        if a.size != self.size:
            raise shape_error(f"upload: {a.size} values for a field of {self.size}")
        self.hier.ctx._check(self.hier.lib.tpmg_field_upload(self._h, _p(a), layout))
        return self

    def download(self, layout: int = X_FASTEST, out: np.ndarray | None = None) -> np.ndarray:
        """Copy to the host; `out` (e.g. a pinned buffer) is filled in place when given."""
        if out is not None:
            if out.dtype != np.float64 or not out.flags.c_contiguous or out.size != self.size:
                raise shape_error("download: out must be a contiguous float64 array of the field size")
            self.hier.ctx._check(self.hier.lib.tpmg_field_download(self._h, _p(out.reshape(-1)), layout))
            return out
        out = np.empty(self.size, dtype=np.float64)
        self.hier.ctx._check(self.hier.lib.tpmg_field_download(self._h, _p(out), layout))
        return out.reshape(self.nz, self.ny, self.nx) if layout == X_FASTEST else out

    def fill(self, v: float) -> "Field":
        self.hier.ctx._check(self.hier.lib.tpmg_field_fill(self._h, C.c_double(v)))
        return self

    def copy_from(self, other: "Field") -> "Field":
        self.hier.ctx._check(self.hier.lib.tpmg_field_copy(self._h, other._h))
        return self

    def norm(self) -> float:
        out = C.c_double()
        self.hier.ctx._check(self.hier.lib.tpmg_norm(self.hier._h, self._h, C.byref(out)))
        return out.value

    def close(self):
        if getattr(self, "_h", None) is not None:
            self.hier.lib.tpmg_field_destroy(self._h)
            self._h = None
            self.hier._child_closed()

    def __del__(self):
        # at interpreter shutdown the destruction order of handles is arbitrary: leave the
        # device memory to the driver instead of freeing through possibly-dead parents
        if sys.is_finalizing():
            return
        try:
            self.close()
        except Exception:
            pass


class Hierarchy:
    """MultigridHierarchy built by build_hierarchy_coefficients (multigrid.hpp:242-272)."""

    def __init__(self, ctx: Context, problem, **over):
        self.ctx, self.lib = ctx, ctx.lib
        P = problem
        kw = P.mg_kwargs()
        kw.update(over)
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in
                      (P.z_faces, P.beta_r, P.alpha_s_r, P.alpha_r_r, P.beta_s, P.alpha_r_s,
                       P.alpha_s_s)]
        z, br, asr, arr, bs, ars, ass = self._keep
        grid = GridDesc(P.nx, P.ny, P.hx, P.hy, P.nz, _p(z))
        xr = xs = None
        if getattr(P, "xi_r_r", None) is not None:
            xr = np.ascontiguousarray(P.xi_r_r, dtype=np.float64)
            xs = np.ascontiguousarray(P.xi_r_s, dtype=np.float64)
            self._keep += [xr, xs]
        prof = FactorizedProfiles(_p(br), _p(asr), _p(arr), _p(xr), _p(bs), _p(ars), _p(xs), _p(ass))
        cfg = MGConfig(kw.get("smoother", 0), kw["relax"], kw["prolongation"], kw["restriction"],
                       kw["nu_pre"], kw["nu_post"], kw["depth"], kw.get("agglomerate", 0))
        h = C.c_void_p()
        self._h = None
        coef = getattr(P, "coef", "factorized")
        if coef == "factorized":
            ctx._check(self.lib.tpmg_hier_create(ctx._h, C.byref(grid), C.byref(prof),
                                                 C.c_double(P.omega), C.byref(cfg), C.byref(h)))
        elif coef == "partial":
            ar = np.ascontiguousarray(P.dense["alpha_r"], dtype=np.float64)
            self._keep.append(ar)
            ctx._check(self.lib.tpmg_hier_create_partial(ctx._h, C.byref(grid), C.byref(prof),
                                                         _p(ar), C.c_double(P.omega),
                                                         C.byref(cfg), C.byref(h)))
        elif coef == "full":
            d = {k: (None if v is None else np.ascontiguousarray(v, dtype=np.float64))
                 for k, v in P.dense.items()}
            self._keep += [v for v in d.values() if v is not None]
            fp = FullProfiles(_p(d["beta"]), _p(d["alpha_s"]), _p(d["alpha_r"]), _p(d["xi_r"]))
            ctx._check(self.lib.tpmg_hier_create_full(ctx._h, C.byref(grid), C.byref(fp),
                                                      C.c_double(P.omega), C.byref(cfg),
                                                      C.byref(h)))
        else:
            raise config_error(f"unknown coefficient storage {coef!r}")
        self._h = h
        ctx._live_children += 1
        self._keep = None
        self.problem = P
        n = C.c_int()
        self.lib.tpmg_hier_n_levels(self._h, C.byref(n))
        self.n_levels = n.value
        self.finest = self.n_levels - 1

    @classmethod
    def from_tables(cls, ctx: Context, nz, nnb, nchild, ncells, nedges, nbr, cedge, children,
                    prol_d1, prol_d2, bv, sv, av, xv, bh, ah, xh, sh, relax, prolongation,
                    restriction, nu_pre, nu_post) -> "Hierarchy":
        """An indirect (e.g. icosahedral) hierarchy from the reference's grid tables and hatted
        coefficients (tpmg_hier_create_generic); lists are per level, coarsest first."""
        self = cls.__new__(cls)
        self.ctx, self.lib = ctx, ctx.lib
        self._h = None
        nl = len(ncells)
        I64P = C.POINTER(C.c_int64)
        keep = []

        def i64(a):
            a = np.ascontiguousarray(a, dtype=np.int64)
            keep.append(a)
            return a.ctypes.data_as(I64P)

        def f64(a):
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            return a.ctypes.data_as(C.POINTER(C.c_double))

        D = C.POINTER(C.c_double)
        h = C.c_void_p()
        ctx._check(self.lib.tpmg_hier_create_generic(
            ctx._h, nl, int(nz), int(nnb), int(nchild), i64(ncells), i64(nedges),
            (I64P * nl)(*[i64(a) for a in nbr]), (I64P * nl)(*[i64(a) for a in cedge]),
            (I64P * nl)(*[i64(a) if a is not None else None for a in children]),
            (C.c_int * nchild)(*prol_d1), (C.c_int * nchild)(*prol_d2), f64(bv), f64(sv), f64(av),
            f64(xv), (D * nl)(*[f64(a) for a in bh]), (D * nl)(*[f64(a) for a in ah]),
            (D * nl)(*[f64(a) for a in xh]), (D * nl)(*[f64(a) for a in sh]), C.c_double(relax),
            int(prolongation), int(restriction), int(nu_pre), int(nu_post), C.byref(h)))
        self._h = h
        ctx._live_children += 1
        self.problem = None
        n = C.c_int()
        self.lib.tpmg_hier_n_levels(self._h, C.byref(n))
        self.n_levels = n.value
        self.finest = self.n_levels - 1
        return self

    def level_shape(self, level: int):
        v = [C.c_int64() for _ in range(5)]
        self.ctx._check(self.lib.tpmg_hier_level_shape(self._h, level, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)  # nx, ny, nz, x0, y0

    def field(self, level: int | None = None) -> Field:
        return Field(self, self.finest if level is None else level)

    def coefficients(self, level: int) -> dict:
        nx, ny, nz = self.level_shape(level)[:3]
        nc = nx * ny
        out = dict(bh=np.empty(nc), ah=np.empty(nc), xh=np.empty(nc), sh=np.empty(2 * nc),
                   bv=np.empty(nz), sv=np.empty(nz), av=np.empty(nz + 1), xv=np.empty(nz + 1))
        self.ctx._check(self.lib.tpmg_hier_get_coefficients(
            self._h, level, *[_p(out[k]) for k in ("bh", "ah", "xh", "sh", "bv", "sv", "av", "xv")]))
        return out

    def time_kernel(self, kernel_id: int, level: int | None = None, reps: int = 20) -> float:
        """Average device milliseconds per launch (tpmg_time_kernel)."""
        out = C.c_double()
        self.ctx._check(self.lib.tpmg_time_kernel(self._h, kernel_id,
                                                  self.finest if level is None else level, reps,
                                                  C.byref(out)))
        return out.value

    def kernel_probe(self, on: bool = True):
        """Live per-launch durations of the finest-level PCG kernels inside later pcg_solve
        calls (CUDA events in the iteration graph); enabling resets the totals."""
        self.ctx._check(self.lib.tpmg_kernel_probe(self._h, 1 if on else 0))

    def kernel_probe_read(self, kernel_id: int):
        """(total ms, launches) of one kernel id since kernel_probe(True)."""
        ms, n = C.c_double(), C.c_int64()
        self.ctx._check(self.lib.tpmg_kernel_probe_read(self._h, kernel_id, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def set_use_graphs(self, on: bool):
        self.lib.tpmg_set_use_graphs(self._h, 1 if on else 0)

    _live_children = 0
    _pending_close = False

    def _child_closed(self):
        self._live_children -= 1
        if self._pending_close and self._live_children == 0:
            self.close()

    def close(self):
        if self._live_children > 0:  # fields still alive: the last one closes this
            self._pending_close = True
            return
        if getattr(self, "_h", None) is not None:
            self.lib.tpmg_hier_destroy(self._h)
            self._h = None
            self.ctx._child_closed()

    def __del__(self):
        # at interpreter shutdown the destruction order of handles is arbitrary: leave the
        # device memory to the driver instead of freeing through possibly-dead parents
        if sys.is_finalizing():
            return
        try:
            self.close()
        except Exception:
            pass


# ---- reference-shaped free functions ----------------------------------------------------------

def build_hierarchy_coefficients(ctx: Context, problem, **over) -> Hierarchy:
    return Hierarchy(ctx, problem, **over)


def apply_operator(h: Hierarchy, u: Field, out: Field) -> Field:
    h.ctx._check(h.lib.tpmg_apply(h._h, u._h, out._h))
    return out


def residual(h: Hierarchy, f: Field, u: Field, r: Field) -> Field:
    h.ctx._check(h.lib.tpmg_residual(h._h, f._h, u._h, r._h))
    return r


def smooth(h: Hierarchy, u: Field, f: Field, sweeps: int) -> Field:
    h.ctx._check(h.lib.tpmg_smooth(h._h, u._h, f._h, sweeps))
    return u


def restrict_field(h: Hierarchy, fine: Field, coarse: Field) -> Field:
    h.ctx._check(h.lib.tpmg_restrict(h._h, fine._h, coarse._h))
    return coarse


def prolongate_field(h: Hierarchy, coarse: Field, fine: Field, add: bool = False) -> Field:
    fn = h.lib.tpmg_prolong_add if add else h.lib.tpmg_prolong
    h.ctx._check(fn(h._h, coarse._h, fine._h))
    return fine


def v_cycle(h: Hierarchy, f: Field, u: Field) -> Field:
    h.ctx._check(h.lib.tpmg_vcycle(h._h, f._h, u._h))
    return u


def measure_cycle_rate(h: Hierarchy, f: Field, n_cycles: int) -> float:
    out = C.c_double()
    h.ctx._check(h.lib.tpmg_measure_cycle_rate(h._h, f._h, n_cycles, C.byref(out)))
    return out.value


def dot(h: Hierarchy, a: Field, b: Field) -> float:
    out = C.c_double()
    h.ctx._check(h.lib.tpmg_dot(h._h, a._h, b._h, C.byref(out)))
    return out.value


class SolveResult:
    def __init__(self, iters, status, history, seconds):
        self.iterations, self.status, self.history, self.seconds = iters, status, history, seconds

    @property
    def converged(self) -> bool:
        return self.status == OK

    def __repr__(self):
        return (f"SolveResult(iterations={self.iterations}, status={self.status}, "
                f"rel_res={self.history[-1] / self.history[0] if len(self.history) else None})")


def pcg_solve(h: Hierarchy, f: Field, x: Field, tol: float, max_iter: int = 500) -> SolveResult:
    hist = np.zeros(max_iter + 1)
    it, st = C.c_int(), C.c_int()
    t0 = time.perf_counter()
    h.ctx._check(h.lib.tpmg_pcg(h._h, f._h, x._h, C.c_double(tol), max_iter, _p(hist),
                                C.byref(it), C.byref(st)))
    return SolveResult(it.value, st.value, hist[: it.value + 1].copy(), time.perf_counter() - t0)


def _outer_solve(fn, h: Hierarchy, f: Field, x: Field, tol: float, max_iter: int, mu: int):
    hist = np.zeros(max_iter + 1)
    it, st = C.c_int(), C.c_int()
    t0 = time.perf_counter()
    h.ctx._check(fn(h._h, f._h, x._h, C.c_double(tol), max_iter, mu, _p(hist), C.byref(it),
                    C.byref(st)))
    return SolveResult(it.value, st.value, hist[: it.value + 1].copy(), time.perf_counter() - t0)


def richardson_solve(h: Hierarchy, f: Field, x: Field, tol: float = 1e-5, max_iter: int = 500,
                     mu: int = 1) -> SolveResult:
    """Preconditioned Richardson, mu V-cycles per step (richardson_solve)."""
    return _outer_solve(h.lib.tpmg_richardson, h, f, x, tol, max_iter, mu)


def bicgstab_solve(h: Hierarchy, f: Field, x: Field, tol: float = 1e-5, max_iter: int = 500,
                   mu: int = 1) -> SolveResult:
    """Right-preconditioned BiCGStab (bicgstab_solve)."""
    return _outer_solve(h.lib.tpmg_bicgstab, h, f, x, tol, max_iter, mu)


def solver_counts(h: Hierarchy):
    """(preconditioner applications, operator applications) of the last outer solve."""
    a, b = C.c_int64(), C.c_int64()
    h.ctx._check(h.lib.tpmg_solver_counts(h._h, C.byref(a), C.byref(b)))
    return a.value, b.value


def pcg_solve_host(h: Hierarchy, f_host: np.ndarray, tol: float, max_iter: int = 500,
                   layout: int = X_FASTEST):
    """End-to-end: host f -> device -> PCG -> host x (tpmg_pcg_host)."""
    f_host = np.ascontiguousarray(f_host, dtype=np.float64).reshape(-1)
    x = np.empty_like(f_host)
    hist = np.zeros(max_iter + 1)
    it, st = C.c_int(), C.c_int()
    h.ctx._check(h.lib.tpmg_pcg_host(h._h, _p(f_host), _p(x), layout, C.c_double(tol), max_iter,
                                     _p(hist), C.byref(it), C.byref(st)))
    return x, SolveResult(it.value, st.value, hist[: it.value + 1].copy(), 0.0)


def pcg_solve_host_batch(h: Hierarchy, f_hosts, x_hosts, tol: float, max_iter: int = 500,
                         layout: int = X_FASTEST):
    """End-to-end solves of several right-hand sides with the transfers overlapped
    (tpmg_pcg_host_batch): f_hosts[i] -> x_hosts[i] (contiguous float64 arrays, pinned for the
    copies to overlap).  Returns one SolveResult per right-hand side."""
    count = len(f_hosts)
    if len(x_hosts) != count:
        raise ValueError("f_hosts and x_hosts differ in length")
    for a in list(f_hosts) + list(x_hosts):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise ValueError("host buffers must be contiguous float64")
    fp = (_capi._D * count)(*[_p(a) for a in f_hosts])
    xp = (_capi._D * count)(*[_p(a) for a in x_hosts])
    hist = np.zeros((count, max_iter + 1))
    it = (C.c_int * count)()
    st = (C.c_int * count)()
    h.ctx._check(h.lib.tpmg_pcg_host_batch(h._h, count, fp, xp, layout, C.c_double(tol), max_iter,
                                           _p(hist), it, st))
    return [SolveResult(it[i], st[i], hist[i, : it[i] + 1].copy(), 0.0) for i in range(count)]


# ---- profile files: save_profiles / load_profiles (profile_io.hpp:125-242) ----------------------

PROFILE_FACTORIZED, PROFILE_FULL = 0, 2
PROFILE_ORDER = {
    PROFILE_FACTORIZED: ("beta_r", "alpha_s_r", "alpha_r_r", "xi_r_r", "beta_s", "alpha_r_s",
                         "xi_r_s", "alpha_s_s"),
    PROFILE_FULL: ("beta", "alpha_s", "alpha_r", "xi_r"),
}


def _profile_shapes(kind: int, nc: int, ne: int, nr: int):
    """Array shapes in the reference's Matrix order: dense arrays (cols, rows), k fastest."""
    if kind == PROFILE_FACTORIZED:
        return ((nr,), (nr,), (nr + 1,), (nr + 1,), (nc,), (nc,), (nc,), (ne,))
    return ((nc, nr), (ne, nr), (nc, nr + 1), (nc, nr + 1))


def _profile_call(rc: int):
    if rc != OK:
        msg = _capi.load().tpmg_profile_last_error().decode()
        raise _ERRORS.get(rc, TpmgError)(msg)


def grid_fingerprint(centers: np.ndarray) -> int:
    """grid_fingerprint (geometry.hpp:335-351) of centres given as (n_cells, 3)."""
    c = np.ascontiguousarray(centers, dtype=np.float64)
    return int(_capi.load().tpmg_grid_fingerprint(_p(c), c.shape[0]))


def profile_grid(type: str, fingerprint: int, level: int, n_r: int, n_cells: int, n_edges: int,
                 nx: int = 0, ny: int = 0) -> _capi.ProfileGrid:
    return _capi.ProfileGrid(type.encode(), fingerprint, level, n_r, n_cells, n_edges, nx, ny)


def _packed(kind: int, grid, arrays: dict) -> np.ndarray:
    shapes = _profile_shapes(kind, grid.n_cells, grid.n_edges, grid.n_r)
    parts = []
    for name, shape in zip(PROFILE_ORDER[kind], shapes):
        a = np.asarray(arrays[name], dtype=np.float64)
        if a.shape != shape:
            raise shape_error(f"profile array {name!r} has shape {a.shape}, expected {shape}")
        parts.append(a.ravel())
    return np.ascontiguousarray(np.concatenate(parts))


def _unpack(kind: int, grid, buf: np.ndarray) -> dict:
    out, off = {}, 0
    for name, shape in zip(PROFILE_ORDER[kind], _profile_shapes(kind, grid.n_cells, grid.n_edges,
                                                                grid.n_r)):
        n = int(np.prod(shape))
        out[name] = buf[off:off + n].reshape(shape).copy()
        off += n
    return out


def save_profile_arrays(path: str, grid, kind: int, arrays: dict,
                        encoding: str = "decimal") -> None:
    """save_profiles on any grid header (tpmg_profile_save_grid)."""
    if encoding not in ("decimal", "base64-f64le"):
        raise config_error(f"unknown encoding {encoding!r}")
    packed = _packed(kind, grid, arrays)
    _profile_call(_capi.load().tpmg_profile_save_grid(path.encode(), C.byref(grid), kind,
                                                      _p(packed),
                                                      int(encoding == "base64-f64le")))


def load_profile_arrays(path: str, grid):
    """load_profiles on any grid header: returns (kind, {name: array})."""
    L = _capi.load()
    cap = max(L.tpmg_profile_packed_size(k, grid.n_cells, grid.n_edges, grid.n_r)
              for k in PROFILE_ORDER)
    buf = np.empty(cap, dtype=np.float64)
    kind = C.c_int()
    _profile_call(L.tpmg_profile_load_grid(path.encode(), C.byref(grid), C.byref(kind), _p(buf),
                                           cap))
    return kind.value, _unpack(kind.value, grid, buf)


def cartesian_profile_grid(P) -> _capi.ProfileGrid:
    z = np.ascontiguousarray(P.z_faces, dtype=np.float64)
    gd = GridDesc(P.nx, P.ny, P.hx, P.hy, P.nz, _p(z))
    fp = int(_capi.load().tpmg_grid_fingerprint_cartesian(C.byref(gd)))
    nc = P.nx * P.ny
    return profile_grid("cartesian", fp, 0, P.nz, nc, 2 * nc, P.nx, P.ny)


def save_profiles(path: str, P, encoding: str = "decimal") -> None:
    """save_profiles (profile_io.hpp:125-165) of P's profile set on P's Cartesian grid: its
    factorised profiles, or its dense ProfileSet when P.coef == "full".  encoding "decimal" or
    "base64-f64le".  A None advection profile is written as zeros (the reference always stores
    xi_r)."""
    nc, nz = P.nx * P.ny, P.nz
    if P.coef == "full":
        d = dict(P.dense)
        if d.get("xi_r") is None:
            d["xi_r"] = np.zeros((nc, nz + 1))
        kind, arrays = PROFILE_FULL, d
    elif P.coef == "factorized":
        arrays = {n: getattr(P, n) for n in PROFILE_ORDER[PROFILE_FACTORIZED]}
        if arrays["xi_r_r"] is None or arrays["xi_r_s"] is None:
            arrays["xi_r_r"], arrays["xi_r_s"] = np.zeros(nz + 1), np.zeros(nc)
        kind = PROFILE_FACTORIZED
    else:
        raise config_error("the profile format stores factorised or full profile sets")
    save_profile_arrays(path, cartesian_profile_grid(P), kind, arrays, encoding)


def load_profiles(path: str, P):
    """load_profiles (profile_io.hpp:168-242): read a profile file written for P's grid and return
    a copy of P with those profiles (coef "factorized" or "full").  Raises fingerprint_error for
    another grid, shape_error for wrong sizes or a malformed file, nonfinite_error for NaN/Inf/null,
    config_error for an unreadable file.  All-zero advection arrays come back as None (xi = 0)."""
    import dataclasses
    kind, arrays = load_profile_arrays(path, cartesian_profile_grid(P))
    Q = dataclasses.replace(P)
    if kind == PROFILE_FACTORIZED:
        if not arrays["xi_r_r"].any() or not arrays["xi_r_s"].any():
            arrays["xi_r_r"] = arrays["xi_r_s"] = None
        for k, v in arrays.items():
            setattr(Q, k, v)
        Q.coef, Q.dense = "factorized", None
    else:
        if not arrays["xi_r"].any():
            arrays["xi_r"] = None
        Q.coef, Q.dense = "full", arrays
    return Q
