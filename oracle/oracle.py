"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of the CPU oracle (oracle/liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.  Arrays
use the reference's Field order (k fastest per column, discretization.hpp:106-120)
unless a function says otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_D = C.POINTER(C.c_double)
_I64 = C.c_int64


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "tpmg_oracle.cpp")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.tpmgo_last_error.restype = C.c_char_p
        L.tpmgo_n_cells.restype = C.c_int64
        L.tpmgo_nz.restype = C.c_int64
        L.tpmgo_dot.restype = C.c_double
        L.tpmgo_dot.argtypes = [C.c_int64, _D, _D]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(_D)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _chk(rc):
    if rc != 0:
        raise OracleError(rc, lib().tpmgo_last_error().decode())


class OracleHierarchy:
    """CPU restatement of MultigridHierarchy + its hot-path operations."""

    def __init__(self, handle, nz):
        self._h = handle
        self.nz = nz

    @classmethod
    def from_problem(cls, P, threads: int = 1, **over):
        kw = P.mg_kwargs()
        kw.update(over)
        h = C.c_void_p()
        f = lambda a: _p(np.ascontiguousarray(a, dtype=np.float64))
        keep = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (P.z_faces, P.beta_r, P.alpha_s_r, P.alpha_r_r, P.beta_s, P.alpha_r_s, P.alpha_s_s)]
        xr = xs = None
        if getattr(P, "xi_r_r", None) is not None:
            xr = np.ascontiguousarray(P.xi_r_r, dtype=np.float64)
            xs = np.ascontiguousarray(P.xi_r_s, dtype=np.float64)
        args = (_I64(P.nx), _I64(P.ny), C.c_double(P.hx), C.c_double(P.hy), _I64(P.nz),
                _p(keep[0]), _p(keep[1]), _p(keep[2]), _p(keep[3]), _p(xr), _p(keep[4]),
                _p(keep[5]), _p(xs), _p(keep[6]), C.c_double(P.omega), C.c_double(kw["relax"]),
                C.c_int(kw["prolongation"]), C.c_int(kw["restriction"]), C.c_int(kw["nu_pre"]),
                C.c_int(kw["nu_post"]), C.c_int(kw["depth"]), C.c_int(threads), C.byref(h))
        coef = getattr(P, "coef", "factorized")
        if coef == "factorized":
            rc = lib().tpmgo_cart_create(*args)
        else:
            d = {k: (None if v is None else np.ascontiguousarray(v, dtype=np.float64))
                 for k, v in P.dense.items()}
            keep += [v for v in d.values() if v is not None]
            mode = 1 if coef == "partial" else 2
            rc = lib().tpmgo_cart_create_dense(
                C.c_int(mode), _p(d["beta"]), _p(d["alpha_s"]), _p(d["alpha_r"]), _p(d["xi_r"]),
                *args)
        _chk(rc)
        # mirror the device's smoother switch (jacobi_uses_t4, tpmg_kernels.cu)
        lib().tpmgo_set_t4(h, 0 if os.environ.get("TPMG_JACOBI_T4", "0") == "0" else 1)
        return cls(h, P.nz)

    @classmethod
    def from_tables(cls, nz, nnb, nchild, ncells, nedges, nbr, cedge, children, prol_d1, prol_d2,
                    bv, sv, av, xv, bh, ah, xh, sh, relax, prolongation, restriction, nu_pre,
                    nu_post, threads=1):
        """Generic tables (tpmgo_generic_create), e.g. the reference's icosahedral hierarchy."""
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
            return a.ctypes.data_as(_D)

        nbr_p = (I64P * nl)(*[i64(a) for a in nbr])
        ced_p = (I64P * nl)(*[i64(a) for a in cedge])
        ch_p = (I64P * nl)(*[i64(a) if a is not None else None for a in children])
        bh_p = (_D * nl)(*[f64(a) for a in bh])
        ah_p = (_D * nl)(*[f64(a) for a in ah])
        xh_p = (_D * nl)(*[f64(a) for a in xh])
        sh_p = (_D * nl)(*[f64(a) for a in sh])
        d1 = (C.c_int * nchild)(*prol_d1)
        d2 = (C.c_int * nchild)(*prol_d2)
        h = C.c_void_p()
        rc = lib().tpmgo_generic_create(
            C.c_int(nl), _I64(nz), C.c_int(nnb), C.c_int(nchild), i64(ncells), i64(nedges),
            nbr_p, ced_p, ch_p, d1, d2, f64(bv), f64(sv), f64(av), f64(xv), bh_p, ah_p, xh_p,
            sh_p, C.c_double(relax), C.c_int(prolongation), C.c_int(restriction),
            C.c_int(nu_pre), C.c_int(nu_post), C.c_int(threads), C.byref(h))
        _chk(rc)
        return cls(h, nz)

    def __del__(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.tpmgo_destroy(self._h)
            self._h = None

    @property
    def n_levels(self) -> int:
        return lib().tpmgo_n_levels(self._h)

    @property
    def finest(self) -> int:
        return self.n_levels - 1

    def n_cells(self, level: int) -> int:
        return lib().tpmgo_n_cells(self._h, level)

    def size(self, level: int) -> int:
        return self.n_cells(level) * self.nz

    def set_threads(self, t: int):
        lib().tpmgo_set_threads(self._h, t)

    def set_device_order(self, on: bool):
        """False: fastest CPU schedule for the PCG vector work (baseline timing only)."""
        lib().tpmgo_set_device_order(self._h, 1 if on else 0)

    def coefficients(self, level: int) -> dict:
        nc, nz = self.n_cells(level), self.nz
        out = dict(bh=np.empty(nc), ah=np.empty(nc), xh=np.empty(nc), sh=np.empty(2 * nc),
                   bv=np.empty(nz), sv=np.empty(nz), av=np.empty(nz + 1), xv=np.empty(nz + 1))
        _chk(lib().tpmgo_get_coefficients(self._h, level, *[_p(out[k]) for k in
                                                             ("bh", "ah", "xh", "sh", "bv", "sv", "av", "xv")]))
        return out

    def build_column(self, level: int, cell: int):
        nz = self.nz
        d, u, l, nb = np.empty(nz), np.empty(nz), np.empty(nz), np.empty(4 * nz)
        _chk(lib().tpmgo_build_column(self._h, level, _I64(cell), _p(d), _p(u), _p(l), _p(nb)))
        return d, u, l, nb.reshape(4, nz)

    def apply(self, level: int, u: np.ndarray) -> np.ndarray:
        y = np.empty(self.size(level))
        _chk(lib().tpmgo_apply(self._h, level, _p(u), _p(y)))
        return y

    def residual(self, level: int, f: np.ndarray, u: np.ndarray) -> np.ndarray:
        r = np.empty(self.size(level))
        _chk(lib().tpmgo_residual(self._h, level, _p(f), _p(u), _p(r)))
        return r

    def smooth(self, level: int, u: np.ndarray, f: np.ndarray, sweeps: int) -> np.ndarray:
        u = np.array(u, dtype=np.float64, copy=True)
        _chk(lib().tpmgo_smooth(self._h, level, _p(u), _p(f), sweeps))
        return u

    def restrict(self, coarse_level: int, fine: np.ndarray) -> np.ndarray:
        c = np.empty(self.size(coarse_level))
        _chk(lib().tpmgo_restrict(self._h, coarse_level, _p(fine), _p(c)))
        return c

    def prolong(self, coarse_level: int, coarse: np.ndarray) -> np.ndarray:
        f = np.empty(self.size(coarse_level + 1))
        _chk(lib().tpmgo_prolong(self._h, coarse_level, _p(coarse), _p(f)))
        return f

    def vcycle(self, f: np.ndarray, u: np.ndarray | None = None, level: int | None = None):
        level = self.finest if level is None else level
        u = np.zeros(self.size(level)) if u is None else np.array(u, dtype=np.float64, copy=True)
        _chk(lib().tpmgo_vcycle(self._h, level, _p(f), _p(u)))
        return u

    def measure_cycle_rate(self, f: np.ndarray, n_cycles: int) -> float:
        r = C.c_double()
        _chk(lib().tpmgo_measure_cycle_rate(self._h, _p(f), n_cycles, C.byref(r)))
        return r.value

    def pcg(self, f: np.ndarray, tol: float, max_iter: int = 200, seconds: bool = False):
        x = np.empty(self.size(self.finest))
        hist = np.zeros(max_iter + 1)
        secs = np.zeros(max_iter + 1)
        it, st = C.c_int(), C.c_int()
        _chk(lib().tpmgo_pcg_timed(self._h, _p(f), _p(x), C.c_double(tol), max_iter, _p(hist),
                                   _p(secs), C.byref(it), C.byref(st)))
        out = (x, hist[: it.value + 1].copy(), it.value, st.value)
        return out + (secs[: it.value + 1].copy(),) if seconds else out


def _outer(fn, o, f, tol, max_iter, mu):
    x = np.empty(o.size(o.finest))
    hist = np.zeros(max_iter + 1)
    it, st = C.c_int(), C.c_int()
    _chk(fn(o._h, _p(np.ascontiguousarray(f, dtype=np.float64)), _p(x), C.c_double(tol), max_iter,
            mu, _p(hist), C.byref(it), C.byref(st)))
    return x, hist[: it.value + 1].copy(), it.value, st.value


def richardson(o: "OracleHierarchy", f, tol=1e-5, max_iter=200, mu=1):
    return _outer(lib().tpmgo_richardson, o, f, tol, max_iter, mu)


def bicgstab(o: "OracleHierarchy", f, tol=1e-5, max_iter=200, mu=1):
    return _outer(lib().tpmgo_bicgstab, o, f, tol, max_iter, mu)


def thomas(diag, upper, lower, rhs):
    x = np.array(rhs, dtype=np.float64, copy=True)
    _chk(lib().tpmgo_thomas(_I64(len(x)), _p(np.ascontiguousarray(diag, dtype=np.float64)),
                            _p(np.ascontiguousarray(upper, dtype=np.float64)),
                            _p(np.ascontiguousarray(lower, dtype=np.float64)), _p(x)))
    return x


def dot(a, b) -> float:
    return lib().tpmgo_dot(len(a), _p(a), _p(b))
