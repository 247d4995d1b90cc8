"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of oracle/libicosa_setup.so, the reference's own
icosahedral test problem set up on the host in the reference's operation order
(build_icosahedral_hierarchy + build_vertical_grid + balanced-flow profiles + courant_default +
the hatted coefficients of every level: geometry.hpp:263-327, profiles.hpp:128-391,
multigrid.hpp:263-268; mirrors the reference's fixture tests/fixtures.hpp:18-62).

Only tests/ import this.  The device hierarchy of the problem is built by the PRODUCT through
its C-ABI boundary for indirect grids (tpmg_hier_create_generic via tpmg.Hierarchy.from_tables),
fed with these tables exactly as a caller holding the reference's GridHierarchy would.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libicosa_setup.so")
_D = C.POINTER(C.c_double)
_VP = C.c_void_p
_lib = None

PROFILE_FACTORIZED, PROFILE_FULL = 0, 2
_ERR_NAMES = {1: "config_error", 6: "cap_error"}


class IcosaParams(C.Structure):  # tpmgo_icosa_params
    _fields_ = [("levels", C.c_int), ("n_r", C.c_int64), ("depth", C.c_double),
                ("geometric", C.c_int), ("ratio", C.c_double), ("buoyancy_frequency", C.c_double),
                ("courant", C.c_double), ("advection", C.c_int)]


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "icosa_setup.cpp")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "libicosa_setup.so"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        I64P = C.POINTER(C.c_int64)
        L.tpmgo_icosa_last_error.restype = C.c_char_p
        L.tpmgo_icosa_create.argtypes = [C.c_void_p, C.POINTER(_VP)]
        L.tpmgo_icosa_destroy.argtypes = [_VP]
        L.tpmgo_icosa_info.argtypes = [_VP, C.POINTER(C.c_int), _D, _D, _D]
        L.tpmgo_icosa_level.argtypes = [_VP, C.c_int, I64P, I64P, C.POINTER(I64P),
                                        C.POINTER(I64P), C.POINTER(_D), C.POINTER(_D)]
        L.tpmgo_icosa_hatted.argtypes = [_VP, C.c_int] + [C.POINTER(_D)] * 8
        L.tpmgo_icosa_profiles.argtypes = [_VP, C.c_int, _D, C.c_int64]
        _lib = L
    return _lib


class IcosaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


def _chk(rc):
    if rc != 0:
        raise IcosaError(rc, lib().tpmgo_icosa_last_error().decode())


class Icosahedral:
    """The reference's icosahedral problem: grids, radial grid, balanced-flow profiles and the
    hatted coefficients of every level, bit for bit the reference's."""

    def __init__(self, levels: int, n_r: int, depth: float, grading: str = "uniform",
                 ratio: float = 1.0, buoyancy_frequency: float = 0.022, courant: float = 10.0,
                 advection: bool = True):
        prm = IcosaParams(levels, n_r, depth, int(grading == "geometric"), ratio,
                          buoyancy_frequency, courant, int(advection))
        h = _VP()
        _chk(lib().tpmgo_icosa_create(C.byref(prm), C.byref(h)))
        self._h = h
        n, om, mu, eps = C.c_int(), C.c_double(), C.c_double(), C.c_double()
        lib().tpmgo_icosa_info(self._h, C.byref(n), C.byref(om), C.byref(mu), C.byref(eps))
        self.n_levels, self.omega, self.mu_dt, self.epsilon = n.value, om.value, mu.value, eps.value
        self.n_r = n_r

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tpmgo_icosa_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def level(self, level: int) -> dict:
        from paper_1408_2981_b200 import tpmg

        nc, ne = C.c_int64(), C.c_int64()
        I64P = C.POINTER(C.c_int64)
        nb, ce = I64P(), I64P()
        cen, ar = _D(), _D()
        _chk(lib().tpmgo_icosa_level(self._h, level, C.byref(nc), C.byref(ne), C.byref(nb),
                                     C.byref(ce), C.byref(cen), C.byref(ar)))
        n, m = nc.value, ne.value
        centers = np.ctypeslib.as_array(cen, (n * 3,)).copy().reshape(n, 3)
        return dict(n_cells=n, n_edges=m,
                    neighbors=np.ctypeslib.as_array(nb, (n * 3,)).copy().reshape(n, 3),
                    cell_edges=np.ctypeslib.as_array(ce, (n * 3,)).copy().reshape(n, 3),
                    centers=centers, areas=np.ctypeslib.as_array(ar, (n,)).copy(),
                    fingerprint=tpmg.grid_fingerprint(centers))

    def hatted(self, level: int) -> dict:
        P = [_D() for _ in range(8)]
        _chk(lib().tpmgo_icosa_hatted(self._h, level, *[C.byref(p) for p in P]))
        lv = self.level(level)
        nc, ne, nr = lv["n_cells"], lv["n_edges"], self.n_r
        sizes = (nc, nc, nc, ne, nr, nr, nr + 1, nr + 1)
        names = ("bh", "ah", "xh", "sh", "bv", "sv", "av", "xv")
        return {k: np.ctypeslib.as_array(p, (n,)).copy() for k, p, n in zip(names, P, sizes)}

    def profile_grid(self):
        from paper_1408_2981_b200 import tpmg

        lv = self.level(self.n_levels - 1)
        return tpmg.profile_grid("icosahedral", lv["fingerprint"], self.n_levels - 1, self.n_r,
                                 lv["n_cells"], lv["n_edges"])

    def profiles(self, kind: int) -> dict:
        """The finest level's profile set (PROFILE_FACTORIZED or PROFILE_FULL), reference shapes."""
        from paper_1408_2981_b200 import _capi, tpmg

        g = self.profile_grid()
        cap = _capi.load().tpmg_profile_packed_size(kind, g.n_cells, g.n_edges, g.n_r)
        buf = np.empty(cap)
        _chk(lib().tpmgo_icosa_profiles(self._h, kind, buf.ctypes.data_as(_D), cap))
        return tpmg._unpack(kind, g, buf)

    def hierarchy(self, ctx, depth: int = 0, relax: float = 0.9, prolongation: int = 0,
                  restriction: int = 0, nu_pre: int = 2, nu_post: int = 2):
        """The device hierarchy of levels L+1-depth .. L (depth <= 0: all), built by the product
        from these tables (tpmg_hier_create_generic): the reference's child order
        (GridHierarchy::child_of(Tc, j) = 4 Tc + j, geometry.hpp:89-90) and linear-prolongation
        corner rule (multigrid.hpp:88-95: corner child j takes the coarse neighbours across edges
        (j+1)%3 and (j+2)%3, the centre child none)."""
        from paper_1408_2981_b200 import tpmg

        finest = self.n_levels - 1
        if depth <= 0 or depth > finest + 1:
            depth = finest + 1  # multigrid.hpp:259-260
        coarsest = finest + 1 - depth
        lv = [self.level(l) for l in range(coarsest, finest + 1)]
        hat = [self.hatted(l) for l in range(coarsest, finest + 1)]
        children = [None] + [np.arange(4 * lv[i - 1]["n_cells"], dtype=np.int64)
                             for i in range(1, depth)]
        hf = hat[-1]
        return tpmg.Hierarchy.from_tables(
            ctx, self.n_r, 3, 4, [x["n_cells"] for x in lv], [x["n_edges"] for x in lv],
            [x["neighbors"].reshape(-1) for x in lv], [x["cell_edges"].reshape(-1) for x in lv],
            children, [1, 2, 0, -1], [2, 0, 1, -1], hf["bv"], hf["sv"], hf["av"], hf["xv"],
            [x["bh"] for x in hat], [x["ah"] for x in hat], [x["xh"] for x in hat],
            [x["sh"] for x in hat], relax, prolongation, restriction, nu_pre, nu_post)
