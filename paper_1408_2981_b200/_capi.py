"""ctypes binding of the C-ABI library ``libtpmg_b200.so`` (declared in include/tpmg_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``python -m
paper_1408_2981_b200.build``).  Loading fails loudly when it is missing: there is no
Python or CPU fallback for the hot path.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_NAMES = {"exact": "libtpmg_b200.so", "fma": "libtpmg_b200_fma.so"}

_D = C.POINTER(C.c_double)
_VP = C.c_void_p

# symbol -> (restype, argtypes); mirrors include/tpmg_b200.h exactly.
SIGNATURES = {
    "tpmg_status_string": (C.c_char_p, [C.c_int]),
    "tpmg_abi_version": (C.c_int, []),
    "tpmg_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "tpmg_init": (C.c_int, [C.c_void_p, C.POINTER(_VP)]),
    "tpmg_init_ipc": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(_VP)]),
    "tpmg_finalize": (C.c_int, [_VP]),
    "tpmg_last_error": (C.c_char_p, [_VP]),
    "tpmg_context_stream": (C.c_int, [_VP, C.POINTER(C.c_void_p)]),
    "tpmg_plan_decomposition": (C.c_int, [C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_int, C.POINTER(C.c_int)] + [C.POINTER(C.c_int64)] * 4
                                + [C.POINTER(C.c_int)]),
    "tpmg_hier_create": (C.c_int, [_VP, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.POINTER(_VP)]),
    "tpmg_hier_destroy": (C.c_int, [_VP]),
    "tpmg_hier_n_levels": (C.c_int, [_VP, C.POINTER(C.c_int)]),
    "tpmg_hier_level_shape": (C.c_int, [_VP, C.c_int] + [C.POINTER(C.c_int64)] * 5),
    "tpmg_hier_get_coefficients": (C.c_int, [_VP, C.c_int] + [_D] * 8),
    "tpmg_field_create": (C.c_int, [_VP, C.c_int, C.POINTER(_VP)]),
    "tpmg_field_destroy": (C.c_int, [_VP]),
    "tpmg_field_level": (C.c_int, [_VP, C.POINTER(C.c_int)]),
    "tpmg_field_upload": (C.c_int, [_VP, _D, C.c_int]),
    "tpmg_field_download": (C.c_int, [_VP, _D, C.c_int]),
    "tpmg_field_fill": (C.c_int, [_VP, C.c_double]),
    "tpmg_field_copy": (C.c_int, [_VP, _VP]),
    "tpmg_field_device_ptr": (C.c_int, [_VP, C.POINTER(_D)]),
    "tpmg_apply": (C.c_int, [_VP, _VP, _VP]),
    "tpmg_residual": (C.c_int, [_VP, _VP, _VP, _VP]),
    "tpmg_smooth": (C.c_int, [_VP, _VP, _VP, C.c_int]),
    "tpmg_restrict": (C.c_int, [_VP, _VP, _VP]),
    "tpmg_prolong_add": (C.c_int, [_VP, _VP, _VP]),
    "tpmg_prolong": (C.c_int, [_VP, _VP, _VP]),
    "tpmg_restrict_kind": (C.c_int, [_VP, _VP, _VP, C.c_int]),
    "tpmg_prolong_kind": (C.c_int, [_VP, _VP, _VP, C.c_int, C.c_int]),
    "tpmg_vcycle": (C.c_int, [_VP, _VP, _VP]),
    "tpmg_measure_cycle_rate": (C.c_int, [_VP, _VP, C.c_int, _D]),
    "tpmg_dot": (C.c_int, [_VP, _VP, _VP, _D]),
    "tpmg_norm": (C.c_int, [_VP, _VP, _D]),
    "tpmg_pcg": (C.c_int, [_VP, _VP, _VP, C.c_double, C.c_int, _D, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "tpmg_richardson": (C.c_int, [_VP, _VP, _VP, C.c_double, C.c_int, C.c_int, _D, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int)]),
    "tpmg_bicgstab": (C.c_int, [_VP, _VP, _VP, C.c_double, C.c_int, C.c_int, _D, C.POINTER(C.c_int),
                                C.POINTER(C.c_int)]),
    "tpmg_solver_counts": (C.c_int, [_VP, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tpmg_hier_create_partial": (C.c_int, [_VP, C.c_void_p, C.c_void_p, _D, C.c_double, C.c_void_p,
                                           C.POINTER(_VP)]),
    "tpmg_hier_create_full": (C.c_int, [_VP, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                        C.POINTER(_VP)]),
    "tpmg_hier_coef_mode": (C.c_int, [_VP, C.POINTER(C.c_int)]),
    "tpmg_hier_create_generic": (C.c_int, [_VP, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                           C.POINTER(C.POINTER(C.c_int64)),
                                           C.POINTER(C.POINTER(C.c_int64)),
                                           C.POINTER(C.POINTER(C.c_int64)),
                                           C.POINTER(C.c_int), C.POINTER(C.c_int), _D, _D, _D, _D,
                                           C.POINTER(_D), C.POINTER(_D), C.POINTER(_D),
                                           C.POINTER(_D), C.c_double, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.POINTER(_VP)]),
    "tpmg_pcg_host": (C.c_int, [_VP, _D, _D, C.c_int, C.c_double, C.c_int, _D, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "tpmg_pcg_host_batch": (C.c_int, [_VP, C.c_int, C.POINTER(_D), C.POINTER(_D), C.c_int, C.c_double, C.c_int, _D, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "tpmg_kernel_launch_count": (C.c_int, [_VP, C.POINTER(C.c_int64)]),
    "tpmg_nccl_call_count": (C.c_int, [C.POINTER(C.c_int64)]),
    "tpmg_set_use_graphs": (C.c_int, [_VP, C.c_int]),
    "tpmg_time_kernel": (C.c_int, [_VP, C.c_int, C.c_int, C.c_int, _D]),
    "tpmg_kernel_probe": (C.c_int, [_VP, C.c_int]),
    "tpmg_kernel_probe_read": (C.c_int, [_VP, C.c_int, _D, C.POINTER(C.c_int64)]),
    "tpmg_profile_packed_size": (C.c_int64, [C.c_int, C.c_int64, C.c_int64, C.c_int64]),
    "tpmg_grid_fingerprint": (C.c_uint64, [_D, C.c_int64]),
    "tpmg_grid_fingerprint_cartesian": (C.c_uint64, [C.c_void_p]),
    "tpmg_profile_save_grid": (C.c_int, [C.c_char_p, C.c_void_p, C.c_int, _D, C.c_int]),
    "tpmg_profile_load_grid": (C.c_int, [C.c_char_p, C.c_void_p, C.POINTER(C.c_int), _D, C.c_int64]),
    "tpmg_profile_save": (C.c_int, [C.c_char_p, C.c_void_p, C.c_int, _D, C.c_int]),
    "tpmg_profile_load": (C.c_int, [C.c_char_p, C.c_void_p, C.POINTER(C.c_int), _D, C.c_int64]),
    "tpmg_profile_last_error": (C.c_char_p, []),
}


class ContextParams(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("world_size", C.c_int), ("px", C.c_int),
                ("py", C.c_int), ("nccl_id", C.c_void_p)]


class GridDesc(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("hx", C.c_double), ("hy", C.c_double),
                ("nz", C.c_int64), ("z_faces", _D)]


class FactorizedProfiles(C.Structure):
    _fields_ = [(n, _D) for n in ("beta_r", "alpha_s_r", "alpha_r_r", "xi_r_r", "beta_s",
                                  "alpha_r_s", "xi_r_s", "alpha_s_s")]


class FullProfiles(C.Structure):  # tpmg_full_profiles
    _fields_ = [(n, _D) for n in ("beta", "alpha_s", "alpha_r", "xi_r")]


class ProfileGrid(C.Structure):  # tpmg_profile_grid
    _fields_ = [("type", C.c_char_p), ("fingerprint", C.c_uint64), ("level", C.c_int64),
                ("n_r", C.c_int64), ("n_cells", C.c_int64), ("n_edges", C.c_int64),
                ("nx", C.c_int64), ("ny", C.c_int64)]


class MGConfig(C.Structure):
    _fields_ = [("smoother", C.c_int), ("relax", C.c_double), ("prolongation", C.c_int),
                ("restriction", C.c_int), ("nu_pre", C.c_int), ("nu_post", C.c_int),
                ("depth", C.c_int), ("agglomerate", C.c_int)]


_libs: dict = {}


def lib_path(variant: str = "exact") -> str:
    # TPMG_LIB_PATH: an alternative build of the product library (A/B kernel timing only)
    if variant == "exact" and os.environ.get("TPMG_LIB_PATH"):
        return os.environ["TPMG_LIB_PATH"]
    return os.path.join(PKG_DIR, LIB_NAMES[variant])


def load(variant: str = "exact"):
    """Load (once) the C-ABI library; raises if the CUDA extension was not built."""
    if variant in _libs:
        return _libs[variant]
    path = lib_path(variant)
    if not os.path.exists(path):
        raise RuntimeError(f"TPMG CUDA extension missing: {path} (run __graft_entry__.build())")
    L = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _libs[variant] = L
    return L
