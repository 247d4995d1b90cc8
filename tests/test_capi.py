"""CPU tests of the drop-in boundary: the C-ABI libraries load, export exactly what
include/tpmg_b200.h declares, carry sm_100a code, fail loudly without a device, and the
pure-host decomposition planner behaves.  No compute calls (no GPU needed)."""
import ctypes as C
import os
import re
import shutil
import subprocess

import pytest

from paper_1408_2981_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tpmg_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(tpmg_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for must in ("tpmg_init", "tpmg_hier_create", "tpmg_apply", "tpmg_smooth", "tpmg_restrict",
                 "tpmg_prolong_add", "tpmg_vcycle", "tpmg_pcg", "tpmg_pcg_host", "tpmg_dot"):
        assert must in fns
    assert set(fns) == set(_capi.SIGNATURES), set(fns) ^ set(_capi.SIGNATURES)


@pytest.mark.parametrize("variant", ["exact", "fma"])
def test_library_exports_every_declared_symbol(variant):
    lib = C.CDLL(_capi.lib_path(variant))
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, missing
    L = _capi.load(variant)
    assert L.tpmg_abi_version() == 2
    assert L.tpmg_status_string(0) == b"ok"
    assert L.tpmg_status_string(5) == b"singular_error"


@pytest.mark.parametrize("variant", ["exact", "fma"])
def test_library_carries_sm100a_code(variant):
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _capi.lib_path(variant)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([cuobjdump, "-sass", _capi.lib_path(variant)], capture_output=True,
                          text=True).stdout
    assert "STTM" in sass and "LDTM" in sass        # tcgen05.st / tcgen05.ld (TMEM scratch)
    assert "LDGSTS" in sass                          # cp.async plane pipeline


def test_init_fails_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1408_2981_b200 import tpmg

    with pytest.raises(tpmg.cuda_error):
        tpmg.Context()


def test_cpp_adapter_builds_and_links(tmp_path):
    """include/tpmg_b200.hpp (reference-shaped C++ calls) compiles and links against the
    C-ABI library; without a device the Context constructor throws (no CPU fallback)."""
    import torch

    src = tmp_path / "use.cpp"
    src.write_text(
        '#include "tpmg_b200.hpp"\n#include <cstdio>\n'
        "int main() {\n"
        "  try { tpmg_b200::Context ctx(0); std::puts(\"device\"); return 0; }\n"
        "  catch (const tpmg_b200::device_error& e) { std::puts(\"no device\"); return 3; }\n"
        "}\n")
    exe = tmp_path / "use"
    pkg = os.path.dirname(_capi.lib_path("exact"))
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                    str(exe), "-L", pkg, "-l:libtpmg_b200.so", f"-Wl,-rpath,{pkg}"], check=True)
    rc = subprocess.run([str(exe)], capture_output=True, text=True)
    assert rc.returncode == (0 if torch.cuda.is_available() else 3), rc.stdout + rc.stderr


def plan(nx, ny, px, py, rank, depth=0):
    L = _capi.load("exact")
    n = C.c_int()
    arrs = [(C.c_int64 * 32)() for _ in range(4)]
    nbr = (C.c_int * 4)()
    rc = L.tpmg_plan_decomposition(nx, ny, px, py, rank, depth, 32, C.byref(n), *arrs, nbr)
    return rc, n.value, [list(a[: n.value]) for a in arrs], list(nbr)


def test_decomposition_plan():
    rc, n, (tnx, tny, x0, y0), nbr = plan(2048, 1024, 4, 2, 5, depth=9)
    assert rc == 0 and n == 9
    assert tnx[-1] == 512 and tny[-1] == 512 and tnx[0] == 2 and tny[0] == 2
    assert x0[-1] == 512 and y0[-1] == 512  # rank 5 = (rx 1, ry 1)
    assert nbr == [4, 6, 1, 1]               # py = 2: S and N neighbours coincide
    rc, n, _, nbr = plan(1024, 1024, 1, 1, 0, depth=8)
    assert rc == 0 and n == 8 and nbr == [0, 0, 0, 0]
    rc, n, _, _ = plan(32, 32, 1, 1, 0)
    assert rc == 0 and n == 4  # depth 0: down to 4x4
    assert plan(1000, 1024, 3, 1, 0)[0] == 1   # config_error: uneven split
    assert plan(64, 64, 2, 2, 0, depth=7)[0] == 1  # tile 32 cannot halve 6 times
