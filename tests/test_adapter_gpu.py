"""The C++ adapters' compute calls on the GPU.

* include/tpmg_b200.hpp (device handles, the reference's call shapes): compiled here by g++
  against the C-ABI (tests/cpp/adapter_cartesian.cpp), run on BASELINE config 1; every result is
  compared with the oracle -- bitwise for the element-wise operations and the solvers (the
  oracle reproduces the device's reduction order), 1e-12 for the cycle rate.
* include/tpmg_b200_ref.hpp (the REFERENCE's own MultigridHierarchy / Field objects): the
  driver oracle/ref_adapter_driver.cpp is compiled with the reference's unmodified headers where
  they exist (oracle/build_ref.py, this container) and travels to the GPU box as
  oracle/_ref/ref_adapter_driver; it compares the device through the adapter with the
  reference's own CPU calls in-process (multigrid.hpp:29-321, discretization.hpp:262-278,
  relaxation.hpp:63-97).
"""
import os
import subprocess

import numpy as np
import pytest

from paper_1408_2981_b200 import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _wr(fh, a):
    a = np.ascontiguousarray(a, dtype=np.float64).ravel()
    np.array([a.size], dtype=np.int64).tofile(fh)
    a.tofile(fh)


def _rd(fh):
    n = int(np.fromfile(fh, dtype=np.int64, count=1)[0])
    return np.fromfile(fh, dtype=np.float64, count=n)


def test_cpp_adapter_compute_calls(tmp_path, oracle_mod):
    exe = tmp_path / "adapter_cartesian"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "adapter_cartesian.cpp"), "-o", str(exe),
                    "-L", os.path.join(ROOT, "paper_1408_2981_b200"), "-ltpmg_b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_1408_2981_b200")], check=True)
    P = synth.baseline_config(1)
    fk = synth.x_fastest_to_k_fastest(P.rhs())
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as fh:
        _wr(fh, [P.nx, P.ny, P.nz, P.hx, P.hy, P.omega, P.relax, P.prolongation, P.restriction,
                 P.nu_pre, P.nu_post, P.depth, P.tol])
        for a in (P.z_faces, P.beta_r, P.alpha_s_r, P.alpha_r_r, P.beta_s, P.alpha_r_s,
                  P.alpha_s_s, fk):
            _wr(fh, a)
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), str(inp), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    o = oracle_mod.OracleHierarchy.from_problem(P)
    L = o.finest
    with open(out, "rb") as fh:
        y, sm, v, c, pc, rate = (_rd(fh) for _ in range(6))
        hist, x, its = _rd(fh), _rd(fh), _rd(fh)
        h_rich, h_bicg, shape = _rd(fh), _rd(fh), _rd(fh)
    np.testing.assert_array_equal(y, o.apply(L, fk))
    np.testing.assert_array_equal(sm, o.smooth(L, fk, fk, 2))
    np.testing.assert_array_equal(v, o.vcycle(fk))
    np.testing.assert_array_equal(c, o.restrict(L - 1, fk))
    np.testing.assert_array_equal(pc, o.prolong(L - 1, o.restrict(L - 1, fk)))
    assert abs(rate[0] - o.measure_cycle_rate(fk, 4)) <= 1e-12 * rate[0]
    xo, hist_o, it_o, st_o = o.pcg(fk, P.tol, 200)
    assert int(its[0]) == it_o and int(its[1]) == st_o == 0
    np.testing.assert_array_equal(hist, hist_o)
    np.testing.assert_array_equal(x, xo)
    _, hr, _, _ = oracle_mod.richardson(o, fk, 1e-5, 200, 1)
    np.testing.assert_array_equal(h_rich, hr)
    _, hb, _, _ = oracle_mod.bicgstab(o, fk, 1e-5, 200, 1)
    np.testing.assert_array_equal(h_bicg, hb)
    assert shape[0] == 1.0


def test_reference_objects_through_the_drop_in_adapter():
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_adapter_driver")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_adapter_driver not built (needs the reference's headers: "
                    "python oracle/build_ref.py)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout + r.stderr
    assert r.stdout.count("bitwise") == 15  # 3 applies, smooth, 2 x 4 transfers, 3 V-cycles
