"""Oracle pinned against the REFERENCE ITSELF.

oracle/build_ref.py compiles the reference's unmodified headers (proj/include/tpmg/*.hpp)
against oracle/eigen_shim and runs oracle/ref_driver.cpp on the reference's own problem
(icosahedral hierarchy, balanced-flow factorised profiles with vertical advection, geometric
vertical grading, block-Jacobi relax 0.9, nu = 2+2).  Its inputs/outputs are committed as
tests/golden/ref_icosa_pin.bin (refreshed from oracle/_ref/ when the reference is present).
Here the oracle, fed the reference's neighbour/edge/child tables and hatted coefficients
through its generic-table entry point, must reproduce every element-wise result BIT FOR BIT:
the operator apply and its explicit matrix, Thomas, two block-Jacobi sweeps, summation and
transpose restriction, linear and injection prolongation, and whole V-cycles for all three
transfer pairs.  Only norm-based diagnostics are compared with a tolerance (the shim's
sequential reduction order stands in for Eigen's vectorised one)."""
import os
import struct

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
FILES = [os.path.join(ROOT, "oracle", "_ref", "ref_pin.bin"),
         os.path.join(HERE, "golden", "ref_icosa_pin.bin")]


def load():
    path = next((p for p in FILES if os.path.exists(p)), None)
    if path is None:
        pytest.skip("no reference pin data")
    out = {}
    with open(path, "rb") as fh:
        buf = fh.read()
    off = 0
    while off < len(buf):
        (nl,) = struct.unpack_from("<I", buf, off); off += 4
        name = buf[off:off + nl].decode(); off += nl
        dt = chr(buf[off]); off += 1
        (nd,) = struct.unpack_from("<I", buf, off); off += 4
        dims = struct.unpack_from("<%dq" % nd, buf, off); off += 8 * nd
        n = int(np.prod(dims))
        arr = np.frombuffer(buf, dtype=np.float64 if dt == "d" else np.int64, count=n, offset=off)
        off += 8 * n
        # 2-D records are column-major (Eigen): reshape (cols, rows) -> flat column-major order
        out[name] = arr.copy()
    return out


@pytest.fixture(scope="module")
def R():
    return load()


def make_oracle(O, R, prolongation=0, restriction=0):
    nl = int(R["n_levels"][0])
    nz = int(R["nr"][0])
    ncells = [len(R["bh%d" % l]) for l in range(nl)]
    nedges = [len(R["sh%d" % l]) for l in range(nl)]
    children = [None] + [np.arange(4 * ncells[l - 1], dtype=np.int64) for l in range(1, nl)]
    return O.OracleHierarchy.from_tables(
        nz, 3, 4, ncells, nedges, [R["nbr%d" % l] for l in range(nl)],
        [R["cedge%d" % l] for l in range(nl)], children, [1, 2, 0, -1], [2, 0, 1, -1],
        R["bv"], R["sv"], R["av"], R["xv"], [R["bh%d" % l] for l in range(nl)],
        [R["ah%d" % l] for l in range(nl)], [R["xh%d" % l] for l in range(nl)],
        [R["sh%d" % l] for l in range(nl)], float(R["relax"][0]), prolongation, restriction,
        2, 2)


def same(a, b, what):
    bad = np.flatnonzero(a != b)
    assert bad.size == 0, f"{what}: {bad.size}/{a.size} differ, first {bad[:5]}, max |d| " \
                          f"{np.max(np.abs(a - b)):.3e}"


def test_apply_bitwise(oracle_mod, R):
    o = make_oracle(oracle_mod, R)
    same(o.apply(o.finest, R["u"]), R["apply"], "apply_operator")


def test_explicit_matrix_bitwise(oracle_mod, R):
    """dense_assemble (discretization.hpp:291-316) entries == oracle build_column."""
    o = make_oracle(oracle_mod, R)
    nz = int(R["nr"][0])
    trip = R["triplets"].reshape(-1, 3)  # (row, col, value) triplets, one after another
    nbr = R["nbr%d" % o.finest].reshape(-1, 3)
    ents = {(int(r), int(c)): v for r, c, v in trip}
    for T in range(0, o.n_cells(o.finest), 7):
        d, up, lo, nb = o.build_column(o.finest, T)
        for k in range(nz):
            row = T * nz + k
            assert ents[(row, row)] == d[k]
            if k + 1 < nz:
                assert ents[(row, row + 1)] == up[k]
            if k > 0:
                assert ents[(row, row - 1)] == lo[k]
            for j in range(3):
                assert ents[(row, int(nbr[T, j]) * nz + k)] == nb[j, k]


def test_thomas_bitwise(oracle_mod, R):
    x = oracle_mod.thomas(R["th_diag"], R["th_upper"], R["th_lower"], R["th_rhs"])
    same(x, R["th_x"], "thomas_solve")


def test_block_jacobi_bitwise(oracle_mod, R):
    o = make_oracle(oracle_mod, R)
    same(o.smooth(o.finest, R["u"], R["f"], 2), R["smooth2"], "smooth x2")


@pytest.mark.parametrize("lc", [0, 1])
def test_transfers_bitwise(oracle_mod, R, lc):
    s = str(lc)
    o_sum = make_oracle(oracle_mod, R, 0, 0)
    o_tr = make_oracle(oracle_mod, R, 0, 1)
    o_inj = make_oracle(oracle_mod, R, 1, 0)
    same(o_sum.restrict(lc, R["tr_fine" + s]), R["restrict_sum" + s], "restrict_field")
    same(o_tr.restrict(lc, R["tr_fine" + s]), R["restrict_T" + s], "restrict_field_transpose")
    same(o_sum.prolong(lc, R["tr_coarse" + s]), R["prolong_lin" + s], "prolongate linear")
    same(o_inj.prolong(lc, R["tr_coarse" + s]), R["prolong_inj" + s], "prolongate injection")


@pytest.mark.parametrize("c,pr", [(0, (0, 0)), (1, (0, 1)), (2, (1, 0))])
def test_vcycle_bitwise(oracle_mod, R, c, pr):
    o = make_oracle(oracle_mod, R, *pr)
    same(o.vcycle(R["f"], R["u0"]), R["vcycle%d" % c], "v_cycle")
    rate = o.measure_cycle_rate(R["f"], 4)
    assert abs(rate - R["rate%d" % c][0]) <= 1e-12 * abs(R["rate%d" % c][0])
