"""CPU tests of the oracle (the parity checker) -- the reference's hot-path property tests
(proj/tests/test_discretization.cpp, test_relaxation.cpp,
test_multigrid.cpp) re-expressed on the doubly periodic Cartesian grid, plus the golden
regression vectors under tests/golden/.  No GPU needed."""
import json
import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from conftest import rng_field
from fv_reference import assemble
from paper_1408_2981_b200 import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def small(nx=8, ny=6, nz=5, **kw):
    base = dict(omega2=2e-2, lambda2=0.3, grading="quadratic", profile="uniform", profile_seed=3,
                depth=1, relax=1.0)
    base.update(kw)
    return synth.make_problem(nx, ny, nz, **base)


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


# ---- discretization (test_discretization.cpp) ------------------------------------------------

def test_apply_matches_independent_fv_assembly(O):
    """matrix-free apply == term-by-term FV matrix (test_discretization.cpp:158-195, :266-289)."""
    for P in (small(), small(12, 8, 7, grading="geometric", ratio=1.3),
              small(8, 8, 4, profile="lognormal", grading="uniform")):
        h = O.OracleHierarchy.from_problem(P)
        A = assemble(P)
        assert np.allclose(h.apply(0, np.zeros(A.shape[0])), 0.0, atol=0)
        for s in range(10):
            u = rng_field(100 + s, A.shape[0])
            ref = A @ u
            assert np.max(np.abs(h.apply(0, u) - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_column_row_sum_identity_and_vertical_symmetry(O):
    """diag = beta_hat - sum(off-diagonals) exactly; upper[k] = lower[k+1] when xi = 0
    (test_discretization.cpp:119-139)."""
    P = small()
    h = O.OracleHierarchy.from_problem(P)
    co = h.coefficients(0)
    for cell in (0, 7, 23, 47):
        d, up, lo, nb = h.build_column(0, cell)
        bh = co["bh"][cell]
        for k in range(P.nz):
            s = ((nb[0, k] + nb[1, k]) + nb[2, k]) + nb[3, k]
            assert d[k] == co["bv"][k] * bh - ((up[k] + lo[k]) + s)
        assert np.array_equal(up[:-1], lo[1:])
        assert up[-1] == 0.0 and lo[0] == 0.0


def test_operator_annihilates_constants_without_mass(O):
    """beta = 0, xi = 0  =>  A 1 = 0 (test_discretization.cpp:141-156)."""
    P = small(lambda2=0.0)
    h = O.OracleHierarchy.from_problem(P)
    y = h.apply(0, np.ones(P.n_dof))
    scale = np.max(np.abs(h.apply(0, rng_field(1, P.n_dof))))
    assert np.max(np.abs(y)) <= 1e-12 * scale


def test_impulse_response_is_the_7_point_stencil(O):
    """support of A e_T = the column and its 4 face neighbours (test_discretization.cpp:197-222)."""
    P = small(8, 8, 6)
    h = O.OracleHierarchy.from_problem(P)
    i, j, k = 3, 4, 2
    e = np.zeros(P.n_dof)
    e[(j * 8 + i) * 6 + k] = 1.0
    y = h.apply(0, e).reshape(8, 8, 6)  # [j][i][k]
    support = {(j, i, k), (j, i, k - 1), (j, i, k + 1), (j, i - 1, k), (j, i + 1, k),
               (j - 1, i, k), (j + 1, i, k)}
    for jj in range(8):
        for ii in range(8):
            for kk in range(6):
                if (jj, ii, kk) in support:
                    assert y[jj, ii, kk] != 0.0
                else:
                    assert y[jj, ii, kk] == 0.0


def test_operator_symmetric_positive_definite(O):
    """xi = 0 => A symmetric, x^T A x > 0 (test_discretization.cpp:224-264)."""
    P = small()
    h = O.OracleHierarchy.from_problem(P)
    A = assemble(P)
    assert abs(A - A.T).max() <= 1e-14 * abs(A).max()
    for s in range(20):
        u, v = rng_field(200 + s, P.n_dof), rng_field(300 + s, P.n_dof)
        a, b = np.dot(h.apply(0, u), v), np.dot(u, h.apply(0, v))
        assert abs(a - b) <= 1e-12 * max(abs(a), 1e-300)
        assert np.dot(u, h.apply(0, u)) > 0.0


def test_thread_count_bitwise_independence(O):
    """apply / Jacobi are bitwise independent of the thread count (test_discretization.cpp:
    337-353, test_relaxation.cpp:190-201)."""
    P = small(16, 16, 8)
    h1 = O.OracleHierarchy.from_problem(P, threads=1)
    h4 = O.OracleHierarchy.from_problem(P, threads=4)
    u, f = rng_field(5, P.n_dof), rng_field(6, P.n_dof)
    assert np.array_equal(h1.apply(0, u), h4.apply(0, u))
    assert np.array_equal(h1.smooth(0, u, f, 3), h4.smooth(0, u, f, 3))


# ---- relaxation (test_relaxation.cpp) ---------------------------------------------------------

def test_thomas_identity_and_1x1(O):
    rhs = np.array([3.0, -1.0, 2.0, 7.0])
    assert np.array_equal(O.thomas(np.ones(4), np.zeros(4), np.zeros(4), rhs), rhs)
    assert O.thomas([4.0], [0.0], [0.0], [2.0])[0] == 0.5


def test_thomas_vs_dense_solve():
    """200 random diagonally dominant 64x64 systems (test_relaxation.cpp:85-108)."""
    import oracle as Ox

    rng = np.random.default_rng(23)
    for _ in range(200):
        n = 64
        up = np.where(np.arange(n) + 1 < n, rng.uniform(-1, 1, n), 0.0)
        lo = np.where(np.arange(n) > 0, rng.uniform(-1, 1, n), 0.0)
        d = rng.uniform(2.5, 4.0, n)
        rhs = rng.uniform(-1, 1, n)
        x = Ox.thomas(d, up, lo, rhs)
        A = np.diag(d) + np.diag(up[:-1], 1) + np.diag(lo[1:], -1)
        ref = np.linalg.solve(A, rhs)
        assert np.max(np.abs(x - ref)) <= 1e-10 * np.max(np.abs(ref))
        assert np.max(np.abs(A @ x - rhs)) <= 1e-10 * np.max(np.abs(rhs))


def test_thomas_zero_pivot_is_singular_error(O):
    """(test_relaxation.cpp:110-126): status 5 = singular_error."""
    with pytest.raises(O.OracleError) as e:
        O.thomas([1.0, 1.0], [1.0, 0.0], [0.0, 1.0], [1.0, 2.0])
    assert e.value.code == 5
    with pytest.raises(O.OracleError) as e:
        O.thomas([0.0], [0.0], [0.0], [1.0])
    assert e.value.code == 5


def test_smoother_fixed_point_at_exact_solution(O):
    """(test_relaxation.cpp:128-141)"""
    P = small()
    h = O.OracleHierarchy.from_problem(P)
    f = rng_field(31, P.n_dof)
    exact = spla.spsolve(assemble(P).tocsc(), f)
    u = h.smooth(0, exact, f, 2)
    assert np.max(np.abs(u - exact)) <= 1e-12 * np.max(np.abs(exact))


def test_block_diagonal_operator_solved_by_one_sweep(O):
    """(test_relaxation.cpp:143-164)"""
    P = small(lambda2=2.5)
    P.alpha_s_s[:] = 0.0
    h = O.OracleHierarchy.from_problem(P)
    f, u = rng_field(1, P.n_dof), rng_field(2, P.n_dof)
    u = h.smooth(0, u, f, 1)
    assert np.max(np.abs(h.apply(0, u) - f)) <= 1e-13 * np.max(np.abs(f))


def test_one_jacobi_sweep_matches_dense_block_jacobi(O):
    """u + relax D^-1 (f - A u), D = block diagonal of A (test_relaxation.cpp:166-188)."""
    P = small(relax=0.9)
    h = O.OracleHierarchy.from_problem(P)
    A = assemble(P).toarray()
    u, f = rng_field(41, P.n_dof), rng_field(42, P.n_dof)
    res = f - A @ u
    ref = u.copy()
    nz = P.nz
    for c in range(P.nx * P.ny):
        s = slice(c * nz, (c + 1) * nz)
        ref[s] += 0.9 * np.linalg.solve(A[s, s], res[s])
    got = h.smooth(0, u, f, 1)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_damped_jacobi_contracts_energy_norm(O):
    """relax = 0.5 (test_relaxation.cpp:222-243)"""
    P = small(relax=0.5)
    h = O.OracleHierarchy.from_problem(P)
    A = assemble(P)
    f = rng_field(71, P.n_dof)
    exact = spla.spsolve(A.tocsc(), f)
    u = rng_field(72, P.n_dof)

    def energy(x):
        e = x - exact
        return np.sqrt(e @ (A @ e))

    prev = energy(u)
    for _ in range(10):
        u = h.smooth(0, u, f, 1)
        now = energy(u)
        assert now <= prev * (1 + 1e-12)
        prev = now


def test_linear_transfers_need_three_coarse_cells(O):
    with pytest.raises(O.OracleError) as e:
        O.OracleHierarchy.from_problem(small(16, 8, 3, depth=3))  # coarsest 4x2
    assert e.value.code == 1


def test_relaxation_factor_validated(O):
    with pytest.raises(O.OracleError) as e:
        O.OracleHierarchy.from_problem(small(relax=2.5))
    assert e.value.code == 1


# ---- multigrid (test_multigrid.cpp) -----------------------------------------------------------

def test_summation_restriction(O):
    """ones -> 4, impulse -> parent, brute-force 4-sums (test_multigrid.cpp:22-52)."""
    P = small(8, 8, 3, depth=2)
    h = O.OracleHierarchy.from_problem(P, restriction=0)
    assert np.array_equal(h.restrict(0, np.ones(P.n_dof)), np.full(h.size(0), 4.0))
    fine = rng_field(3, P.n_dof).reshape(8, 8, 3)  # [j][i][k]
    c = h.restrict(0, fine.reshape(-1)).reshape(4, 4, 3)
    for J in range(4):
        for I in range(4):
            ref = ((fine[2 * J, 2 * I] + fine[2 * J, 2 * I + 1]) + fine[2 * J + 1, 2 * I]) + \
                fine[2 * J + 1, 2 * I + 1]
            assert np.array_equal(c[J, I], ref)


def test_linear_prolongation_properties(O):
    """constants reproduced, linear functions reproduced away from the periodic seam,
    injection = parent (test_multigrid.cpp:54-115)."""
    P = small(16, 16, 2, depth=2)
    h = O.OracleHierarchy.from_problem(P, prolongation=0)
    assert np.array_equal(h.prolong(0, np.full(h.size(0), 2.5)), np.full(P.n_dof, 2.5))
    # coarse linear function in x: c(I) = I  -> child x-centre (2I+a)/2 - 1/4 ... => I + (a-1/2)/2
    cx = np.repeat(np.tile(np.arange(8.0), 8), 2)  # [J][I][k]
    fine = h.prolong(0, cx).reshape(16, 16, 2)
    for j in range(16):
        for i in range(2, 14):
            assert fine[j, i, 0] == pytest.approx((i - 0.5) / 2.0, abs=1e-14)
    hi = O.OracleHierarchy.from_problem(P, prolongation=1)
    c = rng_field(9, hi.size(0))
    f = hi.prolong(0, c).reshape(16, 16, 2)
    cc = c.reshape(8, 8, 2)
    for j in range(16):
        for i in range(16):
            assert np.array_equal(f[j, i], cc[j // 2, i // 2])


def test_transpose_restriction_is_adjoint_of_linear_prolongation(O):
    """<R f, c> = <f, P c> (test_multigrid.cpp:117-133); summation = injection^T exactly."""
    P = small(24, 16, 3, depth=3)  # coarsest 6x4
    for pk, rk in ((0, 1), (1, 0)):
        h = O.OracleHierarchy.from_problem(P, prolongation=pk, restriction=rk)
        for lc in range(h.n_levels - 1):
            f = rng_field(10 + lc, h.size(lc + 1))
            c = rng_field(20 + lc, h.size(lc))
            a, b = np.dot(h.restrict(lc, f), c), np.dot(f, h.prolong(lc, c))
            assert abs(a - b) <= 1e-12 * abs(a)


def test_hierarchy_exact_for_horizontally_constant_profiles(O):
    """coarse coefficients of constant profiles are the rediscretised ones
    (test_multigrid.cpp:135-172): horizontal scalars scale with the cell area, edge scalars
    are level independent."""
    P = synth.make_problem(32, 16, 6, omega2=1e-2, lambda2=1e-4, depth=3)
    h = O.OracleHierarchy.from_problem(P)
    fine, coarse = h.coefficients(2), h.coefficients(0)
    assert np.allclose(coarse["bh"], 16 * fine["bh"][0], rtol=1e-15)
    assert np.allclose(coarse["ah"], 16 * fine["ah"][0], rtol=1e-15)
    assert np.allclose(coarse["sh"], fine["sh"][0], rtol=1e-15)


def test_vcycle_zero_and_linear(O):
    """f = 0 -> 0, linear in f from a zero guess (test_multigrid.cpp:174-198); with the
    transpose pair the V-cycle is also symmetric (the PCG preconditioner requirement)."""
    P = synth.baseline_config(1)
    h = O.OracleHierarchy.from_problem(P)
    n = P.n_dof
    assert np.array_equal(h.vcycle(np.zeros(n)), np.zeros(n))
    f, g = rng_field(1, n), rng_field(2, n)
    v1, v2, v3 = h.vcycle(f), h.vcycle(g), h.vcycle(2.0 * f - 3.0 * g)
    assert np.max(np.abs(v3 - (2.0 * v1 - 3.0 * v2))) <= 1e-12 * np.max(np.abs(v3))
    a, b = np.dot(v1, g), np.dot(f, v2)
    assert abs(a - b) <= 1e-12 * abs(a)


def test_cycle_rate(O):
    """a block-diagonal operator is solved by one V-cycle; config 1 contracts at < 0.5
    (test_multigrid.cpp:200-261)."""
    P = small(16, 16, 8, depth=3, lambda2=1.0)
    P.alpha_s_s[:] = 0.0
    h = O.OracleHierarchy.from_problem(P)
    f = rng_field(4, P.n_dof)
    r = h.residual(h.finest, f, h.vcycle(f))
    assert np.linalg.norm(r) <= 1e-13 * np.linalg.norm(f)
    P1 = synth.baseline_config(1)
    h1 = O.OracleHierarchy.from_problem(P1)
    f = synth.x_fastest_to_k_fastest(P1.rhs())
    assert h1.measure_cycle_rate(f, 6) < 0.5
    with pytest.raises(O.OracleError):
        h1.measure_cycle_rate(f, 1)


def test_pcg_solves_config1(O):
    P = synth.baseline_config(1)
    h = O.OracleHierarchy.from_problem(P)
    f = synth.x_fastest_to_k_fastest(P.rhs())
    x, hist, it, st = h.pcg(f, P.tol, 100)
    assert st == 0 and it == 11
    r = f - assemble(P) @ x
    assert np.linalg.norm(r) <= 1.01 * P.tol * np.linalg.norm(f)
    assert hist[-1] / hist[0] <= P.tol


# ---- golden vectors ---------------------------------------------------------------------------

def _load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def test_golden_config1_pcg_history(O):
    """Regression pin of the oracle's config-1 solve (tests/golden/make_golden.py)."""
    g = _load("oracle_cfg1_pcg.json")
    P = synth.baseline_config(1)
    h = O.OracleHierarchy.from_problem(P)
    f = synth.x_fastest_to_k_fastest(P.rhs())
    x, hist, it, st = h.pcg(f, P.tol, 100)
    assert it == g["iterations"]
    assert [float(v).hex() for v in hist] == g["history_hex"]
    assert float(np.sum(x)).hex() == g["x_sum_hex"]


def test_synthetic_rhs_mean_removed_and_decomposition_independent():
    f = synth.rhs_x_fastest(0, 32, 16, 8)
    assert abs(f.sum()) <= 1e-12 * f.size
    tile = synth.rhs_x_fastest(0, 32, 16, 8, x0=16, y0=8, lnx=16, lny=8)
    assert np.array_equal(tile, f[:, 8:16, 16:32])
    mean = synth.rhs_mean(0, 32 * 16 * 8)
    assert (f + mean).min() >= -1.0 and (f + mean).max() < 1.0
    # distributed mean: exact tile sums add up to the global one
    parts = [synth.tile_m_sum(0, 32, 16, 8, x, y, 16, 8) for x in (0, 16) for y in (0, 8)]
    assert synth.mean_from_m_sum(sum(parts), 32 * 16 * 8) == mean
    t2 = synth.rhs_x_fastest(0, 32, 16, 8, x0=16, y0=8, lnx=16, lny=8, mean=mean)
    assert np.array_equal(t2, tile)


@pytest.mark.parametrize("cfg", ["cfg1", "small_graded"])
def test_forward_pass_rz_matches_direct_dot(O, cfg):
    """The fused schedule's r.z (sum r u + relax sum w d' with w = U^-T r, formed in the
    post-sweep's forward pass; oracle thomas_rz) against the plain schedule's direct r.z dot:
    the same PCG to rounding.  A CG residual history is only reproducible to the rounding of its
    dot products: merely reordering the direct dots (device tree vs host chunks) moves it by up
    to ~4e-9 on the 33-iteration problem, so the reformulation must stay within that envelope
    (and the product matches the oracle's own formula bit for bit)."""
    P = (synth.baseline_config(1) if cfg == "cfg1" else
         synth.make_problem(64, 32, 16, omega2=1e-3, lambda2=1e-4, grading="quadratic",
                            profile="uniform", profile_seed=3, depth=3, name=cfg))
    f = synth.x_fastest_to_k_fastest(P.rhs())

    def run(fused, device_order=True):
        h = O.OracleHierarchy.from_problem(P)
        O.lib().tpmgo_set_pcg_fused(h._h, fused)
        h.set_device_order(device_order)
        return h.pcg(f, P.tol, 200)

    x1, h1, it1, s1 = run(1)
    x0, h0, it0, s0 = run(0)
    _, h0h, it0h, _ = run(0, device_order=False)  # the same dots, another summation order
    assert s1 == s0 == 0 and it1 == it0 == it0h
    d_formula = np.max(np.abs(h1 - h0) / h0)
    d_order = np.max(np.abs(h0h - h0) / h0)
    assert d_formula <= max(2.0 * d_order, 1e-13), (d_formula, d_order)
    assert d_formula <= 1e-8
    assert np.max(np.abs(x1 - x0)) <= 1e-8 * np.max(np.abs(x0))
