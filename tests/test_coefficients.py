"""Partial and full (non-factorised) coefficient storage: the reference's
MixedProfileSet (alpha_r dense) and ProfileSet (every component dense), assembled per level by
assemble_hatted (discretization.hpp:104-141, 187-204) from profiles restricted by
restrict_profiles (multigrid.hpp:146-201), read by build_column through
HattedComponent::operator() (discretization.hpp:39-41).

CPU: the oracle's dense modes against its factorised mode on separable data (equal up to the
association of the products) and as solvers.  GPU: the device's partial / full kernels bit for
bit against the oracle, operator by operator and through the whole fused PCG solve.
"""
import numpy as np
import pytest

from conftest import rng_field
from paper_1408_2981_b200 import synth, tpmg
from paper_1408_2981_b200.tpmg import K_FASTEST


def _cfg2s():
    return synth.make_problem(64, 32, 24, omega2=1e-2, lambda2=1e-4, grading="quadratic",
                              profile="uniform", profile_seed=1, depth=3, name="cfg2-small")


def _adv():
    P = synth.make_problem(64, 32, 12, omega2=1e-2, lambda2=1e-3, grading="geometric", ratio=1.2,
                           profile="uniform", profile_seed=5, depth=3, name="adv")
    rng = np.random.default_rng(9)
    P.xi_r_r = 0.3 * rng.standard_normal(P.nz + 1) / P.omega ** 2
    P.xi_r_s = P.beta_s.copy()
    return P


# ---- CPU: the restatement ---------------------------------------------------------------------

@pytest.mark.parametrize("coef", ["partial", "full"])
def test_dense_storage_of_separable_profiles_matches_factorized(oracle_mod, coef):
    """eps = 0: the dense profiles are exactly the outer products, so the operator, the smoother
    and the V-cycle agree with the factorised hierarchy up to the association of the products
    ((w2 |T|) f_k a versus (f_k a_r) (w2 (|T| a_s)))."""
    P = _cfg2s()
    Q = synth.with_coefficients(P, coef, eps=0.0)
    o, od = (oracle_mod.OracleHierarchy.from_problem(X) for X in (P, Q))
    for l in range(o.n_levels):
        u = rng_field(3 + l, o.size(l))
        a, b = o.apply(l, u), od.apply(l, u)
        assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(a)), (coef, l)
    f = synth.x_fastest_to_k_fastest(P.rhs())
    za, zb = o.vcycle(f), od.vcycle(f)
    assert np.max(np.abs(za - zb)) <= 1e-10 * np.max(np.abs(za))


@pytest.mark.parametrize("coef", ["partial", "full"])
def test_dense_modes_solve(oracle_mod, coef):
    P = synth.with_coefficients(_cfg2s(), coef, eps=0.2)
    o = oracle_mod.OracleHierarchy.from_problem(P)
    f = synth.x_fastest_to_k_fastest(P.rhs())
    x, hist, it, st = o.pcg(f, 1e-8, 200)
    assert st == 0 and hist[-1] <= 1e-8 * hist[0]
    assert np.linalg.norm(o.residual(o.finest, f, x)) <= 1.01e-8 * hist[0]


def test_full_mode_is_really_dense(oracle_mod):
    """With eps > 0 the full operator differs from the factorised one (the test above is not
    vacuous)."""
    P = _cfg2s()
    o = oracle_mod.OracleHierarchy.from_problem(P)
    od = oracle_mod.OracleHierarchy.from_problem(synth.with_coefficients(P, "full", eps=0.2))
    u = rng_field(5, o.size(o.finest))
    a, b = o.apply(o.finest, u), od.apply(od.finest, u)
    assert np.max(np.abs(a - b)) > 1e-3 * np.max(np.abs(a))


# ---- GPU: the device path ---------------------------------------------------------------------

def _pair(gpu_ctx, oracle_mod, P):
    return tpmg.Hierarchy(gpu_ctx, P), oracle_mod.OracleHierarchy.from_problem(P)


def _bitwise(a, b, what):
    bad = np.flatnonzero(a != b)
    assert bad.size == 0, f"{what}: {bad.size} elements differ bitwise (first {bad[:5]})"


@pytest.mark.gpu
@pytest.mark.parametrize("coef", ["partial", "full"])
@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "adv"])
def test_dense_kernels_bitwise(gpu_ctx, oracle_mod, coef, name):
    base = {"cfg1": synth.baseline_config(1), "cfg2s": _cfg2s(), "adv": _adv()}[name]
    P = synth.with_coefficients(base, coef, eps=0.2)
    h, o = _pair(gpu_ctx, oracle_mod, P)
    mode = tpmg.C.c_int()
    h.lib.tpmg_hier_coef_mode(h._h, tpmg.C.byref(mode))
    assert mode.value == {"partial": 1, "full": 2}[coef]
    for l in range(h.n_levels):
        n = o.size(l)
        u, f = rng_field(10 + l, n), rng_field(20 + l, n)
        fu, fy, ff = h.field(l).upload(u, K_FASTEST), h.field(l), h.field(l).upload(f, K_FASTEST)
        tpmg.apply_operator(h, fu, fy)
        _bitwise(fy.download(K_FASTEST), o.apply(l, u), f"apply level {l}")
        tpmg.residual(h, ff, fu, fy)
        _bitwise(fy.download(K_FASTEST), o.residual(l, f, u), f"residual level {l}")
        tpmg.smooth(h, fu, ff, 2)
        _bitwise(fu.download(K_FASTEST), o.smooth(l, u, f, 2), f"smooth level {l}")
    f = synth.x_fastest_to_k_fastest(P.rhs())
    fu = h.field()
    tpmg.v_cycle(h, h.field().upload(f, K_FASTEST), fu)
    _bitwise(fu.download(K_FASTEST), o.vcycle(f), "v_cycle")


@pytest.mark.gpu
@pytest.mark.parametrize("coef", ["partial", "full"])
@pytest.mark.parametrize("name", ["cfg2s", "cfg1"])
def test_dense_pcg_bitwise(gpu_ctx, oracle_mod, coef, name):
    """The fused PCG schedule (direction update + A p, r-update pre-sweep with q = A p inside,
    fused residual + restriction, r.z post-sweep) in the dense modes."""
    base = {"cfg1": synth.baseline_config(1), "cfg2s": _cfg2s()}[name]
    P = synth.with_coefficients(base, coef, eps=0.2)
    h, o = _pair(gpu_ctx, oracle_mod, P)
    f = synth.x_fastest_to_k_fastest(P.rhs())
    xo, hist_o, it_o, st_o = o.pcg(f, P.tol, 200)
    xg = h.field()
    res = tpmg.pcg_solve(h, h.field().upload(P.rhs()), xg, P.tol, 200)
    assert res.status == st_o == 0 and res.iterations == it_o
    assert np.array_equal(res.history, hist_o), "history should be bitwise"
    assert np.array_equal(xg.download(K_FASTEST), xo), "iterate should be bitwise"
