"""Seeded synthetic inputs of BASELINE.json's configs (host-side setup, not the hot path).

The reference problem setup (icosahedral grid + balanced-flow profiles,
``geometry.hpp`` / ``profiles.hpp``) is out of scope;
BASELINE.json instead names a doubly periodic Cartesian grid with factorised
profiles.  Everything here is pinned once so that the
oracle, the GPU path and the CPU baseline see bit-identical inputs:

* vertical grids: uniform / quadratic ``z_k = H (k/nz)^2`` / geometric, the flat
  analogue of ``build_vertical_grid`` (geometry.hpp:294-327);
* counter-based RNG: SplitMix64 of (seed, global linear index), so inputs do not
  depend on the domain decomposition;
* uniform [-1, 1): ``m * 2^-52 - 1`` with the 53-bit integer ``m`` -- exact in fp64;
  the mean is removed with one correctly rounded division of the exact integer sum;
* smoother damping relax = 0.8 (SmootherConfig::relax, relaxation.hpp:20): with BASELINE's
  omega^2 and lambda^2 the horizontal coupling dominates the mass term on every level, and
  undamped (relax = 1) block Jacobi leaves the horizontal checkerboard modes undamped
  (amplification -> -1), which makes the PCG iteration count grow like 1/h (41, 79, 155,
  307 iterations for n = 32..256); relax = 0.8 gives 14 iterations at every size;
* factorised profiles (profiles.hpp:196-210) chosen so the reference's hatted
  assembly (discretization.hpp:144-184) yields ``-w^2 (dxx + dyy) u - dzz u + lam^2 u``:
  beta_r = lam^2, beta_s = h_T; alpha_s_r = 1, alpha_s_s(edge) = (h_T + h_T')/2;
  alpha_r_r = 1/w^2, alpha_r_s = h_T; xi = 0.
"""
from __future__ import annotations

import dataclasses
import math
from fractions import Fraction

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_SEEDMUL = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, idx: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser of ``seed*C1 + (idx+1)*golden`` (uint64 wrap-around)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) * _SEEDMUL + (idx.astype(np.uint64) + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1(seed: int, idx: np.ndarray) -> np.ndarray:
    """Exact uniform values on [-1, 1): m * 2^-52 - 1 with m the top 53 bits."""
    m = splitmix64(seed, idx) >> np.uint64(11)
    return m.astype(np.float64) * (2.0 ** -52) - 1.0


def _exact_sum_m(seed: int, n: int, chunk: int = 1 << 24) -> int:
    """Exact integer sum of the 53-bit mantissa integers m over indices [0, n)."""
    total = 0
    for lo in range(0, n, chunk):
        idx = np.arange(lo, min(n, lo + chunk), dtype=np.uint64)
        m = splitmix64(seed, idx) >> np.uint64(11)
        hi = (m >> np.uint64(26)).sum(dtype=np.uint64)  # < 2^27 each
        lo_ = (m & np.uint64((1 << 26) - 1)).sum(dtype=np.uint64)
        total += (int(hi) << 26) + int(lo_)
    return total


def rhs_mean(seed: int, n: int) -> float:
    """Correctly rounded mean of the n uniform values (exact rational arithmetic)."""
    s = _exact_sum_m(seed, n)
    return float(Fraction(s - n * (1 << 52), n * (1 << 52)))


def tile_m_sum(seed: int, nx: int, ny: int, nz: int, x0: int, y0: int, lnx: int, lny: int) -> int:
    """Exact integer sum of the mantissa integers m over one tile (all levels)."""
    total = 0
    xs = np.arange(x0, x0 + lnx, dtype=np.uint64)
    ys = np.arange(y0, y0 + lny, dtype=np.uint64)
    for k in range(nz):
        idx = (np.uint64(k) * np.uint64(ny) + ys)[:, None] * np.uint64(nx) + xs[None, :]
        m = splitmix64(seed, idx) >> np.uint64(11)
        total += (int((m >> np.uint64(26)).sum(dtype=np.uint64)) << 26) + \
            int((m & np.uint64((1 << 26) - 1)).sum(dtype=np.uint64))
    return total


def mean_from_m_sum(s: int, n: int) -> float:
    """Correctly rounded mean of n uniform values whose mantissa integers sum to s."""
    return float(Fraction(s - n * (1 << 52), n * (1 << 52)))


def rhs_x_fastest(seed: int, nx: int, ny: int, nz: int, x0: int = 0, y0: int = 0,
                  lnx: int | None = None, lny: int | None = None,
                  gnx: int | None = None, gny: int | None = None,
                  mean: float | None = None) -> np.ndarray:
    """RHS tile in device order [k][y][x] (float64), mean of the GLOBAL field removed.

    (nx, ny) is the global grid unless gnx/gny are given; the tile is
    [x0, x0+lnx) x [y0, y0+lny).  Global linear index = (k*ny + y)*nx + x.  `mean` (the
    global mean, e.g. from all-gathered tile_m_sum values) skips the global pass.
    """
    gnx = nx if gnx is None else gnx
    gny = ny if gny is None else gny
    lnx = gnx if lnx is None else lnx
    lny = gny if lny is None else lny
    if mean is None:
        mean = rhs_mean(seed, gnx * gny * nz)
    out = np.empty((nz, lny, lnx), dtype=np.float64)
    xs = np.arange(x0, x0 + lnx, dtype=np.uint64)
    for k in range(nz):
        ys = np.arange(y0, y0 + lny, dtype=np.uint64)
        idx = (np.uint64(k) * np.uint64(gny) + ys)[:, None] * np.uint64(gnx) + xs[None, :]
        out[k] = uniform_pm1(seed, idx) - mean
    return out


def x_fastest_to_k_fastest(a: np.ndarray) -> np.ndarray:
    """[k][y][x] -> reference Field order (column-major n_r x n_cells, k fastest)."""
    nz, ny, nx = a.shape
    return np.ascontiguousarray(a.reshape(nz, ny * nx).T).reshape(-1)


def k_fastest_to_x_fastest(a: np.ndarray, nx: int, ny: int, nz: int) -> np.ndarray:
    return np.ascontiguousarray(a.reshape(ny * nx, nz).T).reshape(nz, ny, nx)


def vertical_faces(nz: int, depth: float = 1.0, grading: str = "uniform",
                   ratio: float = 1.0) -> np.ndarray:
    """Face heights z_0=0 < ... < z_nz=depth (flat analogue of geometry.hpp:294-327)."""
    if nz < 1:
        raise ValueError("vertical grid needs at least one cell")
    if not depth > 0:
        raise ValueError("vertical depth must be positive")
    z = np.empty(nz + 1, dtype=np.float64)
    if grading == "uniform" or (grading == "geometric" and ratio == 1.0):
        for k in range(nz + 1):
            z[k] = depth * float(k) / float(nz)
    elif grading == "quadratic":
        for k in range(nz + 1):
            t = float(k) / float(nz)
            z[k] = depth * (t * t)
    elif grading == "geometric":
        if not ratio > 0:
            raise ValueError("grading ratio must be positive")
        dr0 = depth * (ratio - 1.0) / (math.pow(ratio, float(nz)) - 1.0)
        z[0] = 0.0
        dr = dr0
        for k in range(nz):
            z[k + 1] = z[k] + dr
            dr *= ratio
    else:
        raise ValueError(f"unknown grading {grading!r}")
    z[0] = 0.0
    z[nz] = depth
    return z


def horizontal_profile(kind: str, seed: int, nx: int, ny: int, amp: float = 0.1,
                       sigma: float = 0.5) -> np.ndarray:
    """Per-cell horizontal profile h_T (cell (i,j) at j*nx+i)."""
    n = nx * ny
    if kind == "const":
        return np.ones(n, dtype=np.float64)
    idx = np.arange(n, dtype=np.uint64)
    if kind == "uniform":
        return 1.0 + amp * uniform_pm1(seed, idx)
    if kind == "lognormal":
        # Box-Muller from two independent streams of the same counter.
        u1 = (splitmix64(seed, 2 * idx) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        u2 = (splitmix64(seed, 2 * idx + np.uint64(1)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        g = np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)
        return np.exp(sigma * g)
    raise ValueError(f"unknown profile kind {kind!r}")


@dataclasses.dataclass
class Problem:
    """Inputs of one solve: grid, factorised profiles (profiles.hpp:196-210), omega, MG config."""
    nx: int
    ny: int
    nz: int
    hx: float
    hy: float
    z_faces: np.ndarray
    beta_r: np.ndarray
    alpha_s_r: np.ndarray
    alpha_r_r: np.ndarray
    beta_s: np.ndarray
    alpha_r_s: np.ndarray
    alpha_s_s: np.ndarray
    omega: float
    relax: float = 1.0
    prolongation: int = 0  # 0 linear, 1 injection
    restriction: int = 1   # 0 summation, 1 transpose (R = P^T keeps the V-cycle SPD for PCG)
    nu_pre: int = 1
    nu_post: int = 1
    depth: int = 0
    agglomerate: int = 0  # global column count at or below which a decomposed run replicates levels
    tol: float = 1e-8
    rhs_seed: int = 0
    name: str = ""
    xi_r_r: np.ndarray | None = None  # vertical advection (nz+1), None = xi == 0
    xi_r_s: np.ndarray | None = None  # (nx*ny)
    # coefficient storage: "factorized" (the profiles above), "partial" (dense["alpha_r"]
    # replaces alpha_r: MixedProfileSet) or "full" (dense ProfileSet, see dense_profiles)
    coef: str = "factorized"
    dense: dict | None = None

    @property
    def n_dof(self) -> int:
        return self.nx * self.ny * self.nz

    def rhs(self) -> np.ndarray:
        """Global RHS in device order [k][y][x]."""
        return rhs_x_fastest(self.rhs_seed, self.nx, self.ny, self.nz)

    def mg_kwargs(self) -> dict:
        return dict(relax=self.relax, prolongation=self.prolongation,
                    restriction=self.restriction, nu_pre=self.nu_pre, nu_post=self.nu_post,
                    depth=self.depth, agglomerate=self.agglomerate)


def edge_profile(h: np.ndarray, nx: int, ny: int) -> np.ndarray:
    """alpha_s_s(edge) = (h_T + h_T')/2: east edges (c, c+x) then north edges (c, c+y)."""
    hh = h.reshape(ny, nx)
    east = 0.5 * (hh + np.roll(hh, -1, axis=1))
    north = 0.5 * (hh + np.roll(hh, -1, axis=0))
    return np.concatenate([east.reshape(-1), north.reshape(-1)])


def dense_profiles(P: Problem, eps: float = 0.1, seed: int = 7) -> dict:
    """A genuinely non-separable ProfileSet (profiles.hpp:182-192) near P's factorised one:
    each dense entry is the outer product of P's vertical and horizontal factors times
    (1 + eps * U[-1, 1)) drawn per (level, cell/edge).  Arrays in the reference's Matrix order
    (k fastest): shape (n_cells or n_edges, rows), C-contiguous."""
    rng = np.random.default_rng(seed)
    nc = P.nx * P.ny

    def outer(vert, horiz):
        d = np.outer(np.asarray(horiz, dtype=np.float64), np.asarray(vert, dtype=np.float64))
        return np.ascontiguousarray(d * (1.0 + eps * rng.uniform(-1.0, 1.0, d.shape)))

    out = dict(beta=outer(P.beta_r, P.beta_s), alpha_s=outer(P.alpha_s_r, P.alpha_s_s),
               alpha_r=outer(P.alpha_r_r, P.alpha_r_s), xi_r=None)
    if P.xi_r_r is not None:
        out["xi_r"] = outer(P.xi_r_r, P.xi_r_s)
    assert out["beta"].shape == (nc, P.nz) and out["alpha_s"].shape == (2 * nc, P.nz)
    return out


def with_coefficients(P: Problem, coef: str, eps: float = 0.1, seed: int = 7) -> Problem:
    """Copy of P with partial ("partial": dense alpha_r) or full ("full") coefficients."""
    assert coef in ("factorized", "partial", "full")
    Q = dataclasses.replace(P)
    Q.coef = coef
    Q.dense = None if coef == "factorized" else dense_profiles(P, eps, seed)
    Q.name = f"{P.name}-{coef}"
    return Q


def make_problem(nx: int, ny: int, nz: int, *, omega2: float, lambda2: float,
                 grading: str = "uniform", ratio: float = 1.0, profile: str = "const",
                 profile_seed: int = 1, profile_amp: float = 0.1, profile_sigma: float = 0.5,
                 h: float | None = None, depth: int = 0, nu: int = 1, tol: float = 1e-8,
                 rhs_seed: int = 0, prolongation: int = 0, restriction: int = 1,
                 relax: float = 0.8, name: str = "") -> Problem:
    h = 1.0 / nx if h is None else h
    z = vertical_faces(nz, 1.0, grading, ratio)
    hT = horizontal_profile(profile, profile_seed, nx, ny, profile_amp, profile_sigma)
    omega = math.sqrt(omega2)
    return Problem(
        nx=nx, ny=ny, nz=nz, hx=h, hy=h, z_faces=z,
        beta_r=np.full(nz, lambda2), alpha_s_r=np.ones(nz), alpha_r_r=np.full(nz + 1, 1.0 / omega2),
        beta_s=hT.copy(), alpha_r_s=hT.copy(), alpha_s_s=edge_profile(hT, nx, ny),
        omega=omega, relax=relax, nu_pre=nu, nu_post=nu, depth=depth, tol=tol, rhs_seed=rhs_seed,
        prolongation=prolongation, restriction=restriction, name=name)


def baseline_config(i: int, **over) -> Problem:
    """BASELINE.json configs (1-based).  Config 4 is config 3 per GPU tile."""
    if i == 1:
        kw = dict(nx=32, ny=32, nz=32, omega2=1e-2, lambda2=1e-4, depth=4, nu=1, tol=1e-8,
                  name="cfg1_32x32x32")
    elif i == 2:
        kw = dict(nx=512, ny=512, nz=128, omega2=1e-2, lambda2=1e-4, grading="quadratic",
                  profile="uniform", profile_seed=1, profile_amp=0.1, depth=7, nu=1,
                  name="cfg2_512x512x128")
    elif i == 3:
        kw = dict(nx=1024, ny=1024, nz=128, omega2=1e-3, lambda2=1e-4, grading="quadratic",
                  depth=8, nu=1, tol=1e-8, name="cfg3_1024x1024x128")
    elif i == 5:
        kw = dict(nx=4096, ny=4096, nz=64, omega2=1e-5, lambda2=1e-6, grading="geometric",
                  ratio=1.1, profile="lognormal", profile_seed=2, profile_sigma=0.5, depth=10,
                  nu=2, tol=1e-10, name="cfg5_4096x4096x64")
    else:
        raise ValueError("configs are 1, 2, 3, 5 (4 is 3 per GPU)")
    kw.update(over)
    nx, ny, nz = kw.pop("nx"), kw.pop("ny"), kw.pop("nz")
    return make_problem(nx, ny, nz, **kw)


def parity_problem(name: str) -> Problem:
    """The solves pinned by oracle goldens at BASELINE.json's stated sizes
    (tests/golden/oracle_<name>_pcg.json, made by tests/golden/make_golden_large.py)."""
    if name == "cfg2":
        return baseline_config(2)
    if name == "cfg3":
        return baseline_config(3)
    if name == "cfg4s":  # config 4's strong-scaling problem: 9 levels to a global 8x8
        return baseline_config(3, nx=2048, ny=2048, depth=9, name="cfg4s_2048x2048x128")
    if name == "cfg5t":  # a 2048^2 tile of config 5 (its h = 1/4096), 9 levels to 8x8
        return baseline_config(5, nx=2048, ny=2048, depth=9, h=1.0 / 4096,
                               name="cfg5t_2048x2048x64")
    raise ValueError(f"unknown parity problem {name!r}")
