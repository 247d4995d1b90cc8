"""The reference's own test problem set up on the host by test infrastructure (SURVEY.md §8(f) rank 3:
icosahedral grids + balanced-flow profiles): oracle/icosa_setup.cpp (test infrastructure) restates
build_icosahedral_hierarchy, build_vertical_grid, the balanced-flow profiles, courant_default
and build_hierarchy_coefficients' assemble / restrict loop.

Pinned against the REFERENCE ITSELF, twice, through fixtures its own code wrote:
  * tests/golden/ref_icosa_pin.bin (oracle/build_ref.py): three levels, 8 geometric vertical
    cells, advection -- omega, every neighbour / edge table and every hatted coefficient;
  * tests/golden/profile_io/ (oracle/build_ref_profile_io.py): the level-1 grid's centres and
    fingerprint, its full and factorised balanced-flow profiles, and the profile files the
    reference's save_profiles wrote from them -- re-written here byte for byte.
Host code only (the setup is test infrastructure; the product takes the tables through tpmg_hier_create_generic); the device side of this problem is in test_ref_pin_gpu.py (source="setup").
"""
import filecmp
import os

import numpy as np
import pytest

import icosa  # oracle/: the reference's own icosahedral problem (test infrastructure)
from paper_1408_2981_b200 import tpmg
from test_profile_io import GOLD, _meta
from test_ref_pin import load


@pytest.fixture(scope="module")
def R():
    return load()


@pytest.fixture(scope="module")
def ico_pin(R):
    return icosa.Icosahedral(2, int(R["nr"][0]), 80.0 / 6371.229, "geometric", 1.2, 0.022, 10.0,
                            True)


def test_omega_is_the_references(R, ico_pin):
    assert ico_pin.omega == R["omega"][0]
    assert ico_pin.n_levels == int(R["n_levels"][0])


@pytest.mark.parametrize("level", [0, 1, 2])
def test_grid_tables_bitwise(R, ico_pin, level):
    lv = ico_pin.level(level)
    assert lv["n_cells"] == 20 * 4 ** level and lv["n_edges"] == 30 * 4 ** level
    assert np.array_equal(lv["neighbors"].ravel(), R["nbr%d" % level].ravel())
    assert np.array_equal(lv["cell_edges"].ravel(), R["cedge%d" % level].ravel())
    # sphere: total area 4 pi, centres on the unit sphere
    assert abs(lv["areas"].sum() - 4 * np.pi) <= 1e-12
    assert np.allclose(np.linalg.norm(lv["centers"], axis=1), 1.0, atol=1e-15)


@pytest.mark.parametrize("level", [0, 1, 2])
def test_hatted_coefficients_bitwise(R, ico_pin, level):
    h = ico_pin.hatted(level)
    for k in ("bh", "ah", "xh", "sh"):
        assert np.array_equal(h[k], R[k + str(level)]), (k, level)
    for k in ("bv", "sv", "av", "xv"):
        assert np.array_equal(h[k], R[k]), k


def test_level1_fixture_profiles_and_fingerprint():
    m = _meta()
    ico = icosa.Icosahedral(1, 4, 0.0126)  # tests/test_profile_io.cpp:40-42 of the reference
    lv = ico.level(1)
    assert np.array_equal(lv["centers"].ravel(), m["centers"])
    assert lv["fingerprint"] == int(m["fingerprint"].view(np.uint64)[0])
    for kind, pre in ((tpmg.PROFILE_FULL, "full"), (tpmg.PROFILE_FACTORIZED, "fac")):
        for name, a in ico.profiles(kind).items():
            assert np.array_equal(a.ravel(), m[f"{pre}.{name}"]), (pre, name)


@pytest.mark.parametrize("kind,pre", [(tpmg.PROFILE_FULL, "full"), (tpmg.PROFILE_FACTORIZED, "fac")])
@pytest.mark.parametrize("enc,suf", [("decimal", "dec"), ("base64-f64le", "b64")])
def test_profile_files_byte_identical_to_the_references(tmp_path, kind, pre, enc, suf):
    """Grid -> balanced-flow profiles -> save_profiles, end to end, equals the reference's file."""
    ico = icosa.Icosahedral(1, 4, 0.0126)
    out = tmp_path / "p.json"
    tpmg.save_profile_arrays(str(out), ico.profile_grid(), kind, ico.profiles(kind), enc)
    assert filecmp.cmp(str(out), os.path.join(GOLD, f"{pre}_{suf}.json"), shallow=False)


def test_without_advection_and_separability():
    ico = icosa.Icosahedral(1, 6, 0.0126, advection=False)
    fac = ico.profiles(tpmg.PROFILE_FACTORIZED)
    full = ico.profiles(tpmg.PROFILE_FULL)
    assert not fac["xi_r_r"].any() and not full["xi_r"].any()
    # epsilon = (N/N*)^2 - 1 > 0 at N = 0.022: the full profiles are genuinely non-separable,
    # and factorise exactly only at N = N* (profiles.hpp:125-127)
    assert ico.epsilon > 0
    dense = np.outer(fac["beta_s"], fac["beta_r"])
    assert not np.allclose(dense, full["beta"], rtol=1e-12)


def test_courant_default_and_deterministic_geometry():
    a, b = icosa.Icosahedral(3, 2, 0.01), icosa.Icosahedral(3, 2, 0.01)
    la, lb = a.level(3), b.level(3)
    assert la["fingerprint"] == lb["fingerprint"]
    # omega = 10 x mean great-circle edge length of the finest grid
    lv = a.level(3)
    assert a.omega > 0 and a.mu_dt > 0
    nbr = lv["neighbors"]
    assert (nbr >= 0).all() and (nbr < lv["n_cells"]).all()
    # every edge shared by exactly two cells
    counts = np.bincount(lv["cell_edges"].ravel(), minlength=lv["n_edges"])
    assert (counts == 2).all()


@pytest.mark.parametrize("kw,exc", [(dict(levels=10), icosa.IcosaError),
                                    (dict(n_r=0), icosa.IcosaError),
                                    (dict(depth=0.0), icosa.IcosaError),
                                    (dict(buoyancy_frequency=0.001), icosa.IcosaError)])
def test_configuration_errors(kw, exc):
    """geometry.hpp:266-267, 298-300; profiles.hpp:136-137."""
    args = dict(levels=1, n_r=4, depth=0.0126)
    args.update(kw)
    with pytest.raises(exc):
        icosa.Icosahedral(**args)
