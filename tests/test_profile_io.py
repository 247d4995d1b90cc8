"""Profile files: save_profiles / load_profiles (profile_io.hpp:125-242).

Pinned against the REFERENCE itself: tests/golden/profile_io/ holds files written by the
reference's own save_profiles on its icosahedral level-1 grid and the outcomes of its own
load_profiles on every malformed-file case of profile_io_cases.py (recipe:
oracle/build_ref_profile_io.py).  The library must read the reference's files to the same bits,
write byte-identical files from the same arrays, and classify every bad file as the reference
does.  Then the Cartesian flavour: round trips and the reference's own test cases
(tests/test_profile_io.cpp) on the grids of tpmg_hier_create.  Host code only: no GPU needed,
except the last test, which solves with profiles read from a file.
"""
import json
import os
import struct

import numpy as np
import pytest

import profile_io_cases as cases
from paper_1408_2981_b200 import synth, tpmg
from paper_1408_2981_b200.tpmg import K_FASTEST

GOLD = os.path.join(os.path.dirname(__file__), "golden", "profile_io")
CLASSES = {"ok": None, "shape_error": tpmg.shape_error, "nonfinite_error": tpmg.nonfinite_error,
           "fingerprint_error": tpmg.fingerprint_error, "config_error": tpmg.config_error}


def _meta():
    d, b, o = {}, open(os.path.join(GOLD, "meta.bin"), "rb").read(), 0
    while o < len(b):
        nl = struct.unpack_from("<I", b, o)[0]
        name = b[o + 4:o + 4 + nl].decode()
        o += 4 + nl
        n = struct.unpack_from("<q", b, o)[0]
        d[name] = np.frombuffer(b[o + 8:o + 8 + 8 * n], dtype="<f8").copy()
        o += 8 + 8 * n
    return d


@pytest.fixture(scope="module")
def ref():
    m = _meta()
    nc, ne, nr, level = (int(v) for v in m["sizes"][:4])
    fp = int(m["fingerprint"].view(np.uint64)[0])
    return dict(meta=m, nc=nc, ne=ne, nr=nr, level=level, fp=fp,
                grid=lambda n_r=nr: tpmg.profile_grid("icosahedral", fp, level, n_r, nc, ne))


def _read(name):
    with open(os.path.join(GOLD, name)) as f:
        return f.read()


# ---- pinned against the reference's own writer and reader ----------------------------------------

def test_fingerprint_of_reference_grid(ref):
    """grid_fingerprint (geometry.hpp:335-351) of the reference's centres equals the fingerprint
    the reference computed and wrote into its files."""
    centers = ref["meta"]["centers"].reshape(ref["nc"], 3)
    assert tpmg.grid_fingerprint(centers) == ref["fp"]
    assert json.loads(_read("full_dec.json"))["grid"]["fingerprint"] == "%016x" % ref["fp"]


@pytest.mark.parametrize("kind,pre", [(tpmg.PROFILE_FULL, "full"), (tpmg.PROFILE_FACTORIZED, "fac")])
@pytest.mark.parametrize("enc,suf", [("decimal", "dec"), ("base64-f64le", "b64")])
def test_reads_reference_files_bitwise(ref, kind, pre, enc, suf):
    k, arrays = tpmg.load_profile_arrays(os.path.join(GOLD, f"{pre}_{suf}.json"), ref["grid"]())
    assert k == kind
    for name, a in arrays.items():
        assert np.array_equal(a.ravel(), ref["meta"][f"{pre}.{name}"]), name


@pytest.mark.parametrize("kind,pre", [(tpmg.PROFILE_FULL, "full"), (tpmg.PROFILE_FACTORIZED, "fac")])
@pytest.mark.parametrize("enc,suf", [("decimal", "dec"), ("base64-f64le", "b64")])
def test_writes_reference_bytes(ref, tmp_path, kind, pre, enc, suf):
    """Same arrays, same grid header -> the reference writer's exact bytes (nlohmann dump(1):
    sorted keys, shortest round-trip doubles, one element per line)."""
    g = ref["grid"]()
    shapes = tpmg._profile_shapes(kind, g.n_cells, g.n_edges, g.n_r)
    arrays = {n: ref["meta"][f"{pre}.{n}"].reshape(s)
              for n, s in zip(tpmg.PROFILE_ORDER[kind], shapes)}
    out = tmp_path / "ours.json"
    tpmg.save_profile_arrays(str(out), g, kind, arrays, enc)
    assert out.read_text() == _read(f"{pre}_{suf}.json")


def test_number_formatting_matches_reference(ref, tmp_path):
    """The reference writer's text of ~800 doubles chosen to hit every formatting branch."""
    vals = np.fromfile(os.path.join(GOLD, "echo_values.bin"), dtype="<f8")
    assert np.array_equal(vals, cases.echo_values())
    nr, nc, ne = vals.size, ref["nc"], ref["ne"]
    g = tpmg.profile_grid("icosahedral", ref["fp"], ref["level"], nr, nc, ne)
    z = np.zeros
    arrays = dict(beta_r=vals, alpha_s_r=vals, alpha_r_r=z(nr + 1), xi_r_r=z(nr + 1),
                  beta_s=z(nc), alpha_r_s=z(nc), xi_r_s=z(nc), alpha_s_s=z(ne))
    out = tmp_path / "echo.json"
    tpmg.save_profile_arrays(str(out), g, tpmg.PROFILE_FACTORIZED, arrays, "decimal")
    ours, theirs = out.read_text().splitlines(), _read("echo.json").splitlines()
    bad = [(a, b) for a, b in zip(ours, theirs) if a != b]
    assert not bad and len(ours) == len(theirs), bad[:5]
    k, back = tpmg.load_profile_arrays(os.path.join(GOLD, "echo.json"), g)
    assert np.array_equal(back["beta_r"].view(np.int64), vals.view(np.int64))  # -0.0 included


@pytest.mark.parametrize("case", sorted(cases.MUTATIONS))
def test_error_taxonomy_matches_reference(ref, tmp_path, case):
    """load_profiles' verdict on each malformed file (the reference's, recorded by
    oracle/build_ref_profile_io.py) -- types.hpp:24-58 via tpmg_status."""
    expected = json.loads(_read("verdicts.json"))[case]
    src, n_r, mutate = cases.MUTATIONS[case]
    text = mutate(_read(src))
    if case not in ("as_written", "as_written_b64", "n_r_mismatch"):
        assert text != _read(src), "mutation did not change the file"
    path = tmp_path / f"{case}.json"
    path.write_text(text)
    exc = CLASSES[expected]
    if exc is None:
        tpmg.load_profile_arrays(str(path), ref["grid"](n_r))
    else:
        with pytest.raises(exc):
            tpmg.load_profile_arrays(str(path), ref["grid"](n_r))


def test_missing_file_is_config_error(ref):
    assert json.loads(_read("verdicts.json"))["missing_file"] == "config_error"
    with pytest.raises(tpmg.config_error):
        tpmg.load_profile_arrays("/nonexistent/profile.json", ref["grid"]())


def test_duplicate_key_last_wins(ref, tmp_path):
    src, n_r, mutate = cases.MUTATIONS["duplicate_key_last_wins"]
    p = tmp_path / "dup.json"
    p.write_text(mutate(_read(src)))
    k, _ = tpmg.load_profile_arrays(str(p), ref["grid"]())
    assert k == tpmg.PROFILE_FACTORIZED


# ---- the Cartesian grids of tpmg_hier_create -----------------------------------------------------

def _cfg(xi: bool = False):
    P = synth.make_problem(16, 8, 6, omega2=1e-2, lambda2=1e-3, grading="geometric", ratio=1.2,
                           profile="uniform", profile_seed=5, depth=2, name="io")
    if xi:
        rng = np.random.default_rng(3)
        P.xi_r_r = 0.3 * rng.standard_normal(P.nz + 1)
        P.xi_r_s = P.beta_s.copy()
    return P


@pytest.mark.parametrize("coef", ["factorized", "full"])
@pytest.mark.parametrize("enc", ["decimal", "base64-f64le"])
@pytest.mark.parametrize("xi", [False, True])
def test_cartesian_round_trip_is_bit_exact(tmp_path, coef, enc, xi):
    """tests/test_profile_io.cpp:39-77 on the Cartesian grid."""
    P = synth.with_coefficients(_cfg(xi), coef, eps=0.2) if coef == "full" else _cfg(xi)
    path = str(tmp_path / "p.json")
    tpmg.save_profiles(path, P, enc)
    Q = tpmg.load_profiles(path, P)
    assert Q.coef == coef
    if coef == "full":
        for n in ("beta", "alpha_s", "alpha_r", "xi_r"):
            a, b = P.dense[n], Q.dense[n]
            assert (a is None and b is None) or np.array_equal(a, b), n
    else:
        for n in tpmg.PROFILE_ORDER[tpmg.PROFILE_FACTORIZED]:
            a, b = getattr(P, n), getattr(Q, n)
            assert (a is None and b is None) or np.array_equal(a, b), n
    doc = json.loads(open(path).read())  # plain JSON, readable by any parser
    assert doc["format_version"] == 1 and doc["grid"]["type"] == "cartesian"
    assert (doc["grid"]["nx"], doc["grid"]["ny"], doc["grid"]["n_r"]) == (P.nx, P.ny, P.nz)


def test_cartesian_fingerprint_is_grid_fingerprint_of_the_centres():
    P = _cfg()
    i, j = np.meshgrid(np.arange(P.nx), np.arange(P.ny))
    centers = np.stack([((i + 0.5) * P.hx).ravel(), ((j + 0.5) * P.hy).ravel(),
                        np.zeros(P.nx * P.ny)], axis=1)
    assert tpmg.cartesian_profile_grid(P).fingerprint == tpmg.grid_fingerprint(centers)


def test_cartesian_vertical_shape_mismatch(tmp_path):
    """tests/test_profile_io.cpp:79-88."""
    P = _cfg()
    path = str(tmp_path / "p.json")
    tpmg.save_profiles(path, P)
    Q = synth.make_problem(P.nx, P.ny, P.nz + 1, omega2=1e-2, lambda2=1e-3, depth=2)
    with pytest.raises(tpmg.shape_error):
        tpmg.load_profiles(path, Q)


@pytest.mark.parametrize("other", ["nx", "hx"])
def test_cartesian_fingerprint_mismatch(tmp_path, other):
    """tests/test_profile_io.cpp:90-98: another horizontal grid (cell count or spacing)."""
    P = _cfg()
    path = str(tmp_path / "p.json")
    tpmg.save_profiles(path, P)
    import dataclasses
    Q = dataclasses.replace(P, nx=2 * P.nx) if other == "nx" else dataclasses.replace(P, hx=0.5 * P.hx)
    with pytest.raises(tpmg.fingerprint_error):
        tpmg.load_profiles(path, Q)


@pytest.mark.parametrize("enc", ["decimal", "base64-f64le"])
def test_cartesian_nonfinite(tmp_path, enc):
    """tests/test_profile_io.cpp:100-115: NaN is written (as null in decimal) and rejected on
    load as non-finite."""
    P = synth.with_coefficients(_cfg(), "full", eps=0.2)
    P.dense["beta"][7, 2] = np.nan
    path = str(tmp_path / "p.json")
    tpmg.save_profiles(path, P, enc)
    if enc == "decimal":
        assert "null" in open(path).read()
    with pytest.raises(tpmg.nonfinite_error):
        tpmg.load_profiles(path, P)


def test_cartesian_missing_file_is_config_error():
    with pytest.raises(tpmg.config_error):
        tpmg.load_profiles("/nonexistent/profile.json", _cfg())


# ---- a solve from a profile file ---------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("coef", ["factorized", "full"])
def test_solve_from_profile_file_bitwise(gpu_ctx, oracle_mod, tmp_path, coef):
    """Profiles read back from a file drive the device PCG to the oracle's bits on the original
    profiles (bit-exact round trip + bitwise solver)."""
    base = synth.baseline_config(1)
    P = synth.with_coefficients(base, coef, eps=0.2) if coef == "full" else base
    path = str(tmp_path / "p.json")
    tpmg.save_profiles(path, P, "base64-f64le")
    Q = tpmg.load_profiles(path, synth.baseline_config(1))
    h = tpmg.Hierarchy(gpu_ctx, Q)
    o = oracle_mod.OracleHierarchy.from_problem(P)
    f = synth.x_fastest_to_k_fastest(P.rhs())
    xo, hist_o, it_o, st_o = o.pcg(f, P.tol, 200)
    xg = h.field()
    res = tpmg.pcg_solve(h, h.field().upload(P.rhs()), xg, P.tol, 200)
    assert res.status == st_o == 0 and res.iterations == it_o
    assert np.array_equal(res.history, hist_o)
    assert np.array_equal(xg.download(K_FASTEST), xo)
