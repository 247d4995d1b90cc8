"""Cases shared by oracle/build_ref_profile_io.py (which runs the REFERENCE's load_profiles /
save_profiles on them to record the expected outcomes under tests/golden/profile_io/) and
tests/test_profile_io.py (which replays them through the library's reader and writer).

Every malformed file is derived deterministically from a golden file the reference wrote, by a
text edit, so the fixture holds only the reference's outputs and its verdicts.
"""
import base64
import re
import struct

import numpy as np


def echo_values() -> np.ndarray:
    """Doubles exercising every branch of the reference writer's number formatting (nlohmann
    dump_float): integral values, the decimal / scientific switch at exponents -5/-4 and 15/16,
    subnormals, extremes, signed zero, and random doubles across the whole exponent range."""
    edge = [0.0, -0.0, 1.0, -1.0, 0.5, 0.1, 0.2, 0.3, 1.0 / 3.0, 2.0 / 3.0, 123.0, 1e15, 1e16,
            9.999999999999998e15, 1e17, 123456789012345.0, 1234567890123456.0, 1e-4, 1e-5,
            1.5e-4, 1.5e-5, 0.00012345, 1.2345e-5, 5e-324, 2.2250738585072014e-308,
            1.7976931348623157e308, 1e308, 1e100, 1e-100, 4.35, 0.07, 100.0, 1e21, 1e22,
            2.0 ** 53, 2.0 ** 53 + 2, 2.0 ** -1074 * 3, 6.02214076e23, 1.602176634e-19,
            299792458.0, 3.141592653589793, 2.718281828459045, 9.81, 7.2921e-5, 6371229.0]
    rng = np.random.default_rng(20260119)
    mant = rng.uniform(1.0, 10.0, 600)
    expo = rng.integers(-30, 31, 600)
    sign = np.where(rng.random(600) < 0.5, -1.0, 1.0)
    rand = sign * mant * 10.0 ** expo
    bits = rng.integers(0, 2 ** 62, 200, dtype=np.int64).view(np.float64)  # raw bit patterns
    bits = bits[np.isfinite(bits)]
    return np.concatenate([np.array(edge), rand, bits])


def _sub_array_text(text: str, name: str, fn) -> str:
    """Apply fn to the body of JSON array / string `name` (as the reference writer laid it out)."""
    m = re.search(r'"%s": (\[[^\]]*\]|"[^"]*")' % re.escape(name), text)
    assert m, name
    return text[:m.start(1)] + fn(m.group(1)) + text[m.end(1):]


def _first_number(body: str, repl: str) -> str:
    return re.sub(r"-?\d[\d.eE+-]*", repl, body, count=1)


def _b64_with_nan(body: str) -> str:
    raw = bytearray(base64.b64decode(body.strip('"')))
    raw[8 * 5:8 * 6] = struct.pack("<d", float("nan"))
    return '"' + base64.b64encode(bytes(raw)).decode() + '"'


def _drop_last(body: str) -> str:
    return re.sub(r",\n\s*[^,\n]+\n(\s*)\]$", r"\n\1]", body)


def _dup_first(body: str) -> str:
    return re.sub(r"^\[\n(\s*)([^,\n]+),", r"[\n\1\2,\n\1\2,", body, count=1)


# name -> (golden source file, n_r the loader is given, text mutation)
MUTATIONS = {
    "as_written": ("full_dec.json", 4, lambda t: t),
    "as_written_b64": ("fac_b64.json", 4, lambda t: t),
    "n_r_mismatch": ("full_dec.json", 5, lambda t: t),
    "fingerprint_changed": ("full_dec.json", 4,
                            lambda t: re.sub(r'("fingerprint": ")(.)', lambda m: m.group(1) + (
                                "0" if m.group(2) != "0" else "1"), t, count=1)),
    "fingerprint_missing": ("fac_dec.json", 4, lambda t: re.sub(r'\s*"fingerprint": "[0-9a-f]+",', "", t)),
    "level_mismatch": ("full_dec.json", 4, lambda t: t.replace('"level": 1', '"level": 2')),
    "level_missing": ("full_dec.json", 4, lambda t: t.replace('"level": 1,', "")),
    "n_r_as_float": ("fac_dec.json", 4, lambda t: t.replace('"n_r": 4', '"n_r": 4.0')),
    "nan_base64": ("full_b64.json", 4, lambda t: _sub_array_text(t, "beta", _b64_with_nan)),
    "null_decimal": ("full_dec.json", 4, lambda t: _sub_array_text(
        t, "beta", lambda b: _first_number(b, "null"))),
    "nan_token": ("full_dec.json", 4, lambda t: _sub_array_text(
        t, "alpha_r", lambda b: _first_number(b, "NaN"))),
    "infinity_token": ("fac_dec.json", 4, lambda t: _sub_array_text(
        t, "beta_s", lambda b: _first_number(b, "Infinity"))),
    "overflow_number": ("fac_dec.json", 4, lambda t: _sub_array_text(
        t, "beta_s", lambda b: _first_number(b, "1e400"))),
    "string_entry": ("fac_dec.json", 4, lambda t: _sub_array_text(
        t, "alpha_s_s", lambda b: _first_number(b, '"1.0"'))),
    "bool_entry": ("fac_dec.json", 4, lambda t: _sub_array_text(
        t, "xi_r_s", lambda b: _first_number(b, "true"))),
    "short_array": ("full_dec.json", 4, lambda t: _sub_array_text(t, "alpha_r", _drop_last)),
    "long_array": ("fac_dec.json", 4, lambda t: _sub_array_text(t, "beta_r", _dup_first)),
    "missing_array": ("fac_dec.json", 4, lambda t: t.replace('"xi_r_s"', '"xi_r_x"')),
    "b64_missing_array": ("full_b64.json", 4, lambda t: t.replace('"alpha_s"', '"alpha_z"')),
    "b64_bad_length": ("full_b64.json", 4, lambda t: _sub_array_text(
        t, "xi_r", lambda b: b[:-5] + '"')),
    "b64_bad_char": ("fac_b64.json", 4, lambda t: _sub_array_text(
        t, "beta_s", lambda b: b[:3] + "!" + b[4:])),
    "b64_as_decimal": ("fac_b64.json", 4, lambda t: t.replace('"encoding": "base64-f64le",', "")),
    "decimal_as_b64": ("fac_dec.json", 4, lambda t: t.replace(
        '"format_version"', '"encoding": "base64-f64le",\n "format_version"')),
    "unknown_encoding": ("fac_dec.json", 4, lambda t: t.replace(
        '"format_version"', '"encoding": "hex",\n "format_version"')),
    "unknown_kind": ("full_dec.json", 4, lambda t: t.replace('"kind": "full"', '"kind": "partial"')),
    "kind_missing": ("full_dec.json", 4, lambda t: t.replace('"kind": "full",', "")),
    "grid_missing": ("fac_dec.json", 4, lambda t: t.replace('"grid"', '"gird"')),
    "arrays_missing": ("fac_dec.json", 4, lambda t: t.replace('"arrays"', '"arrayz"')),
    "truncated": ("full_dec.json", 4, lambda t: t[:len(t) // 2]),
    "empty_file": ("full_dec.json", 4, lambda t: ""),
    "trailing_garbage": ("fac_dec.json", 4, lambda t: t + "}}garbage"),
    "duplicate_key_last_wins": ("fac_dec.json", 4, lambda t: t.replace(
        '"kind": "factorized"', '"kind": "full",\n "kind": "factorized"')),
    "whitespace_compact": ("fac_dec.json", 4, lambda t: re.sub(r"\s+", "", t.replace(
        "column-major, k fastest", "column-major,k_fastest"))),
}
