"""TEST INFRASTRUCTURE: compile the reference's own profile_io.hpp (read in place under
/root/reference/proj/include, never copied) against oracle/eigen_shim and the nlohmann json.hpp
vendored in this image into oracle/_ref/ref_profile_io, and record its outputs as the golden
fixtures of tests/test_profile_io.py under tests/golden/profile_io/:

  {full,fac}_{dec,b64}.json   files written by the reference's save_profiles
  meta.bin                    grid centres / sizes / fingerprint and the arrays written
  echo_values.bin, echo.json  number-formatting pin (ref_profile_io echo)
  verdicts.json               the reference's load_profiles outcome on every case of
                              tests/profile_io_cases.py

Only possible where /root/reference exists (the build container).  Recipe:
    python oracle/build_ref_profile_io.py
"""
import glob
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_INC = "/root/reference/proj/include"
GOLD = os.path.join(ROOT, "tests", "golden", "profile_io")


def _nlohmann_dir() -> str:
    hits = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "include",
                                  "**", "nlohmann", "json.hpp"), recursive=True)
    if not hits:
        raise SystemExit("nlohmann/json.hpp not found in this image")
    return os.path.dirname(hits[0])


def main() -> int:
    if not os.path.isdir(REF_INC):
        print("reference sources not present; keeping the committed fixtures")
        return 0
    out = os.path.join(HERE, "_ref")
    os.makedirs(out, exist_ok=True)
    os.makedirs(GOLD, exist_ok=True)
    exe = os.path.join(out, "ref_profile_io")
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I",
                    os.path.join(HERE, "eigen_shim"), "-I", REF_INC, "-I", _nlohmann_dir(),
                    os.path.join(HERE, "ref_profile_io.cpp"), "-o", exe], check=True)
    subprocess.run([exe, "write", GOLD], check=True)

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import profile_io_cases as cases
    vals = cases.echo_values()
    vals.astype("<f8").tofile(os.path.join(GOLD, "echo_values.bin"))
    subprocess.run([exe, "echo", os.path.join(GOLD, "echo_values.bin"),
                    os.path.join(GOLD, "echo.json")], check=True)

    verdicts = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, (src, n_r, mutate) in cases.MUTATIONS.items():
            with open(os.path.join(GOLD, src)) as f:
                text = mutate(f.read())
            path = os.path.join(tmp, name + ".json")
            with open(path, "w") as f:
                f.write(text)
            r = subprocess.run([exe, "load", path, str(n_r)], check=True, capture_output=True,
                               text=True)
            verdicts[name] = r.stdout.strip()
        r = subprocess.run([exe, "load", os.path.join(tmp, "does_not_exist.json"), "4"],
                           check=True, capture_output=True, text=True)
        verdicts["missing_file"] = r.stdout.strip()
    with open(os.path.join(GOLD, "verdicts.json"), "w") as f:
        json.dump(verdicts, f, indent=1, sort_keys=True)
        f.write("\n")
    for k, v in sorted(verdicts.items()):
        print(f"{k:28s} {v}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
