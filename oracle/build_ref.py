"""TEST INFRASTRUCTURE: compile the reference's own headers (read in place under
/root/reference/proj/include, never copied) against oracle/eigen_shim into oracle/_ref/, run
the driver, and refresh the committed golden fixture tests/golden/ref_icosa_pin.bin from it.

Only possible where /root/reference exists (the build container); the GPU box uses the
committed fixture.  Recipe:  python oracle/build_ref.py
"""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_INC = "/root/reference/proj/include"
OUT = os.path.join(HERE, "_ref")


def main() -> int:
    if not os.path.isdir(REF_INC):
        print("reference sources not present; keeping the committed fixture")
        return 0
    os.makedirs(OUT, exist_ok=True)
    exe = os.path.join(OUT, "ref_driver")
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", os.path.join(HERE, "eigen_shim"),
           "-I", REF_INC, os.path.join(HERE, "ref_driver.cpp"), "-o", exe]
    subprocess.run(cmd, check=True)
    data = os.path.join(OUT, "ref_pin.bin")
    subprocess.run([exe, data], check=True)
    # the drop-in adapter driver: the reference's own objects handed to the device through
    # include/tpmg_b200_ref.hpp (run on the GPU box by tests/test_ref_adapter_gpu.py)
    lib_dir = os.path.join(ROOT, "paper_1408_2981_b200")
    if os.path.exists(os.path.join(lib_dir, "libtpmg_b200.so")):
        cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", os.path.join(HERE, "eigen_shim"),
               "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
               os.path.join(HERE, "ref_adapter_driver.cpp"), "-o",
               os.path.join(OUT, "ref_adapter_driver"), "-L", lib_dir, "-ltpmg_b200",
               "-Wl,-rpath,$ORIGIN/../../paper_1408_2981_b200"]
        subprocess.run(cmd, check=True)
    golden = os.path.join(ROOT, "tests", "golden", "ref_icosa_pin.bin")
    os.makedirs(os.path.dirname(golden), exist_ok=True)
    shutil.copyfile(data, golden)
    print("reference outputs:", data, "->", golden)
    return 0


if __name__ == "__main__":
    sys.exit(main())
