"""Per-level kernel times of a BASELINE config (profiling helper, not a pytest file): the
coarse levels are latency-bound, this shows by how much.  python tests/prof_levels.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1408_2981_b200 import synth, tpmg  # noqa: E402

KERNELS = {"jacobi": tpmg.K_JACOBI, "jacobi0": tpmg.K_JACOBI_ZERO, "rr": tpmg.K_RESID_RESTRICT,
           "prolong": tpmg.K_PROLONG_ADD}


def main():
    ctx = tpmg.Context()
    P = synth.baseline_config(int(os.environ.get("TPMG_CFG", "3")))
    h = tpmg.Hierarchy(ctx, P)
    names = sys.argv[1:] or list(KERNELS)
    print("level  " + "  ".join(f"{n:>9s}" for n in names))
    for lv in range(h.finest, -1, -1):
        row = []
        for n in names:
            if n in ("rr", "prolong") and lv == 0:
                row.append("        -")
                continue
            row.append(f"{h.time_kernel(KERNELS[n], lv, reps=20) * 1e3:9.1f}")
        print(f"{lv:5d}  " + "  ".join(row), flush=True)


if __name__ == "__main__":
    main()
