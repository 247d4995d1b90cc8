"""A/B kernel timing (profiling helper, not a pytest file): median and min over R rounds of
tpmg_time_kernel on the finest level of a BASELINE config, for the library TPMG_LIB_PATH
selects.  Usage: python tests/ab_kernels.py [kernel ...]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1408_2981_b200 import synth, tpmg  # noqa: E402

KERNELS = {"apply": tpmg.K_APPLY, "jacobi": tpmg.K_JACOBI, "jacobi0": tpmg.K_JACOBI_ZERO,
           "rr": tpmg.K_RESID_RESTRICT, "prolong": tpmg.K_PROLONG_ADD, "resid": tpmg.K_RESIDUAL,
           "ap": tpmg.K_PCG_DIRECTION, "rupdate": tpmg.K_PCG_RUPDATE, "restrict": tpmg.K_RESTRICT,
           "post": tpmg.K_PCG_POSTSWEEP}


def main():
    names = sys.argv[1:] or ["jacobi", "jacobi0", "rr"]
    rounds = int(os.environ.get("TPMG_ROUNDS", "5"))
    reps = int(os.environ.get("TPMG_REPS", "20"))
    ctx = tpmg.Context()
    P = synth.baseline_config(int(os.environ.get("TPMG_CFG", "3")))
    h = tpmg.Hierarchy(ctx, P)
    lib = os.path.basename(os.environ.get("TPMG_LIB_PATH", "product"))
    t = {n: [] for n in names}
    for _ in range(rounds):
        for n in names:
            t[n].append(h.time_kernel(KERNELS[n], h.finest, reps=reps))
    for n in names:
        print(f"{lib:24s} {n:8s} median {statistics.median(t[n]):.4f} ms  min {min(t[n]):.4f} ms",
              flush=True)


if __name__ == "__main__":
    main()
