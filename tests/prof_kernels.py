"""Profiling driver (run under ncu on the GPU box): each finest-level hot-path kernel of
BASELINE config 3 a few times through tpmg_time_kernel.  Not a pytest file."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1408_2981_b200 import synth, tpmg  # noqa: E402

KERNELS = {"apply": tpmg.K_APPLY, "jacobi": tpmg.K_JACOBI, "jacobi0": tpmg.K_JACOBI_ZERO,
           "rr": tpmg.K_RESID_RESTRICT, "prolong": tpmg.K_PROLONG_ADD, "resid": tpmg.K_RESIDUAL,
           "post": tpmg.K_PCG_POSTSWEEP, "rupdate": tpmg.K_PCG_RUPDATE, "ap": tpmg.K_PCG_DIRECTION}


def main():
    cfg = int(os.environ.get("TPMG_CFG", "3"))
    names = sys.argv[1:] or list(KERNELS)
    reps = int(os.environ.get("TPMG_REPS", "2"))
    ctx = tpmg.Context()
    over = {k.lower(): int(os.environ["TPMG_" + k]) for k in ("NX", "NY", "DEPTH")
            if "TPMG_" + k in os.environ}
    P = synth.baseline_config(cfg, **over)
    if os.environ.get("TPMG_COEF", "factorized") != "factorized":
        P = synth.with_coefficients(P, os.environ["TPMG_COEF"])
    h = tpmg.Hierarchy(ctx, P)
    for n in names:
        ms = h.time_kernel(KERNELS[n], h.finest, reps=reps)
        print(f"{n}: {ms:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
