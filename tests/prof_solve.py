"""Profiling driver: BASELINE config 3 PCG solves through the public API (one warm-up solve,
then TPMG_SOLVES timed solves).  Run under `ncu --metrics gpu__time_duration.sum` on the GPU
box for the per-launch list.  Not a pytest file."""
import os
import sys

# ncu / CUPTI do not see kernels inside conditional graph bodies: profile the host PCG loop
os.environ.setdefault("TPMG_DEVLOOP", "0")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1408_2981_b200 import synth, tpmg  # noqa: E402


def main():
    P = synth.baseline_config(int(os.environ.get("TPMG_CFG", "3")))
    if os.environ.get("TPMG_COEF", "factorized") != "factorized":
        P = synth.with_coefficients(P, os.environ["TPMG_COEF"])
    ctx = tpmg.Context()
    h = tpmg.Hierarchy(ctx, P)
    h.set_use_graphs(os.environ.get("TPMG_GRAPHS", "1") == "1")
    f = h.field().upload(P.rhs())
    x = h.field()
    for i in range(1 + int(os.environ.get("TPMG_SOLVES", "1"))):
        res = tpmg.pcg_solve(h, f, x, P.tol, 200)
        print(f"solve {i}: {res.iterations} iterations, {res.seconds * 1e3:.1f} ms wall", flush=True)


if __name__ == "__main__":
    main()
