"""Regenerates the oracle goldens of the PCG solve at BASELINE.json's stated sizes:

  cfg2   512^2 x 128   (config 2's operator and profile, solved with PCG + V(1,1) to 1e-8)
  cfg3   1024^2 x 128  (config 3: the benchmarked solve)
  cfg4s  2048^2 x 128  (config 4's strong-scaling problem, 9 levels to a global 8x8)
  cfg5t  2048^2 x 64   (a tile of config 5 that fits the CPU host: config 5's h = 1/4096,
                        omega^2, lambda^2, lognormal profile sigma 0.5, geometric grading 1.1,
                        V(2,2), tol 1e-10; 9 levels to 8x8)

Each file holds the oracle's residual history as exact hex floats, the iteration count,
the status and two checksums of the iterate: the SHA-256 of its bytes in device order
([k][y][x], float64 little endian) and its sum in the reference's k-fastest order.  The GPU
tests (tests/test_gpu_parity_large.py) require the B200 solve to reproduce them; the oracle
is pinned against the reference itself in tests/test_ref_pin.py.

Run on the CPU host (no GPU needed): ~12 GB of RAM for cfg3, ~25 GB for cfg4s / cfg5t.
    python tests/golden/make_golden_large.py cfg2 cfg3 cfg5t [--threads N]
"""
import argparse
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402

from paper_1408_2981_b200 import synth  # noqa: E402


large_problem = synth.parity_problem


MAX_ITER = {"cfg2": 100, "cfg3": 100, "cfg4s": 100, "cfg5t": 200}


def x_digest(x_fastest: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x_fastest, dtype="<f8").tobytes()).hexdigest()


def main():
    import oracle as O

    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    O.build()
    for name in args.configs:
        P = large_problem(name)
        t0 = time.time()
        h = O.OracleHierarchy.from_problem(P, threads=args.threads)
        f = synth.x_fastest_to_k_fastest(P.rhs())
        x, hist, it, st = h.pcg(f, P.tol, MAX_ITER[name])
        del h, f
        xs = synth.k_fastest_to_x_fastest(x, P.nx, P.ny, P.nz)
        out = {"config": P.name, "nx": P.nx, "ny": P.ny, "nz": P.nz, "tol": P.tol,
               "iterations": it, "status": st, "history_hex": [float(v).hex() for v in hist],
               "x_sha256_device_order": x_digest(xs), "x_sum_hex": float(np.sum(x)).hex(),
               "x_absmax_hex": float(np.max(np.abs(x))).hex(),
               "oracle_seconds": round(time.time() - t0, 1)}
        with open(os.path.join(HERE, f"oracle_{name}_pcg.json"), "w") as fh:
            json.dump(out, fh, indent=1)
        print(name, it, st, hist[-1] / hist[0], f"{time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
