"""BASELINE config 4's strong-scaling problem (2048²×128, 9 levels to a global 8×8) on ONE B200:
the single-GPU reference point for the 2/4/8-GPU strong-scaling runs.  Validation driver, not
a pytest file."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1408_2981_b200 import synth, tpmg  # noqa: E402


def main():
    P = synth.baseline_config(3, nx=2048, ny=2048, depth=9, name="cfg4s_2048x2048x128")
    ctx = tpmg.Context()
    h = tpmg.Hierarchy(ctx, P)
    f = h.field().upload(P.rhs())
    x = h.field()
    print(f"{P.name}: {h.n_levels} levels, "
          f"{(torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 2**30:.1f} GiB used",
          flush=True)
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = tpmg.pcg_solve(h, f, x, P.tol, 300)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"solve {rep}: status {res.status}, {res.iterations} iterations, {dt * 1e3:.1f} ms, "
              f"{P.n_dof * res.iterations / dt / 1e9:.2f} GDOF/s", flush=True)


if __name__ == "__main__":
    main()
