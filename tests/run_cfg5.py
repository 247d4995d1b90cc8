"""BASELINE config 5 (4096²×64, extreme anisotropy: ω²=1e-5, λ²=1e-6, lognormal horizontal
profile σ=0.5, geometric grading 1.1, V(2,2), tol 1e-10) solved on ONE B200 — the config the
reference quotes for 8 GPUs; 1.07e9 unknowns fit in one GPU's HBM.  Prints iterations, time and
the true residual.  Profiling/validation driver, not a pytest file."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1408_2981_b200 import synth, tpmg  # noqa: E402


def main():
    P = synth.baseline_config(5)
    ctx = tpmg.Context()
    t0 = time.perf_counter()
    h = tpmg.Hierarchy(ctx, P)
    f = h.field().upload(P.rhs())
    x = h.field()
    print(f"setup {time.perf_counter() - t0:.1f} s, {h.n_levels} levels, "
          f"{torch.cuda.max_memory_allocated() / 2**30:.1f} GiB torch / "
          f"{(torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 2**30:.1f} GiB used",
          flush=True)
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = tpmg.pcg_solve(h, f, x, P.tol, 300)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"solve {rep}: status {res.status}, {res.iterations} iterations, {dt * 1e3:.1f} ms, "
              f"{P.n_dof * res.iterations / dt / 1e9:.2f} GDOF/s, rel res "
              f"{res.history[-1] / res.history[0]:.3e}", flush=True)
    # true residual |f - A x| / |f| through the library's own operator
    r = h.field()
    tpmg.residual(h, f, x, r)
    rel = (tpmg.dot(h, r, r) / tpmg.dot(h, f, f)) ** 0.5
    print(f"true |f - A x| / |f| = {rel:.3e}", flush=True)
    print("history", np.array2string(res.history[:6] / res.history[0], precision=3), "...")


if __name__ == "__main__":
    main()
