"""Live per-launch durations of the finest-level PCG kernels and of the dot reductions inside
PCG solves (tpmg_kernel_probe), plus the solve time.  Profiling driver, not a pytest file.

    TPMG_CFG=3 [TPMG_DEBUG_TIMING=1] python tests/prof_probes.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1408_2981_b200 import synth, tpmg  # noqa: E402

NAMES = {tpmg.K_PCG_DIRECTION: "direction+Ap", tpmg.K_PCG_RUPDATE: "r-update pre-sweep",
         tpmg.K_PCG_POSTSWEEP: "post-sweep r.z", tpmg.K_RESID_RESTRICT: "resid+restrict (finest)",
         tpmg.K_PROLONG_ADD: "prolong (finest)", tpmg.K_REDUCE: "reduce (last of each iteration)"}


def main():
    P = synth.baseline_config(int(os.environ.get("TPMG_CFG", "3")))
    ctx = tpmg.Context()
    h = tpmg.Hierarchy(ctx, P)
    f = h.field().upload(P.rhs())
    x = h.field()
    h.kernel_probe(True)
    for _ in range(2):
        tpmg.pcg_solve(h, f, x, P.tol, 200)
    h.kernel_probe(True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.ExternalStream(ctx.stream_handle())
    n = 3
    e0.record(st)
    for _ in range(n):
        res = tpmg.pcg_solve(h, f, x, P.tol, 200)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{P.name}: {res.iterations} iterations, {ms:.2f} ms per solve")
    for kid, name in NAMES.items():
        tot, cnt = h.kernel_probe_read(kid)
        if cnt:
            print(f"  {name:32s} {cnt:4d} launches  {tot / cnt * 1e3:8.1f} us/launch  "
                  f"{tot / n:7.2f} ms/solve")


if __name__ == "__main__":
    main()
