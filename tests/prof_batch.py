"""Timeline of the overlapped end-to-end batch (tpmg_pcg_host_batch) on config 3: memcpy and
kernel spans per stream from CUPTI.  Profiling helper for the GPU box, not a pytest file."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1408_2981_b200 import synth, tpmg  # noqa: E402


def main():
    P = synth.baseline_config(3)
    ctx = tpmg.Context()
    h = tpmg.Hierarchy(ctx, P)
    n = P.nx * P.ny * P.nz
    fk = torch.from_numpy(synth.x_fastest_to_k_fastest(P.rhs()).reshape(-1)).pin_memory().numpy()
    xs = [torch.empty(n, dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
    K = int(os.environ.get("TPMG_K", "5"))
    tpmg.pcg_solve_host_batch(h, [fk] * 2, xs, P.tol, 200, layout=tpmg.K_FASTEST)
    for _ in range(2):
        t0 = time.perf_counter()
        tpmg.pcg_solve_host_batch(h, [fk] * K, [xs[i % 2] for i in range(K)], P.tol, 200,
                                  layout=tpmg.K_FASTEST)
        print(f"batch of {K}: {(time.perf_counter() - t0) * 1e3 / K:.2f} ms per step", flush=True)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        tpmg.pcg_solve_host_batch(h, [fk] * K, [xs[i % 2] for i in range(K)], P.tol, 200,
                                  layout=tpmg.K_FASTEST)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    big = [e for e in ev if "Memcpy" in e.name or "kfast" in e.name or "xfast" in e.name
           or "k_pcg_xfinal" in e.name or "k_dot_tiles" in e.name]
    for e in big:
        print(f"{(e.time_range.start - t0) / 1e3:9.2f} ms +{e.time_range.elapsed_us() / 1e3:7.2f} ms "
              f"{e.name[:60]}")


if __name__ == "__main__":
    main()
