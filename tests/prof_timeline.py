"""Live kernel timeline of one PCG solve (CUPTI through torch.profiler, graph replays included):
per-kernel live time, the sum of kernel time against the solve's span, and the gaps between
consecutive kernels.  Profiling driver for the GPU box, not a pytest file.

    TPMG_CFG=3 python tests/prof_timeline.py
"""
import collections
import os
import sys

# ncu / CUPTI do not see kernels inside conditional graph bodies: profile the host PCG loop
os.environ.setdefault("TPMG_DEVLOOP", "0")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1408_2981_b200 import synth, tpmg  # noqa: E402


def _name(e) -> str:
    n = e.name.replace("(anonymous namespace)::", "").replace("void ", "").replace("tpmg::", "")
    return n.split("(")[0][:90]


def main():
    P = synth.baseline_config(int(os.environ.get("TPMG_CFG", "3")))
    ctx = tpmg.Context()
    h = tpmg.Hierarchy(ctx, P)
    h.set_use_graphs(os.environ.get("TPMG_GRAPHS", "1") == "1")
    f = h.field().upload(P.rhs())
    x = h.field()
    for _ in range(2):
        tpmg.pcg_solve(h, f, x, P.tol, 200)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        res = tpmg.pcg_solve(h, f, x, P.tol, 200)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
          and e.time_range.elapsed_us() > 0 and "Memcpy" not in e.name and "Memset" not in e.name]
    ev.sort(key=lambda e: e.time_range.start)
    if not ev:
        print("no kernel events captured")
        return
    span = ev[-1].time_range.end - ev[0].time_range.start
    busy = sum(e.time_range.elapsed_us() for e in ev)
    gaps = [max(0.0, b.time_range.start - a.time_range.end) for a, b in zip(ev, ev[1:])]
    print(f"iterations {res.iterations}; kernels {len(ev)}; span {span / 1e3:.3f} ms; "
          f"kernel time {busy / 1e3:.3f} ms; gaps {sum(gaps) / 1e3:.3f} ms "
          f"(mean {sum(gaps) / max(1, len(gaps)):.2f} us, max {max(gaps):.1f} us)")
    per = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        k = _name(e) + f" <{e.time_range.elapsed_us() > 0}>" * 0
        per[k][0] += 1
        per[k][1] += e.time_range.elapsed_us()
    print(f"{'kernel':90s} {'n':>4s} {'ms':>8s} {'us/launch':>10s}")
    for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{k:90s} {n:4d} {t / 1e3:8.3f} {t / n:10.1f}")
    # gaps by the kernel that follows them
    gk = collections.defaultdict(float)
    for g, b in zip(gaps, ev[1:]):
        gk[_name(b)[:60]] += g
    print("gap before kernel (top):")
    for k, g in sorted(gk.items(), key=lambda kv: -kv[1])[:10]:
        print(f"  {k:60s} {g / 1e3:.3f} ms")
    print("largest gaps (predecessor -> successor):")
    big = sorted(zip(gaps, ev, ev[1:]), key=lambda t: -t[0])[:8]
    for g, a, b in big:
        print(f"  {g:8.1f} us  {_name(a)[:45]:45s} -> {_name(b)[:45]}")


if __name__ == "__main__":
    main()
