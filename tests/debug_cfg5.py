"""Locates the first operation where the device and the oracle part on config-5-like problems
(nz = 64, lognormal profile, geometric grading, V(2,2)) as the horizontal size grows.  Debug
driver for the GPU box, not a pytest file.

    python tests/debug_cfg5.py [n ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402  (checker)
from conftest import rng_field  # noqa: E402
from paper_1408_2981_b200 import synth, tpmg  # noqa: E402
from paper_1408_2981_b200.tpmg import K_FASTEST  # noqa: E402


def diff(a, b):
    bad = np.flatnonzero(a != b)
    if bad.size == 0:
        return "bitwise"
    rel = np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)
    return f"{bad.size} differ (first {bad[:4]}), max rel {rel:.2e}"


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [64, 128, 256, 512]
    ctx = tpmg.Context()
    for n in sizes:
        depth = int(np.log2(n // 8)) + 1
        P = synth.baseline_config(5, nx=n, ny=n, depth=depth, h=1.0 / 4096,
                                  name=f"cfg5like_{n}")
        h = tpmg.Hierarchy(ctx, P)
        o = O.OracleHierarchy.from_problem(P, threads=os.cpu_count() or 1)
        print(f"== {n}x{n}x{P.nz}, {h.n_levels} levels", flush=True)
        for l in range(h.n_levels):
            g, r = h.coefficients(l), o.coefficients(l)
            for k in g:
                if not np.array_equal(g[k], r[k]):
                    print(f"  coef level {l} {k}: {diff(g[k], r[k])}")
        for l in range(h.n_levels - 1, -1, -1):
            m = o.size(l)
            u, f = rng_field(10 + l, m), rng_field(20 + l, m)
            fu, fy, ff = h.field(l).upload(u, K_FASTEST), h.field(l), h.field(l).upload(f, K_FASTEST)
            tpmg.apply_operator(h, fu, fy)
            print(f"  level {l} apply: {diff(fy.download(K_FASTEST), o.apply(l, u))}")
            tpmg.smooth(h, fu, ff, 2)
            print(f"  level {l} smooth x2: {diff(fu.download(K_FASTEST), o.smooth(l, u, f, 2))}")
            z = h.field(l)
            tpmg.smooth(h, z, ff, 1)  # zero guess
            print(f"  level {l} smooth from 0: {diff(z.download(K_FASTEST), o.smooth(l, np.zeros_like(f), f, 1))}")
            if l > 0:
                c = h.field(l - 1)
                tpmg.restrict_field(h, ff, c)
                print(f"  level {l} restrict: {diff(c.download(K_FASTEST), o.restrict(l - 1, f))}")
        f = synth.x_fastest_to_k_fastest(P.rhs())
        ff, fu = h.field().upload(f, K_FASTEST), h.field()
        tpmg.v_cycle(h, ff, fu)
        print(f"  v_cycle: {diff(fu.download(K_FASTEST), o.vcycle(f))}", flush=True)
        x = h.field()
        res = tpmg.pcg_solve(h, ff, x, P.tol, 300)
        xo, hist_o, it_o, st_o = o.pcg(f, P.tol, 300)
        k = min(len(hist_o), len(res.history))
        hd = np.flatnonzero(res.history[:k] != hist_o[:k])
        print(f"  pcg: iterations {res.iterations} vs {it_o}; history first differing entry "
              f"{hd[:1]}; max rel {np.max(np.abs(res.history[:k] - hist_o[:k]) / hist_o[:k]):.2e}",
              flush=True)
        del h, o


if __name__ == "__main__":
    main()
