"""Ad-hoc GPU diagnostic: each kernel at a tiled-path size vs the oracle (not a pytest file)."""
import os
import sys
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O  # noqa: E402
from paper_1408_2981_b200 import synth, tpmg  # noqa: E402
from paper_1408_2981_b200.tpmg import K_FASTEST  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def main(variant="exact"):
    ctx = tpmg.Context(variant=variant)
    for (nx, ny, nz) in [(64, 8, 16), (32, 4, 8), (128, 64, 32)]:
        P = synth.make_problem(nx, ny, nz, omega2=1e-2, lambda2=1e-4, grading="quadratic",
                               profile="uniform", depth=1)
        h = tpmg.Hierarchy(ctx, P)
        o = O.OracleHierarchy.from_problem(P)
        n = nx * ny * nz
        rng = np.random.default_rng(1)
        u, f = rng.standard_normal(n), rng.standard_normal(n)
        fu, ff, fy = h.field().upload(u, K_FASTEST), h.field().upload(f, K_FASTEST), h.field()
        for name, fn in [
            ("apply", lambda: (tpmg.apply_operator(h, fu, fy), fy.download(K_FASTEST), o.apply(0, u))),
            ("resid", lambda: (tpmg.residual(h, ff, fu, fy), fy.download(K_FASTEST), o.residual(0, f, u))),
            ("smooth1", lambda: (tpmg.smooth(h, fy.copy_from(fu), ff, 1), fy.download(K_FASTEST), o.smooth(0, u, f, 1))),
            ("smooth0", lambda: (tpmg.smooth(h, fy.fill(0.0), ff, 1), fy.download(K_FASTEST), o.smooth(0, np.zeros(n), f, 1))),
        ]:
            try:
                _, g, r = fn()
                bad = np.flatnonzero(g != r)
                print(f"{variant} {nx}x{ny}x{nz} {name}: rel {rel(g, r):.3e} nbad {bad.size} first {bad[:6]}", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"{variant} {nx}x{ny}x{nz} {name}: EXC {type(e).__name__} {e}", flush=True)
                traceback.print_exc()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "exact")
