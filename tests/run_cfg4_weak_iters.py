"""BASELINE config 4's weak-scaling problems (1024^2 x 128 per GPU on px x py GPUs, each
GPU's tile coarsened to 8x8, i.e. 8 levels whatever the GPU count) solved as ONE global problem
on one B200.  A decomposed solve is bitwise the one-rank solve of the same global problem (the
dots reduce in the one-rank tile order, tests/test_ipc_multirank.py), so the iteration counts
printed here are those of the 1/2/4/8-GPU runs: they show how the convergence responds to the
growing global coarse grid (8x8 per GPU).  Validation driver, not a pytest file.

    python tests/run_cfg4_weak_iters.py [max_gpus] [--coarsening=tile|global|agglomerate]

tile (default here, BASELINE's literal reading): 8 levels per GPU tile, the global coarse grid
grows with N; global: every level decomposed, coarsened as deep as the decomposition allows
(depth 0); agglomerate (bench.py's multi-GPU default): the global grid coarsened to 8 cells along
its longer side, levels of <= 128^2 columns replicated on every GPU -- bitwise the one-rank
solve of the same global problem, so these one-GPU runs give its iteration counts exactly.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1408_2981_b200 import tpmg  # noqa: E402

sys.path.insert(0, ROOT)
import bench  # noqa: E402  (the problem definition bench.py --config 4w uses)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    top = int(args[0]) if args else 8
    mode = "tile"
    for a in sys.argv[1:]:
        if a.startswith("--coarsening="):
            mode = a.split("=", 1)[1]
        elif a == "--global":
            mode = "global"
    ctx = tpmg.Context()
    for n in (1, 2, 4, 8):
        if n > top:
            break
        px, py = bench.proc_grid(n)
        P, workload, _, _ = bench.make_problem("4w", px, py, mode)
        h = tpmg.Hierarchy(ctx, P)
        f = h.field().upload(P.rhs())
        x = h.field()
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            res = tpmg.pcg_solve(h, f, x, P.tol, 300)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            best = dt if best is None else min(best, dt)
        print(f"{n} GPU(s) {px}x{py}: global {P.nx}x{P.ny}x{P.nz}, {h.n_levels} levels "
              f"(coarsest {P.nx >> (h.n_levels - 1)}x{P.ny >> (h.n_levels - 1)}), status "
              f"{res.status}, {res.iterations} iterations, final rel. residual "
              f"{res.history[-1] / res.history[0]:.2e}; one B200: {best * 1e3:.1f} ms, "
              f"{P.n_dof * res.iterations / best / 1e9:.2f} GDOF/s", flush=True)
        f.close()
        x.close()
        h.close()


if __name__ == "__main__":
    main()
