"""One rank of a multi-process run on the CUDA-IPC transport (tpmg_init_ipc): spawned by
tests/test_ipc_multirank.py, several ranks may share one GPU.  Builds its tile of a global
problem through the product's own rank wiring (tile offsets from the hierarchy, the exact-mean
RHS from per-tile integer sums), then runs apply, a V-cycle and a PCG solve and saves its tiles.

    python tests/mp/ipc_rank.py RANK WORLD PX PY SESSION PROBLEM OUTDIR
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1408_2981_b200 import synth, tpmg  # noqa: E402

def _agg(P, cols):
    P.agglomerate = cols
    return P


PROBLEMS = {
    "cfg1": lambda: synth.baseline_config(1),
    # 32x4-tiled kernels and the TMA pipelines on every rank's finest tiles
    "tiled": lambda: synth.make_problem(128, 64, 16, omega2=1e-2, lambda2=1e-4,
                                        grading="quadratic", profile="uniform", profile_seed=3,
                                        depth=4, name="tiled"),
    # every rank's finest tile above the coarse regime (> 4096 columns): the decomposed fused
    # residual + transpose restriction with its two-cell halo, corners and coefficient ring
    "rr2": lambda: synth.make_problem(256, 128, 16, omega2=1e-2, lambda2=1e-4,
                                      grading="geometric", ratio=1.2, profile="lognormal",
                                      profile_seed=6, profile_sigma=0.5, depth=4, name="rr2"),
    # coarse-grid agglomeration: levels of <= 512 global columns replicated on every rank
    "tiled_agg": lambda: _agg(synth.make_problem(128, 64, 16, omega2=1e-2, lambda2=1e-4,
                                                 grading="quadratic", profile="uniform",
                                                 profile_seed=3, depth=4, name="tiled-agg"), 512),
    "rr2_agg": lambda: _agg(synth.make_problem(256, 128, 16, omega2=1e-2, lambda2=1e-4,
                                               grading="geometric", ratio=1.2, profile="lognormal",
                                               profile_seed=6, profile_sigma=0.5, depth=5,
                                               name="rr2-agg"), 2048),
    "cfg5s": lambda: synth.make_problem(64, 64, 16, omega2=1e-5, lambda2=1e-6,
                                        grading="geometric", ratio=1.1, profile="lognormal",
                                        profile_seed=2, depth=4, nu=2, tol=1e-10, name="cfg5-small"),
}


def main():
    rank, world, px, py = (int(v) for v in sys.argv[1:5])
    session, name, out = sys.argv[5], sys.argv[6], sys.argv[7]
    P = PROBLEMS[name]()
    ctx = tpmg.Context(device=0, rank=rank, world_size=world, px=px, py=py, ipc_session=session)
    h = tpmg.Hierarchy(ctx, P)
    lnx, lny, nz, x0, y0 = h.level_shape(h.finest)
    # the distributed exact mean: every tile's integer mantissa sum (the tiles of all ranks,
    # from the hierarchy's own decomposition), one correctly rounded division
    msum = 0
    for r in range(world):
        rx, ry = r % px, r // px
        msum += synth.tile_m_sum(P.rhs_seed, P.nx, P.ny, P.nz, rx * lnx, ry * lny, lnx, lny)
    mean = synth.mean_from_m_sum(msum, P.n_dof)
    f_host = synth.rhs_x_fastest(P.rhs_seed, P.nx, P.ny, P.nz, x0, y0, lnx, lny, mean=mean)
    f = h.field().upload(f_host)
    y = h.field()
    tpmg.apply_operator(h, f, y)
    v = h.field().fill(0.0)
    tpmg.v_cycle(h, f, v)
    x = h.field()
    res = tpmg.pcg_solve(h, f, x, P.tol, 300)
    dots = tpmg.dot(h, f, f)
    np.savez(os.path.join(out, f"rank{rank}.npz"), x0=x0, y0=y0, lnx=lnx, lny=lny,
             f=f_host, y=y.download(), v=v.download(), x=x.download(), hist=res.history,
             iters=res.iterations, status=res.status, ff=dots, levels=h.n_levels)
    for fld in (f, y, v, x):
        fld.close()
    h.close()
    ctx.close()


if __name__ == "__main__":
    main()
