"""The product's multi-rank code across PROCESSES: 2x1,
1x2 and 2x2 process grids on the CUDA-IPC transport (tpmg_init_ipc), several ranks sharing the
one B200 of the pool.  Every rank is a separate process (tests/mp/ipc_rank.py) running the
product's rank wiring -- tile offsets, the exact-mean RHS from per-tile sums, per-tile
coarsening, face halos written into the neighbours' receive buffers, dot products reduced over
the ranks -- and the assembled global results are compared with the GLOBAL oracle:

  * operator apply and a V-cycle (no reductions): bitwise;
  * PCG: the north_star bar (residual history within 1e-10 relative, iterations +-1), and --
    where every rank's tile is a multiple of the 32x4 reduction tile, as in all of BASELINE's
    multi-GPU configs -- BITWISE: the ranks gather their tile partials and reduce them in the
    one-rank tile order (k_reduce_tiles), so the solve does not depend on the rank count.

No kernel waits on another process: every exchange is ordered by host barriers around stream
synchronisations (see tpmg_init_ipc in include/tpmg_b200.h).
"""
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

from paper_1408_2981_b200 import synth

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "mp"))
import ipc_rank  # noqa: E402


def run_ranks(tmp_path, name, px, py):
    world = px * py
    session = f"t{uuid.uuid4().hex[:12]}"
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp", "ipc_rank.py"), str(r),
                               str(world), str(px), str(py), session, name, str(tmp_path)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=240)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{outs[r][-3000:]}"
    return [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(world)]


def assemble(parts, key, P):
    g = np.empty((P.nz, P.ny, P.nx))
    for d in parts:
        x0, y0, lnx, lny = int(d["x0"]), int(d["y0"]), int(d["lnx"]), int(d["lny"])
        g[:, y0:y0 + lny, x0:x0 + lnx] = d[key].reshape(P.nz, lny, lnx)
    return g


@pytest.mark.parametrize("name", ["cfg1", "tiled", "cfg5s", "rr2", "tiled_agg", "rr2_agg"])
@pytest.mark.parametrize("grid", [(2, 1), (1, 2), (2, 2)])
def test_ipc_ranks_match_global_oracle(tmp_path, oracle_mod, name, grid):
    px, py = grid
    P = ipc_rank.PROBLEMS[name]()
    parts = run_ranks(tmp_path, name, px, py)
    o = oracle_mod.OracleHierarchy.from_problem(P)
    f = P.rhs()
    np.testing.assert_array_equal(assemble(parts, "f", P), f)  # distributed exact mean
    fk = synth.x_fastest_to_k_fastest(f)
    # element-wise paths: bitwise
    yk = synth.x_fastest_to_k_fastest(assemble(parts, "y", P))
    np.testing.assert_array_equal(yk, o.apply(o.finest, fk))
    vk = synth.x_fastest_to_k_fastest(assemble(parts, "v", P))
    np.testing.assert_array_equal(vk, o.vcycle(fk))
    # PCG: every rank took the same decisions; the bar of BASELINE.json against the oracle
    xo, hist_o, it_o, st_o = o.pcg(fk, P.tol, 300)
    for d in parts[1:]:
        assert int(d["iters"]) == int(parts[0]["iters"])
        np.testing.assert_array_equal(d["hist"], parts[0]["hist"])
    it, hist = int(parts[0]["iters"]), parts[0]["hist"]
    assert int(parts[0]["status"]) == st_o == 0
    assert abs(it - it_o) <= 1, (it, it_o)
    n = min(len(hist), len(hist_o))
    rel = np.max(np.abs(hist[:n] - hist_o[:n]) / hist_o[:n])
    assert rel <= 1e-10, rel
    xk = synth.x_fastest_to_k_fastest(assemble(parts, "x", P))
    assert np.max(np.abs(xk - xo)) <= 1e-8 * np.max(np.abs(xo))
    if (P.nx // px) % 32 == 0 and (P.ny // py) % 4 == 0:  # tile-aligned: decomposition-invariant
        assert it == it_o
        np.testing.assert_array_equal(hist, hist_o)
        np.testing.assert_array_equal(xk, xo)
    # the all-reduced dot is the global one up to summation order
    ff = float(np.dot(f.ravel(), f.ravel()))
    assert abs(float(parts[0]["ff"]) - ff) <= 1e-12 * ff
