"""The NCCL transport itself, executed on the pool's single B200 (
PAPER.md:518-521).  NCCL cannot put two ranks on one GPU, but a ONE-rank communicator can send
to and receive from itself: with TPMG_LOOPBACK=2 at tpmg_init the decomposed schedule's halos and
reductions go through the product's NCCL code -- the grouped ncclSend / ncclRecv of the face and
two-cell exchanges (the rank is every neighbour of a 1x1 periodic process grid, so the pieces are
matched in order exactly as between two ranks of a px = 2 grid), the f halos on the side stream
with the ncclCommSplit communicator, ncclAllGather of the tile partials and of the agglomerated
block, the all-reduced zero-pivot flag -- eagerly and inside the captured PCG iteration graphs.
Results must be the one-rank oracle's bits.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1408_2981_b200 import synth

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "mp"))
import ipc_rank  # noqa: E402


def _run(args, timeout):
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "WARN"))
    p = subprocess.run([sys.executable, os.path.join(HERE, "mp", "nccl_self_rank.py"), *args],
                       stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, env=env,
                       timeout=timeout)
    assert p.returncode == 0, p.stdout[-4000:]


@pytest.mark.parametrize("name", ["cfg1", "tiled", "rr2", "tiled_agg", "rr2_agg", "cfg5s"])
def test_nccl_self_transport_matches_oracle(tmp_path, oracle_mod, name):
    out = str(tmp_path / "r.npz")
    _run([name, out], 300)
    d = dict(np.load(out))
    P = ipc_rank.PROBLEMS[name]()
    o = oracle_mod.OracleHierarchy.from_problem(P)
    fk = synth.x_fastest_to_k_fastest(P.rhs())
    k = synth.x_fastest_to_k_fastest
    np.testing.assert_array_equal(k(d["y"].reshape(P.nz, P.ny, P.nx)), o.apply(o.finest, fk))
    np.testing.assert_array_equal(k(d["v"].reshape(P.nz, P.ny, P.nx)), o.vcycle(fk))
    xo, hist_o, it_o, st_o = o.pcg(fk, P.tol, 300)
    assert int(d["status"]) == st_o == 0 and int(d["iters"]) == it_o
    np.testing.assert_array_equal(d["hist"], hist_o)
    np.testing.assert_array_equal(k(d["x"].reshape(P.nz, P.ny, P.nx)), xo)
    # the transport really was NCCL: at least one grouped exchange per stencil kernel and one
    # gather per dot product were issued (captured iterations count once, at capture)
    assert int(d["nccl"]) > 200, int(d["nccl"])


@pytest.mark.parametrize("agg", [0, 128 * 128])
def test_nccl_self_transport_matches_golden_at_config3(tmp_path, agg):
    """BASELINE config 3 (1024^2 x 128) on the decomposed schedule with NCCL carrying every halo
    and reduction: the oracle golden, bit for bit."""
    g = json.load(open(os.path.join(HERE, "golden", "oracle_cfg3_pcg.json")))
    out = str(tmp_path / "r.npz")
    _run(["cfg3", out, "golden", str(agg)], 600)
    d = dict(np.load(out))
    assert int(d["status"]) == 0 and int(d["iters"]) == g["iterations"]
    assert [float(v).hex() for v in d["hist"]] == g["history_hex"]
    assert str(d["sha"]) == g["x_sha256_device_order"]
    assert int(d["nccl"]) > 200, int(d["nccl"])
