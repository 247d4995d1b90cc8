"""The product's NCCL transport on the one-GPU pool: a one-rank NCCL communicator
(TPMG_LOOPBACK=2 at tpmg_init) carries the loopback halos, so every ncclSend / ncclRecv group of
exchange(), exchange_deep() and the side-stream f halos (second communicator from
ncclCommSplit), the all-gathers of the tile partials and of the agglomerated block, and the
all-reduced zero-pivot flag really execute -- eagerly and inside the captured PCG graphs.
Spawned by tests/test_nccl_self.py (its own process: an NCCL failure or hang cannot take the
test session with it).

    python tests/mp/nccl_self_rank.py PROBLEM OUTFILE [golden]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ["TPMG_LOOPBACK"] = "2"
import numpy as np  # noqa: E402

import ipc_rank  # noqa: E402
from paper_1408_2981_b200 import synth, tpmg  # noqa: E402


def main():
    name, out = sys.argv[1], sys.argv[2]
    golden = len(sys.argv) > 3 and sys.argv[3] == "golden"
    if golden:
        P = synth.parity_problem(name)
        if len(sys.argv) > 4:
            P.agglomerate = int(sys.argv[4])
    else:
        P = ipc_rank.PROBLEMS[name]()
    ctx = tpmg.Context(device=0)
    h = tpmg.Hierarchy(ctx, P)
    f_host = P.rhs()
    f = h.field().upload(f_host)
    n0 = ctx.kernel_launches()
    x = h.field()
    res = tpmg.pcg_solve(h, f, x, P.tol, 300)
    launches = ctx.kernel_launches() - n0
    if golden:
        import hashlib

        xs = x.download()
        np.savez(out, hist=res.history, iters=res.iterations, status=res.status,
                 launches=launches, nccl=ctx.nccl_calls(),
                 sha=hashlib.sha256(np.ascontiguousarray(xs, dtype="<f8").tobytes()).hexdigest())
    else:
        y = h.field()
        tpmg.apply_operator(h, f, y)
        v = h.field().fill(0.0)
        tpmg.v_cycle(h, f, v)
        np.savez(out, y=y.download(), v=v.download(), x=x.download(), hist=res.history,
                 iters=res.iterations, status=res.status, launches=launches,
                 nccl=ctx.nccl_calls(), ff=tpmg.dot(h, f, f))
    h.close()
    ctx.close()


if __name__ == "__main__":
    main()
