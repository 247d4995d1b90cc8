"""Cost of the decomposed schedule and of the NCCL transport on one GPU (profiling helper, not a
pytest file): BASELINE config 3 solved one-rank, on the decomposed schedule with loopback halos
(TPMG_LOOPBACK=1) and with NCCL itself carrying every halo and reduction (TPMG_LOOPBACK=2, a
one-rank communicator: sends / receives to self), each in its own process; min / median of 5
solves after 2 warm-up solves, with and without coarse-grid agglomeration.

    python tests/prof_transport.py
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SOLVE = r"""
import sys, time, os
sys.path.insert(0, '.')
import torch
from paper_1408_2981_b200 import synth, tpmg
P = synth.baseline_config(3)
P.agglomerate = int(os.environ.get('AGG', '0'))
ctx = tpmg.Context(); h = tpmg.Hierarchy(ctx, P)
f = h.field().upload(P.rhs()); x = h.field()
for i in range(2): tpmg.pcg_solve(h, f, x, P.tol, 200)
ts = []
n0 = ctx.nccl_calls(); k0 = ctx.kernel_launches()
for i in range(5):
    torch.cuda.synchronize(); t = time.perf_counter(); r = tpmg.pcg_solve(h, f, x, P.tol, 200)
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
print('SOLVE', r.iterations, '%.2f %.2f' % (min(ts), sorted(ts)[2]), (ctx.kernel_launches() - k0) // 5,
      ctx.nccl_calls())
"""


def main():
    for agg in ("0", str(128 * 128)):
        for lb, name in (("0", "one rank"), ("1", "decomposed, loopback halos"),
                         ("2", "decomposed, NCCL transport")):
            if lb == "0" and agg != "0":
                continue
            env = dict(os.environ, TPMG_LOOPBACK=lb, AGG=agg)
            p = subprocess.run([sys.executable, "-c", SOLVE], cwd=ROOT, env=env, text=True,
                               stdout=subprocess.PIPE, stderr=subprocess.STDOUT, timeout=600)
            line = [l for l in p.stdout.splitlines() if l.startswith("SOLVE")]
            print(f"{name:30s} agglomerate={agg:6s} " +
                  (line[0] if line else "FAILED\n" + p.stdout[-2000:]), flush=True)


if __name__ == "__main__":
    main()
