"""A/B timing of alternative builds of the product library (profiling helper for the GPU box,
not a pytest file).  Each library runs in its own process (TPMG_LIB_PATH), the libraries
interleaved over TPMG_ROUNDS rounds; per library: finest-level kernel medians
(tests/ab_kernels.py) and config-3 solve times (min / median of 5 after 2 warm-up solves).

    python tests/ab_libs.py build/ab/base.so build/ab/x.so -- post rr ap
"""
import os
import re
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SOLVE = r"""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_1408_2981_b200 import synth, tpmg
P = synth.baseline_config(int(__import__('os').environ.get('TPMG_CFG', '3')))
ctx = tpmg.Context(); h = tpmg.Hierarchy(ctx, P)
f = h.field().upload(P.rhs()); x = h.field()
for i in range(2): tpmg.pcg_solve(h, f, x, P.tol, 200)
ts = []
for i in range(5):
    torch.cuda.synchronize(); t = time.perf_counter(); r = tpmg.pcg_solve(h, f, x, P.tol, 200)
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
hist = ' '.join(float(v).hex() for v in r.history)
import hashlib
print('SOLVE', r.iterations, min(ts), sorted(ts)[2], hashlib.sha256(hist.encode()).hexdigest()[:12])
"""


def main():
    args = sys.argv[1:]
    libs = args[:args.index("--")] if "--" in args else args
    ks = args[args.index("--") + 1:] if "--" in args else ["post", "rupdate", "ap", "rr"]
    rounds = int(os.environ.get("TPMG_ROUNDS", "2"))
    kt = {lib: {k: [] for k in ks} for lib in libs}
    st = {lib: [] for lib in libs}
    digests = {lib: set() for lib in libs}
    for _ in range(rounds):
        for lib in libs:
            env = dict(os.environ, TPMG_LIB_PATH=os.path.abspath(lib), TPMG_ROUNDS="3")
            if ks:
                out = subprocess.run([sys.executable, "tests/ab_kernels.py", *ks], cwd=ROOT, env=env,
                                     capture_output=True, text=True, timeout=600).stdout
                for line in out.splitlines():
                    m = re.search(r"(\S+)\s+median ([\d.]+) ms", line)
                    if m and m.group(1) in kt[lib]:
                        kt[lib][m.group(1)].append(float(m.group(2)))
            out = subprocess.run([sys.executable, "-c", SOLVE], cwd=ROOT, env=env,
                                 capture_output=True, text=True, timeout=600)
            for line in out.stdout.splitlines():
                if line.startswith("SOLVE"):
                    _, it, mn, md, dg = line.split()
                    st[lib].append((float(mn), float(md), int(it)))
                    digests[lib].add(dg)
            if out.returncode:
                print(lib, "solve failed:", out.stderr[-2000:])
    for lib in libs:
        ktxt = "  ".join(f"{k} {statistics.median(v):.4f}" for k, v in kt[lib].items() if v)
        s = st[lib]
        stxt = (f"solve min {min(x[0] for x in s):.2f} med {statistics.median(x[1] for x in s):.2f} ms"
                f" it {s[0][2]} hist {','.join(sorted(digests[lib]))}" if s else "solve -")
        print(f"{os.path.basename(lib):16s} {ktxt}  | {stxt}", flush=True)


if __name__ == "__main__":
    main()
