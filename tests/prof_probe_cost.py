"""Cost of the live kernel probes (event-record nodes in the iteration graph) on the timed
solve: config-3 solves back to back, CUDA events on the library stream, probes off / on.
Profiling helper for the GPU box, not a pytest file."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1408_2981_b200 import synth, tpmg  # noqa: E402


def main():
    P = synth.baseline_config(3)
    ctx = tpmg.Context()
    h = tpmg.Hierarchy(ctx, P)
    f = h.field().upload(P.rhs())
    x = h.field()
    stream = torch.cuda.ExternalStream(ctx.stream_handle())
    for probe in (False, True, False, True):
        h.kernel_probe(probe)
        for _ in range(2):
            tpmg.pcg_solve(h, f, x, P.tol, 200)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            tpmg.pcg_solve(h, f, x, P.tol, 200)
        e1.record(stream)
        e1.synchronize()
        print(f"probes {'on ' if probe else 'off'}: {e0.elapsed_time(e1) / 5:.2f} ms per solve", flush=True)


if __name__ == "__main__":
    main()
