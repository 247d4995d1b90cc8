"""Regenerates tests/golden/oracle_cfg1_pcg.json: the oracle's BASELINE config-1 PCG solve
(residual history as exact hex floats, iteration count, sum of the iterate).  The GPU path is
compared against the oracle live; this file pins the oracle itself against regressions."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_1408_2981_b200 import synth  # noqa: E402

P = synth.baseline_config(1)
h = O.OracleHierarchy.from_problem(P)
f = synth.x_fastest_to_k_fastest(P.rhs())
x, hist, it, st = h.pcg(f, P.tol, 100)
out = {"config": P.name, "tol": P.tol, "iterations": it, "status": st,
       "history_hex": [float(v).hex() for v in hist], "x_sum_hex": float(np.sum(x)).hex()}
with open(os.path.join(HERE, "oracle_cfg1_pcg.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(it, hist[-1] / hist[0])
