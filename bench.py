#!/usr/bin/env python
"""Headline benchmark: the PCG + TPMG solve of BASELINE.json on the sm_100a path, one process
per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 3|4w|4s|5]

One STEP = one complete PCG solve (x0 = 0 -> |r|/|r0| <= tol) of the synthetic problem.
--config (BASELINE.json configs; seeded synthetic inputs of their shapes, no dataset exists):
  3   (default, N = 1)  config 3: 1024^2 x 128, V(1,1), 8 levels to 8x8, tol 1e-8
  4w  (default, N > 1)  config 4 weak scaling: 1024^2 x 128 per GPU, (1024 px) x (1024 py)
                        global, each GPU's tile coarsened to 8x8
  4s                    config 4 strong scaling: 2048^2 x 128 global on N GPUs, 9 levels to a
                        global 8x8
  5                     config 5: 4096^2 x 64, omega^2 = 1e-5, lambda^2 = 1e-6, lognormal
                        profile, geometric grading 1.1, V(2,2), tol 1e-10, 10 levels
value = whole-job throughput in GDOF/s = global DOF x PCG iterations / second (max over
ranks).  The line also carries PCG iterations/s, V-cycle GDOF/s, live per-launch durations of
the finest-level kernels (CUDA event probes in the iteration graphs, over K solves right after
the timed region -- the probes' event nodes are kept out of the timed solves themselves), the
roofline of the one with the largest share of the solve, parity against the committed
oracle golden of the same solve, and the CPU baseline (the oracle port on the host cores).
--impl reference times the CPU restatement of the reference path (oracle/) on the host.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG+MG iterations/sec and GDOF/s per V-cycle; achieved HBM GB/s vs peak"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.samples, self._proc = device, [], None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._active = False

    def _run(self):
        try:
            for line in self._proc.stdout:
                if self._active and line.strip():
                    self.samples.append([x.strip() for x in line.split(",")])
        except Exception:
            pass

    def __enter__(self):
        try:  # one streaming process (every 50 ms) instead of one process per sample
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self._t.start()
            time.sleep(0.15)
        except Exception:
            self._proc = None
        self._active = True
        return self

    def __exit__(self, *a):
        self._active = False
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def proc_grid(n: int):
    """px x py = n with py the largest divisor of n not above sqrt(n):
    1->(1,1) 2->(2,1) 3->(3,1) 4->(2,2) 6->(3,2) 8->(4,2)."""
    py = max(d for d in range(1, int(math.isqrt(n)) + 1) if n % d == 0)
    return n // py, py


# Coarse-grid agglomeration threshold of the multi-GPU runs: levels whose GLOBAL grid has at
# most this many columns (128^2) are kept whole on every GPU and solved redundantly there (one
# all-gather per V-cycle instead of ~6 halo exchanges per level on grids of a few thousand columns
# split N ways, where every kernel is latency-bound anyway).
AGGLOMERATE_COLS = 128 * 128


def global_depth(nx: int, ny: int, coarsest: int = 8) -> int:
    """Levels of the global grid down to `coarsest` cells along its longer side (BASELINE
    config 3's 8x8 at 1024^2; 8x4 for the 2:1 grids of 2 and 8 GPUs)."""
    return int(math.log2(max(nx, ny) // coarsest)) + 1


def make_problem(cfg: str, px: int, py: int, coarsening: str = "agglomerate"):
    """(problem, workload name, scaling, parity golden name or None).

    coarsening (multi-GPU runs): "agglomerate" -- the global grid coarsened to 8 cells along its
    longer side with the levels of at most AGGLOMERATE_COLS columns replicated on every GPU (the
    solve is bitwise the one-GPU solve of the same global problem); "tile" -- BASELINE's 8x8 per
    GPU tile with every level decomposed (the global coarse grid grows with N); "global" -- every
    level decomposed, coarsened as deep as the decomposition allows."""
    from paper_1408_2981_b200 import synth

    n = px * py
    if cfg == "3" and n > 1:
        cfg = "4w"
    agg = AGGLOMERATE_COLS if (n > 1 and coarsening == "agglomerate") else 0
    if cfg == "3":
        return synth.baseline_config(3), "config 3 (1 GPU solve)", "weak", "cfg3"
    if cfg == "4w":  # 1024^2 x 128 per GPU, same h, operator and RHS distribution
        nx, ny = 1024 * px, 1024 * py
        depth = {"agglomerate": global_depth(nx, ny), "tile": 8, "global": 0}[coarsening]
        P = synth.make_problem(
            nx, ny, 128, omega2=1e-3, lambda2=1e-4, grading="quadratic", depth=depth,
            nu=1, tol=1e-8, h=1.0 / 1024, name=f"cfg4w_{nx}x{ny}x128")
        P.agglomerate = agg
        work = f"config 4 weak scaling ({px}x{py} GPUs"
        work += {"agglomerate": ", global coarse grid agglomerated below 128^2 columns)" if n > 1
                 else ")", "tile": ", 8x8 per GPU tile)", "global": ", global coarsening)"}[coarsening]
        return P, work, "weak", "cfg3" if n == 1 else None
    if cfg == "4s":  # the same global hierarchy (9 levels) at every GPU count: one golden
        P = synth.parity_problem("cfg4s")
        P.agglomerate = agg
        return P, f"config 4 strong scaling ({px}x{py} GPUs)", "strong", "cfg4s"
    if cfg == "5":
        P = synth.baseline_config(5)
        P.agglomerate = agg
        return P, f"config 5 ({px}x{py} GPUs)", "strong", None
    raise SystemExit(f"unknown --config {cfg}")


def config_dict(P, workload: str, px: int, py: int, levels=None) -> dict:
    """The one config dict both arms print (same workload, same keys)."""
    return {"workload": f"{P.name}: {workload}", "global_grid": [P.nx, P.ny, P.nz],
            "tile": [P.nx // px, P.ny // py, P.nz], "process_grid": [px, py],
            "solver": f"PCG + TPMG V({P.nu_pre},{P.nu_post}), block line-Jacobi relax={P.relax}, "
                      f"{'linear' if P.prolongation == 0 else 'injection'} prolongation + "
                      f"{'transpose' if P.restriction == 1 else 'summation'} restriction, "
                      f"coarsest level 1 sweep",
            "tol": P.tol, "levels": levels if levels is not None else P.depth,
            "agglomerate_columns": P.agglomerate,
            "omega2": P.omega ** 2, "lambda2": float(P.beta_r[0]),
            "l2": "inputs larger than L2 (one field >= 1.07 GB)"}


def load_golden(name):
    if name is None:
        return None
    path = os.path.join(ROOT, "tests", "golden", f"oracle_{name}_pcg.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        g = json.load(fh)
    g["path"] = os.path.relpath(path, ROOT)
    return g


class CpuPort:
    """The oracle port (the reference's algorithm, parallel_for threading) on the host cores.
    One sample = r0, the prologue V-cycle and `iters` PCG iterations of the same solve; its
    step time is the iterations' span from the solve's ConvergenceHistory seconds column."""

    def __init__(self, P, threads: int):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        from paper_1408_2981_b200 import synth

        O.build()
        self.P = P
        self.o = O.OracleHierarchy.from_problem(P, threads=threads)
        self.o.set_device_order(False)  # no checker machinery in the timed CPU path
        self.f = synth.x_fastest_to_k_fastest(P.rhs())

    def sample(self, iters: int = 2):
        """seconds of `iters` PCG iterations (prologue excluded)."""
        _, hist, it, st, secs = self.o.pcg(self.f, self.P.tol, iters, seconds=True)
        return secs[it] - secs[0], it


def cpu_sample_problem(P):
    """The CPU leg's workload: the same problem, or a 2048^2 tile of config 5 (its 4096^2 x 64
    grid needs ~80 GB on the host)."""
    from paper_1408_2981_b200 import synth

    if P.nx * P.ny * P.nz > 2048 * 2048 * 128:
        return synth.parity_problem("cfg5t"), "a 2048^2 x 64 tile of config 5 (same h, operator)"
    return P, "the same problem"


def run_reference(args):
    """--impl reference: the CPU restatement of the reference path (oracle port), all host
    threads; one step = 2 PCG iterations of the same solve (bounded sample)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    px, py = proc_grid(world)
    P, workload, scaling, _ = make_problem(args.config, px, py, args.coarsening)
    Q, what = cpu_sample_problem(P)
    threads = os.cpu_count() or 1
    port = CpuPort(Q, threads)
    per, its = [], 2
    for s in range(args.warmup + args.steps):
        t, its = port.sample(iters=2)
        if s >= args.warmup:
            per.append(t)
    t_step = statistics.median(per)
    value = Q.n_dof * its / t_step / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GDOF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based RNG, BASELINE.json config shapes)",
        "config": config_dict(P, workload, px, py),
        "pcg_iterations_per_s": its / t_step,
        "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": threads, "kind": "port",
                         "sample": f"{Q.name} ({what}): per step {its} PCG iterations of an "
                                   f"oracle solve (after r0 and the prologue V-cycle)"},
        "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="3", choices=["3", "4w", "4s", "5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--max-iter", type=int, default=500)
    ap.add_argument("--no-coef", action="store_true", help="skip the coefficient-storage comparison")
    ap.add_argument("--coarsening", default="agglomerate", choices=["agglomerate", "tile", "global"],
                    help="multi-GPU coarse levels (see make_problem): agglomerate (default), "
                         "tile = BASELINE's 8x8 per GPU tile, global = decomposed to the bottom")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import hashlib

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1408_2981_b200 import synth, tpmg

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    px, py = proc_grid(world)
    P, workload, scaling, golden_name = make_problem(args.config, px, py, args.coarsening)
    torch.cuda.set_device(local)

    nccl_id = None
    if world > 1:
        obj = [tpmg.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = tpmg.Context(device=local, rank=rank, world_size=world, px=px, py=py, nccl_id=nccl_id)
    h = tpmg.Hierarchy(ctx, P)
    lnx, lny, nz, x0, y0 = h.level_shape(h.finest)
    if world == 1:
        f_host = synth.rhs_x_fastest(P.rhs_seed, P.nx, P.ny, P.nz, x0, y0, lnx, lny)
    else:  # each rank sums its own tile exactly; the integer sums are all-gathered
        part = synth.tile_m_sum(P.rhs_seed, P.nx, P.ny, P.nz, x0, y0, lnx, lny)
        sums = [None] * world
        dist.all_gather_object(sums, part)
        mean = synth.mean_from_m_sum(sum(sums), P.n_dof)
        f_host = synth.rhs_x_fastest(P.rhs_seed, P.nx, P.ny, P.nz, x0, y0, lnx, lny, mean=mean)
    f = h.field().upload(f_host)
    x = h.field()
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=local)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up ------------------------------------------------------------------------------
    res = None
    for _ in range(args.warmup):
        res = tpmg.pcg_solve(h, f, x, P.tol, args.max_iter)
    # ---- timed region: K solves, device time by CUDA events on the library stream -------------
    launches0 = ctx.kernel_launches()
    iters, hists = [], []
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            res = tpmg.pcg_solve(h, f, x, P.tol, args.max_iter)
            iters.append(res.iterations)
            hists.append(res.history)
        e1.record(stream)
        e1.synchronize()
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    launches = ctx.kernel_launches() - launches0
    total_iters = sum(iters)
    ms_per_step = ms / args.steps
    it_per_s = total_iters / (ms / 1e3)
    value = P.n_dof * it_per_s / 1e9

    # ---- live per-launch durations of the finest-level kernels in the timed solves -------------
    peak, peak_kind = _peaks()
    n_local = lnx * lny * nz
    C_cols, N_dof = lnx * lny, n_local
    # algorithmic bytes per launch: fields read + written once, 2 B/DOF for a
    # quarter-size coarse field, 32 B per column of hatted scalars
    live_defs = (("pcg_direction_Ap", tpmg.K_PCG_DIRECTION, 40 * N_dof + 32 * C_cols,
                  "k_pcg_ap: x += a p_old; p = z + b p_old; A p, p.(A p)"),
                 ("pcg_rupdate_presweep", tpmg.K_PCG_RUPDATE, 32 * N_dof + 32 * C_cols,
                  "k_jacobi_t3 PCGF=3: q = A p re-formed, r -= a q, |r|^2, sweep from zero"),
                 ("pcg_postsweep_rz", tpmg.K_PCG_POSTSWEEP, 24 * N_dof + 32 * C_cols,
                  "k_jacobi_t3 PCGF=2: line-Jacobi sweep + r.z partials"),
                 ("resid_restrict", tpmg.K_RESID_RESTRICT, 18 * N_dof + 32 * C_cols,
                  "k_resid_restrict_T2: coarse = P^T (f - A u)"),
                 ("prolong_add", tpmg.K_PROLONG_ADD, 18 * N_dof,
                  "k_prolong_flat: u += P e"))
    # live kernel probes: CUDA event pairs around the finest-level PCG kernels, recorded into the
    # iteration graphs (re-captured with the event nodes), over K more solves of the same problem
    # right after the timed region -- the event nodes cost ~1 ms per solve, so the headline
    # value above is timed without them
    h.kernel_probe(True)
    tpmg.pcg_solve(h, f, x, P.tol, args.max_iter)  # captures the probed graphs
    h.kernel_probe(True)  # resets the totals (the graphs captured with probes are kept)
    torch.cuda.synchronize()
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record(stream)
    for _ in range(args.steps):
        tpmg.pcg_solve(h, f, x, P.tol, args.max_iter)
    e5.record(stream)
    e5.synchronize()
    probed_ms = max_over_ranks(e4.elapsed_time(e5))
    kernels_live = {}
    for name, kid, by, what in live_defs:
        tot, n = h.kernel_probe_read(kid)
        tot, n = max_over_ranks(tot), n
        if n == 0:
            continue
        avg = tot / n
        kernels_live[name] = {"kernel": what, "launches": n, "avg_ms": avg,
                              "share_of_timed_region": tot / probed_ms, "algorithmic_bytes": by,
                              "GBps": by / (avg * 1e-3) / 1e9,
                              "frac": by / (avg * 1e-3) / 1e9 / peak}
    h.kernel_probe(False)
    top = max(kernels_live, key=lambda k: kernels_live[k]["share_of_timed_region"]) if kernels_live else None

    # ---- e2e: the same solve through the public API, host buffers in the reference's k-fastest
    # Field order (permutation kernels at the boundary), pinned host memory -------------------------
    # K right-hand sides through tpmg_pcg_host_batch: step i's upload and step i-1's download run
    # on a copy stream while step i is solved (timed by the host clock around the whole call,
    # which returns once the last solution is in host memory)
    f_k = synth.x_fastest_to_k_fastest(f_host)
    f_pin = torch.from_numpy(f_k.reshape(-1)).pin_memory()
    x_pins = [torch.empty(n_local, dtype=torch.float64).pin_memory() for _ in range(2)]
    fnp, xnps = f_pin.numpy(), [xp.numpy() for xp in x_pins]
    tpmg.pcg_solve_host_batch(h, [fnp] * 2, xnps, P.tol, args.max_iter, layout=tpmg.K_FASTEST)  # warm
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rs = tpmg.pcg_solve_host_batch(h, [fnp] * args.steps,
                                   [xnps[i % 2] for i in range(args.steps)], P.tol,
                                   args.max_iter, layout=tpmg.K_FASTEST)
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3)
    barrier()
    e2e_iters = sum(r.iterations for r in rs)
    e2e_value = P.n_dof * e2e_iters / (e2e_ms / 1e3) / 1e9

    # ---- parity: the timed solves against the committed oracle golden of the same solve ------
    parity = None
    g = load_golden(golden_name)
    if g is not None:
        hist_o = np.array([float.fromhex(v) for v in g["history_hex"]])
        n = min(len(hist_o), len(res.history))
        rel = float(np.max(np.abs(res.history[:n] - hist_o[:n]) / hist_o[:n]))
        xs = x.download() if world == 1 else None
        parity = {"golden": g["path"], "iterations": res.iterations,
                  "oracle_iterations": g["iterations"],
                  "history_max_rel_diff": rel,
                  "history_bitwise": [float(v).hex() for v in res.history] == g["history_hex"],
                  "all_timed_solves_identical": all(
                      len(hh) == len(res.history) and bool(np.all(hh == res.history)) for hh in hists),
                  "iterate_sha256_match": None if xs is None else hashlib.sha256(
                      np.ascontiguousarray(xs, dtype="<f8").tobytes()).hexdigest()
                      == g["x_sha256_device_order"],
                  "north_star_bar": "history <= 1e-10 relative, iterations +-1",
                  "pass": rel <= 1e-10 and abs(res.iterations - g["iterations"]) <= 1}
    elif world > 1:
        parity = {"note": "no golden of this global problem; a decomposed solve is bitwise the "
                          "one-GPU solve of the same global problem (tests/test_ipc_multirank.py)"}

    # ---- standalone kernel timings (scratch operands, back-to-back launches) ------------------
    standalone = {}
    for name, kid, by in (("jacobi", tpmg.K_JACOBI, 24 * N_dof + 32 * C_cols),
                          ("jacobi_zero_guess", tpmg.K_JACOBI_ZERO, 16 * N_dof + 32 * C_cols),
                          ("apply", tpmg.K_APPLY, 16 * N_dof + 32 * C_cols)):
        t = h.time_kernel(kid, h.finest, reps=10)
        standalone[name] = {"ms": t, "GBps": by / (t * 1e-3) / 1e9, "frac": by / (t * 1e-3) / 1e9 / peak}
    # V-cycle alone
    vz = h.field()
    torch.cuda.synchronize()
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record(stream)
    for _ in range(5):
        vz.fill(0.0)
        tpmg.v_cycle(h, f, vz)
    e5.record(stream)
    e5.synchronize()
    vcycle_ms = e4.elapsed_time(e5) / 5
    del vz

    # ---- coefficient storage trade-off (PAPER's TPMG(full) vs
    # TPMG(partial) vs tensor-product): the same PCG solve with partial and full (dense) hatted
    # coefficients, at BASELINE config 2's size so that the default run stays short -----------
    coef_modes = None
    if world == 1 and not args.no_coef and args.config == "3":
        P2 = synth.baseline_config(2)
        coef_modes = {"workload": f"{P2.name}: PCG + V(1,1) to 1e-8, one warm and one timed solve",
                      "coef_bytes_per_dof": {"factorized": 0, "partial": 8, "full": 48}}
        f2 = P2.rhs()
        for mode in ("factorized", "partial", "full"):
            Q = P2 if mode == "factorized" else synth.with_coefficients(P2, mode)
            h2 = tpmg.Hierarchy(ctx, Q)
            ff2, x2 = h2.field().upload(f2), h2.field()
            tpmg.pcg_solve(h2, ff2, x2, Q.tol, args.max_iter)  # warm (captures the graph)
            torch.cuda.synchronize()
            e6, e7 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e6.record(stream)
            r6 = tpmg.pcg_solve(h2, ff2, x2, Q.tol, args.max_iter)
            e7.record(stream)
            e7.synchronize()
            ms6 = e6.elapsed_time(e7)
            coef_modes[mode] = {"ms_per_solve": ms6, "iterations": r6.iterations,
                                "gdof_per_s": Q.n_dof * r6.iterations / (ms6 * 1e-3) / 1e9,
                                "jacobi_ms": h2.time_kernel(tpmg.K_JACOBI, h2.finest, reps=10)}
            del ff2, x2
            h2.close()

    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(prof_json) and top is not None:
        try:
            with open(prof_json) as fh:
                traffic = json.load(fh).get(top, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    roofline = None
    if top is not None:
        k = kernels_live[top]
        roofline = {"bound": "hbm", "kernel": f"{k['kernel']} (finest level; largest share of "
                                              f"the timed solves)",
                    "achieved": k["GBps"], "peak": peak, "unit": "GB/s", "frac": k["frac"],
                    "traffic": traffic, "algorithmic_bytes": k["algorithmic_bytes"],
                    "launch_ms": k["avg_ms"], "launches_timed": k["launches"],
                    "timing": "CUDA events around each launch (library stream, event nodes in "
                              "the iteration graphs) over K solves run right after the timed "
                              "region, identical to it but for the event nodes",
                    "probed_ms_per_step": probed_ms / args.steps,
                    "peak_kind": peak_kind}

    line = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based RNG, BASELINE.json config shapes)",
        "config": config_dict(P, workload, px, py, h.n_levels),
        "pcg_iterations_per_s": it_per_s, "pcg_iterations_per_solve": iters,
        "vcycle_gdof_per_s": N_dof / (vcycle_ms * 1e-3) / 1e9, "vcycle_ms": vcycle_ms,
        "gpu_launches": launches,
        "roofline": roofline,
        "kernels_live": kernels_live,
        "kernels_standalone": standalone,
        "parity": parity,
        "coef_modes": coef_modes,
        "e2e": {"value": e2e_value, "unit": "GDOF/s", "h2d_bytes_per_step": 8 * n_local,
                "d2h_bytes_per_step": 8 * n_local, "ms_per_step": e2e_ms / args.steps,
                "layout": "host buffers in the reference's k-fastest Field order (pinned)",
                "api": "tpmg_pcg_host_batch: K right-hand sides, each step's upload / download "
                       "overlapped with the neighbouring steps' solves; host clock around the call"},
        "clocks": clk.summary(),
    }
    # ---- CPU baseline: oracle port on the host cores (rank 0, N = 1 only) -----------------------
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            Q, what = cpu_sample_problem(P)
            t_cpu, its = CpuPort(Q, threads).sample(iters=2)
            line["cpu_baseline"] = {"value": Q.n_dof * its / t_cpu / 1e9, "unit": "GDOF/s",
                                    "cores": threads, "kind": "port",
                                    "sample": f"{Q.name} ({what}): {its} PCG iterations of an "
                                              f"oracle solve ({t_cpu / its:.2f} s/iteration)"}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": "GDOF/s", "cores": 0, "kind": "port",
                                    "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
