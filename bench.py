#!/usr/bin/env python
"""Headline benchmark: PCG + TPMG V(1,1) solve of BASELINE.json config 3 (1024x1024x128,
fp64) on the sm_100a path, one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One STEP = one complete PCG solve (x0 = 0 -> |r|/|r0| <= 1e-8) of the synthetic problem.
N = 1: config 3.  N > 1 (torchrun): weak scaling, a (1024*px) x (1024*py) x 128 global grid,
1024^2 x 128 columns per GPU, decomposed horizontally (columns never split).
value = whole-job throughput in GDOF/s = global DOF x PCG iterations / second (max over
ranks).  Extra keys give PCG iterations/s, V-cycle GDOF/s, the roofline of the dominant
kernel (line-Jacobi sweep) and the CPU baseline (the oracle port on the host cores).
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


def make_problem(px: int, py: int):
    from paper_1408_2981_b200 import synth

    if px * py == 1:
        return synth.baseline_config(3)
    # config 4 (weak): 1024^2 x 128 per GPU, same h, operator and RHS distribution
    return synth.make_problem(
        1024 * px, 1024 * py, 128, omega2=1e-3, lambda2=1e-4, grading="quadratic", depth=8,
        nu=1, tol=1e-8, h=1.0 / 1024, name=f"cfg4_weak_{px}x{py}")


class CpuPort:
    """The oracle port (the reference's algorithm, parallel_for threading) on the host cores:
    seconds per PCG iteration from the solve's ConvergenceHistory seconds column."""

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
        _, hist, it, st, secs = self.o.pcg(self.f, self.P.tol, iters, seconds=True)
        return (secs[it] - secs[1]) / max(it - 1, 1) if it >= 2 else secs[it]


def cpu_port_sample(P, threads: int, iters: int = 2):
    return CpuPort(P, threads).sample(iters), iters


def run_reference(args):
    """--impl reference: the CPU restatement of the reference path (oracle port), all host
    threads, bounded sample per step (2 PCG iterations of the same config)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    P = make_problem(*proc_grid(world))
    threads = os.cpu_count() or 1
    port = CpuPort(P, threads)
    per = []
    for s in range(args.warmup + args.steps):
        t = port.sample(iters=2)
        if s >= args.warmup:
            per.append(t)
    t_iter = statistics.median(per)
    value = P.n_dof / t_iter / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GDOF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_iter * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE configs)",
        "config": {"workload": P.name, "nx": P.nx, "ny": P.ny, "nz": P.nz, "sample": "per step: 2 PCG iterations"},
        "pcg_iterations_per_s": 1.0 / t_iter,
        "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": threads, "kind": "port",
                         "sample": f"{P.name}: PCG iterations 2.. of an oracle solve, per-iteration time"},
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--max-iter", type=int, default=500)
    ap.add_argument("--no-coef", action="store_true", help="skip the coefficient-storage comparison")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1408_2981_b200 import synth, tpmg

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    px, py = proc_grid(world)
    P = make_problem(px, py)
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
    iters = []
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            res = tpmg.pcg_solve(h, f, x, P.tol, args.max_iter)
            iters.append(res.iterations)
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

    # ---- e2e: the same solve through the public API from pinned host memory ---------------------
    n_local = lnx * lny * nz
    f_pin = torch.from_numpy(f_host.reshape(-1)).pin_memory()
    x_pin = torch.empty(n_local, dtype=torch.float64).pin_memory()
    fnp, xnp = f_pin.numpy(), x_pin.numpy()
    ef = h.field()
    tpmg.pcg_solve(h, ef.upload(fnp), x, P.tol, args.max_iter)  # warm
    barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_iters = 0
    e2.record(stream)
    for _ in range(args.steps):
        ef.upload(fnp)
        r2 = tpmg.pcg_solve(h, ef, x, P.tol, args.max_iter)
        x.download(out=xnp)
        e2e_iters += r2.iterations
    e3.record(stream)
    e3.synchronize()
    barrier()
    e2e_ms = max_over_ranks(e2.elapsed_time(e3))
    e2e_value = P.n_dof * e2e_iters / (e2e_ms / 1e3) / 1e9

    # ---- dominant kernel roofline (live CUDA-event timing on the library stream) -----------------
    peak, peak_kind = _peaks()
    C_cols, N_dof = lnx * lny, n_local
    t_jac = h.time_kernel(tpmg.K_JACOBI, h.finest, reps=20)
    jac_bytes = 24 * N_dof + 32 * C_cols  # read u, f; write u'; 4 per-column scalars
    achieved = jac_bytes / (t_jac * 1e-3) / 1e9
    kernels = {}
    # algorithmic bytes: fields read + written once, 2 B/DOF for a quarter-size coarse field,
    # 32 B per column of hatted scalars
    for name, kid, by in (("pcg_direction_Ap", tpmg.K_PCG_DIRECTION, 40 * N_dof + 32 * C_cols),
                          ("pcg_rupdate_presweep", tpmg.K_PCG_RUPDATE, 32 * N_dof + 32 * C_cols),
                          ("jacobi_zero_guess", tpmg.K_JACOBI_ZERO, 16 * N_dof + 32 * C_cols),
                          ("resid_restrict", tpmg.K_RESID_RESTRICT, 16 * N_dof + 2 * N_dof + 32 * C_cols),
                          ("prolong_add", tpmg.K_PROLONG_ADD, 16 * N_dof + 2 * N_dof),
                          ("apply", tpmg.K_APPLY, 16 * N_dof + 32 * C_cols)):
        t = h.time_kernel(kid, h.finest, reps=10)
        kernels[name] = {"ms": t, "GBps": by / (t * 1e-3) / 1e9, "frac": by / (t * 1e-3) / 1e9 / peak}
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

    # ---- coefficient storage trade-off (PAPER's TPMG(full) vs
    # TPMG(partial) vs tensor-product): the same PCG solve with partial and full (dense) hatted
    # coefficients, at BASELINE config 2's size so that the default run stays short -----------
    coef_modes = None
    if world == 1 and not args.no_coef:
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
    prof_json = os.path.join(ROOT, "profiles", "jacobi_traffic.json")
    if os.path.exists(prof_json):
        try:
            with open(prof_json) as fh:
                traffic = json.load(fh).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based RNG, BASELINE.json config shapes)",
        "config": {"workload": P.name + (" (config 3)" if world == 1 else " (config 4 weak)"),
                   "global_grid": [P.nx, P.ny, P.nz], "tile": [lnx, lny, nz],
                   "solver": "PCG + TPMG V(1,1), line-Jacobi, linear/transpose transfers",
                   "tol": P.tol, "levels": h.n_levels, "process_grid": [px, py],
                   "l2": "inputs larger than L2 (1.07 GB per vector)"},
        "pcg_iterations_per_s": it_per_s, "pcg_iterations_per_solve": iters,
        "vcycle_gdof_per_s": N_dof / (vcycle_ms * 1e-3) / 1e9, "vcycle_ms": vcycle_ms,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "k_jacobi (line-Jacobi sweep, finest level)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "algorithmic_bytes": jac_bytes, "launch_ms": t_jac,
                     "peak_kind": peak_kind},
        "kernels": kernels,
        "coef_modes": coef_modes,
        "e2e": {"value": e2e_value, "unit": "GDOF/s", "h2d_bytes_per_step": 8 * n_local,
                "d2h_bytes_per_step": 8 * n_local, "ms_per_step": e2e_ms / args.steps},
        "clocks": clk.summary(),
    }
    # ---- CPU baseline: oracle port on the host cores (rank 0, N = 1 only) -----------------------
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            t_cpu, _ = cpu_port_sample(P, threads, iters=2)
            line["cpu_baseline"] = {"value": P.n_dof / t_cpu / 1e9, "unit": "GDOF/s",
                                    "cores": threads, "kind": "port",
                                    "sample": f"{P.name}: PCG iteration 2 of an oracle solve "
                                              f"({t_cpu:.2f} s/iteration)"}
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
