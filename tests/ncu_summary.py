"""Summarise ncu outputs into profiles/ (run here, on the CPU box, after a gpurun call).

    python tests/ncu_summary.py launches <launches.csv> <out.md>
        per-kernel share of one PCG solve (the second half of the launch list = the timed solve)
    python tests/ncu_summary.py full <report.ncu-rep> <out.md> [--traffic-json profiles/jacobi_traffic.json]
        key metrics of each captured launch (duration, DRAM bytes, throughput, occupancy, IPC)
    python tests/ncu_summary.py table <report.ncu-rep> <out.md> [--peak 6558.4] [--json profiles/roofline_traffic.json]
        one row per finest-level config-3 kernel variant: algorithmic bytes | DRAM bytes | ratio |
        ncu duration | fraction of the HBM peak | fp64 pipe | issue | warps active | registers | top stalls
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

N_DOF = 1024 * 1024 * 128
COLS = 1024 * 1024


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    data = [dict(zip(hdr, r)) for r in rows[hi + 1:]]
    data = [d for d in data if d.get("Metric Name") == "gpu__time_duration.sum"]
    sel = data[len(data) // 2:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in sel:
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void tpmg::<unnamed>::", "")
        name = name.replace("tpmg::<unnamed>::", "")
        key = f"{name} grid={d.get('Grid Size', '')}"
        unit = d.get("Metric Unit", "ns")
        v = float(d["Metric Value"].replace(",", ""))
        v = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        agg[key][0] += 1
        agg[key][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"# Launch list of one config-3 PCG solve (ncu gpu__time_duration, serialised, cold cache)",
             "", f"source: `{path}`; {len(sel)} launches, {tot / 1e3:.2f} ms total "
             "(ncu serialises launches and flushes caches: compare SHARES, not absolutes)", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e3:.3f} | {100 * v[1] / tot:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:20]))


def full(rep, out, traffic_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "smsp__inst_executed.sum", "launch__grid_size",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    lines = [f"# ncu --set full summary: `{rep}`", "",
             "| metric | " + " | ".join(f"launch {i}" for i in range(len(rows) - 2)) + " |",
             "|---|" + "---|" * (len(rows) - 2)]
    recs = []
    for r in rows[2:]:
        recs.append({w: (r[i], units[i]) for w, i in idx.items()})
    for w in want:
        if w in idx:
            lines.append(f"| {w} | " + " | ".join(f"{rc[w][0]} {rc[w][1]}".strip() for rc in recs) + " |")
    # warp-state samples (where the warps wait), top 6 of the last launch
    stall = [(hdr[i], float(v.replace(",", ""))) for i, v in enumerate(rows[-1])
             if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_")
             and not hdr[i].endswith("_not_issued") and v not in ("", "n/a")]
    tot = sum(v for _, v in stall) or 1.0
    lines += ["", "| stall reason (pc samples, last launch) | share |", "|---|---|"]
    for k, v in sorted(stall, key=lambda x: -x[1])[:6]:
        lines.append(f"| {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {100 * v / tot:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json and recs:
        def val(rc, key, scale):
            v, u = rc[key]
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1) if scale else v
        rc = recs[-1]
        traffic = val(rc, "dram__bytes_read.sum", True) + val(rc, "dram__bytes_write.sum", True)
        json.dump({"kernel": rc["Kernel Name"][0][:120], "dram_bytes_per_launch": traffic,
                   "algorithmic_bytes_per_launch": 24 * N_DOF + 32 * COLS, "source": rep},
                  open(traffic_json, "w"), indent=1)


def kernel_key(name):
    """bench.py's kernels_live / kernels_standalone name and algorithmic bytes of a launch."""
    N, C = N_DOF, COLS
    m = re.search(r"k_jacobi_t3<([^>]*)>", name)
    if m:
        a = [x.strip() for x in m.group(1).split(",")]
        zero, pcgf = a[1] in ("true", "1"), int(a[6])
        if pcgf == 2:
            return "pcg_postsweep_rz", 24 * N + 32 * C
        if pcgf == 3:
            return "pcg_rupdate_presweep", 32 * N + 32 * C
        if pcgf == 1:
            return "pcg_rupdate_q_stored", 32 * N + 32 * C
        return ("jacobi_zero_guess", 16 * N + 32 * C) if zero else ("jacobi", 24 * N + 32 * C)
    if "k_pcg_ap" in name:
        return "pcg_direction_Ap", 40 * N + 32 * C
    if "k_resid_restrict_T2" in name:
        return "resid_restrict", 18 * N + 32 * C
    if "k_prolong_flat" in name:
        return "prolong_add", 18 * N
    m = re.search(r"k_apply_t3<(\d+)", name)
    if m:
        return ("apply", 16 * N + 32 * C) if m.group(1) == "0" else ("residual", 24 * N + 32 * C)
    return None, None


def table(reps, out, peak=6558.4, json_out=None):
    """`reps`: one report, or several separated by commas (one per kernel variant)."""
    best = {}
    for rep in reps.split(","):
        _table_rows(rep, peak, best)
    rep = reps
    lines = _table_lines(rep, peak, best)
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if json_out:
        json.dump(best, open(json_out, "w"), indent=1)


def _table_rows(rep, peak, best):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}

    def num(r, key):
        i = col.get(key)
        if i is None or r[i] in ("", "n/a"):
            return None
        v = float(r[i].replace(",", ""))
        u = units[i]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
                    "usecond": 1, "msecond": 1e3}.get(u, 1)

    for r in rows[2:]:
        key, alg = kernel_key(r[col["Kernel Name"]])
        if key is None:
            continue
        us = num(r, "gpu__time_duration.sum")
        dram = (num(r, "dram__bytes_read.sum") or 0) + (num(r, "dram__bytes_write.sum") or 0)
        stall = [(hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "")))
                 for i, v in enumerate(r) if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_")
                 and not hdr[i].endswith("_not_issued") and v not in ("", "n/a")]
        tot = sum(v for _, v in stall) or 1.0
        top = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(stall, key=lambda x: -x[1])[:3])
        rec = {"kernel": re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("void ", "")
               .replace("tpmg::<unnamed>::", "")[:90], "algorithmic_bytes": alg,
               "dram_bytes_per_launch": dram, "ratio": dram / alg, "ncu_us": us,
               "frac_of_peak": alg / (us * 1e-6) / 1e9 / peak,
               "fp64_pipe_pct": num(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
               "issue_pct": num(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
               "warps_active_pct": num(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
               "registers": num(r, "launch__registers_per_thread"),
               "l2_hit_pct": num(r, "lts__t_sector_hit_rate.pct"), "top_stalls": top, "source": rep}
        best[key] = rec  # the last launch of each variant (warm)


def _table_lines(rep, peak, best):
    lines = [f"# ncu --set full, finest level of BASELINE config 3 (1024^2 x 128): `{rep}`", "",
             f"Algorithmic bytes per SURVEY.md §8(d); fraction = algorithmic bytes / ncu duration / "
             f"{peak} GB/s (measured copy peak). ncu serialises and flushes caches, so durations "
             "are cold-cache (bench.py's live CUDA-event numbers are the ones reported).", "",
             "| kernel | variant | algorithmic GB | DRAM GB | DRAM/alg | ncu us | frac | fp64 pipe | "
             "issue | warps active | regs | L2 hit | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, v in best.items():
        f = lambda x, d=1: "-" if x is None else f"{x:.{d}f}"
        lines.append(f"| {k} | `{v['kernel']}` | {v['algorithmic_bytes'] / 1e9:.3f} | "
                     f"{v['dram_bytes_per_launch'] / 1e9:.3f} | {v['ratio']:.2f} | {f(v['ncu_us'])} | "
                     f"{v['frac_of_peak']:.3f} | {f(v['fp64_pipe_pct'])}% | {f(v['issue_pct'])}% | "
                     f"{f(v['warps_active_pct'])}% | {f(v['registers'], 0)} | {f(v['l2_hit_pct'])}% | "
                     f"{v['top_stalls']} |")
    return lines


if __name__ == "__main__":
    if sys.argv[1] == "table":
        pk = float(sys.argv[sys.argv.index("--peak") + 1]) if "--peak" in sys.argv else 6558.4
        js = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
        table(sys.argv[2], sys.argv[3], pk, js)
        sys.exit(0)
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        full(sys.argv[2], sys.argv[3], tj)
