"""Summarise ncu outputs into profiles/ (run here, on the CPU box, after a gpurun call).

    python tests/ncu_summary.py launches <launches.csv> <out.md>
        per-kernel share of one PCG solve (the second half of the launch list = the timed solve)
    python tests/ncu_summary.py full <report.ncu-rep> <out.md> [--traffic-json profiles/jacobi_traffic.json]
        key metrics of each captured launch (duration, DRAM bytes, throughput, occupancy, IPC)
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


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        full(sys.argv[2], sys.argv[3], tj)
