"""Aggregate the warp-stall samples of an `ncu --page source --csv --print-source sass` dump
(profiling helper, not a pytest file): top instructions and per-reason totals."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    idx = h.index("Warp Stall Sampling (All Samples)")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    data = []
    for i, r in enumerate(rows[2:]):
        if len(r) > idx and r[idx].isdigit():
            st = {c: int(r[h.index(c)] or 0) for c in reasons}
            data.append((int(r[idx]), i, r[1].strip(), st))
    tot = sum(d[0] for d in data) or 1
    print("total samples", tot, "instructions", len(data))
    agg = collections.Counter()
    for d in data:
        agg.update(d[3])
    for k, v in agg.most_common(10):
        print(f"  {k:22s} {v * 100 / tot:5.1f}%")
    for d in sorted(data, key=lambda x: -x[0])[:top]:
        main_r = sorted(d[3].items(), key=lambda x: -x[1])[:2]
        print(f"{d[0] * 100 / tot:5.2f}% #{d[1]:5d} {d[2][:70]:70s} "
              + " ".join(f"{k[6:]}={v}" for k, v in main_r))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
