"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel, launch count,
total device time and share of the step (ncu launches are cold-cache and serialised: compare
SHARES with bench.py's in-run numbers, not absolutes)."""
import collections
import csv
import sys


def summarize(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'share':>6s}"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k[:60]:60s} {n:8d} {us:12.1f} {us / tot:6.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
