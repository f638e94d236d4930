"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum]
--csv` launch list: per kernel, launch count, total device time, share of the step and (when
captured) DRAM bytes per launch. ncu launches are cold-cache and serialised: compare SHARES with
bench.py's in-run numbers, not absolutes."""
import collections
import csv
import sys


def summarize(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tscale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        val = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            agg[name][0] += 1
            agg[name][1] += val * tscale[r[ui]]
        elif r[mi].startswith("dram__bytes"):
            agg[name][2] += val * bscale[r[ui]]
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':64s} {'launches':>8s} {'total_us':>12s} {'share':>6s} {'dram_B/launch':>14s}"]
    for k, (n, us, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k[:64]:64s} {n:8d} {us:12.1f} {us / tot:6.3f} {by / max(n, 1):14.4g}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
