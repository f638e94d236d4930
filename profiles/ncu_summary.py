"""Summarise `ncu --set full` raw-page CSV exports (tools/ncu_capture.sh): per captured kernel the
device time, SM clock, DRAM bytes, tensor-pipe / TMEM / issue / L2 / shared-memory activity and
the top warp-stall reasons; with the source-page export, the SASS lines with the most stall
samples. usage: python profiles/ncu_summary.py <prefix> [<prefix> ...]   (prefix = path without
_raw.csv, e.g. gpurun_out/r02b_e2_hist)"""
import csv
import gzip
import os
import sys

KEYS = [
    ("time", "gpu__time_duration.sum"),
    ("sm clock", "sm__cycles_elapsed.avg.per_second"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM throughput % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor pipe active % (realtime)",
     "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("TMEM (mem_tensor) active %", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("L2 throughput %", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 read hit rate %", "lts__t_sector_op_read_hit_rate.pct"),
    ("smem LSU wavefronts %", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("registers / thread", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
]


def raw(prefix):
    rows = list(csv.reader(open(prefix + "_raw.csv")))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def summarize(prefix):
    d = raw(prefix)
    out = [f"== {os.path.basename(prefix)}: {d.get('Kernel Name', ('?',))[0][:100]}"]
    for label, key in KEYS:
        if key in d:
            v, u = d[key]
            out.append(f"   {label:34s} {v} {u}")
    stalls = sorted(((k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v or 0))
                     for k, (v, _) in d.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                    key=lambda x: -x[1])[:6]
    out.append("   stalls per issued instruction: " + ", ".join(f"{k} {v:.2f}" for k, v in stalls))
    src = prefix + "_source.csv.gz"
    if os.path.exists(src):
        rows = list(csv.reader(gzip.open(src, "rt")))
        hdr = rows[1]
        ia, isrc, iall = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
        cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        data = rows[2:]
        tot = sum(int(r[iall] or 0) for r in data) or 1
        out.append(f"   top SASS lines by stall samples (of {tot}):")
        for r in sorted(data, key=lambda r: -int(r[iall] or 0))[:8]:
            why = max(((hdr[i][6:], int(r[i] or 0)) for i in cols), key=lambda x: x[1])
            out.append(f"     {100.0 * int(r[iall]) / tot:5.1f}%  {r[isrc].strip()[:64]:64s} ({why[0]})")
    return "\n".join(out)


if __name__ == "__main__":
    print("\n".join(summarize(p) for p in sys.argv[1:]))
