"""Regenerate profiles/ncu_traffic.json (bench.py's roofline.traffic) from one round's ncu files:
dram__bytes_read.sum + dram__bytes_write.sum per launch of each config's dominant kernel class.
  E2: mean over the bank_hist_kernel launches of the launch list (<tag>_e2_launches.csv)
  E3: the captured stage launch of mimo_gemm_pair_tf32_kernel (<tag>_e3_pair_tf32_raw.csv)
  E4: mean over the stage launches of mimo_gemm_pair_kernel in the launch list (per step the
      first pair launch is the Krylov head and the last the folded output step: excluded)
usage: python tools/make_traffic.py <tag> [E2=<tag2>]   (files under profiles/; E2=<tag2> takes the
  E2 launch list from another capture of the same round)"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path):
    """[(kernel, {metric: value})] in launch order."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ii, ki, mi, vi, ui = (hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"),
                          hdr.index("Metric Value"), hdr.index("Metric Unit"))
    out = collections.OrderedDict()
    for r in rows[1:]:
        key = int(r[ii])
        name, d = out.setdefault(key, (r[ki].split("(")[0], {}))
        if r[mi].startswith("dram__bytes"):
            d[r[mi]] = float(r[vi].replace(",", "")) * BS[r[ui]]
    return list(out.values())


def dram(d):
    return d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)


def main():
    tag = sys.argv[1]
    over = dict(a.split("=", 1) for a in sys.argv[2:])
    t2 = over.get("E2", tag)
    P = os.path.join(ROOT, "profiles")
    res = {}
    e2 = [dram(d) for k, d in launches(os.path.join(P, f"{t2}_e2_launches.csv")) if "bank_hist_kernel" in k]
    res["E2"] = {"bank_stage": sum(e2) / len(e2)}
    raw = list(csv.reader(open(os.path.join(P, f"{tag}_e3_pair_tf32_raw.csv"))))
    h, u, v = raw[0], raw[1], raw[2]
    g = lambda n: float(v[h.index(n)].replace(",", "")) * BS[u[h.index(n)]]  # noqa: E731
    res["E3"] = {"mimo_tc_stage": g("dram__bytes_read.sum") + g("dram__bytes_write.sum")}
    seq = [(k, dram(d)) for k, d in launches(os.path.join(P, f"{tag}_e4_launches.csv"))]
    stage, group = [], []
    for k, b in seq + [("end", 0.0)]:
        if k.startswith("mimo_gemm_pair_kernel"):
            group.append(b)
        elif group:                      # a step's run of pair launches ends at another kernel
            stage += group[1:-1]
            group = []
    res["E4"] = {"mimo_tc_stage": sum(stage) / len(stage)}
    res["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch of the class's dominant kernel "
                    f"({tag}{'' if t2 == tag else ', E2 ' + t2}; tools/make_traffic.py): E2 = mean over {len(e2)} bank_hist_kernel launches "
                    f"({t2}_e2_launches.csv); E3 = the captured mimo_gemm_pair_tf32_kernel stage launch "
                    f"({tag}_e3_pair_tf32_raw.csv); E4 = mean over {len(stage)} stage launches of "
                    f"mimo_gemm_pair_kernel ({tag}_e4_launches.csv; Krylov head and folded output step "
                    "excluded). ncu launches are cold-cache and serialised. Used as roofline.traffic by bench.py.")
    json.dump(res, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
