"""A/B timing of one config's device step (powers + apply) for two or more library builds on ONE
box (run-to-run spread between boxes is larger than most effects): each build runs in its own
subprocess (CASC_LIB_OVERRIDE), alternating, median of the timed steps (CUDA events, L2 flushed).
usage: python tools/ab_time.py CFG [L batch] -- lib1.so lib2.so ...   (diagnostics)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys, statistics, torch
sys.path.insert(0, {root!r})
from synth import configs as S
from paper_2411_17729_b200.runner import DeviceWorkload
kw = {kw!r}
wl = {{"E2": S.make_E2, "E3": S.make_E3, "E4": S.make_E4, "E5": S.make_E5}}[{cfg!r}](**kw)
dw = DeviceWorkload(wl)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3): dw.step()
torch.cuda.synchronize()
ts = []
for _ in range({steps}):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); dw.step(); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({{"median_ms": statistics.median(ts), "min_ms": min(ts)}}))
'''


def main():
    args = sys.argv[1:]
    sep = args.index("--")
    cfg, rest, libs = args[0], args[1:sep], args[sep + 1:]
    kw = {}
    if rest:
        kw["L"] = int(rest[0])
    if len(rest) > 1:
        kw["batch"] = int(rest[1])
    res = {lib: [] for lib in libs}
    for rnd in range(3):
        for lib in libs:
            env = dict(os.environ, CASC_LIB_OVERRIDE=os.path.abspath(lib))
            out = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, kw=kw, cfg=cfg, steps=10)],
                                 env=env, capture_output=True, text=True, timeout=1200)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
            res[lib].append(line)
            print(rnd, lib, line, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
