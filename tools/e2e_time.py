"""Diagnostics: median e2e ms of casc_run_host on one config (E2 / E3 / E4 / E5), then (E2) the PCIe copy rates and scattered-vs-contiguous D2H; CASC_LIB_OVERRIDE selects the build, REPS the calls, CASC_TIMING=1 prints the host pipeline timeline.
   usage (on a B200): python tools/e2e_time.py E2"""
import json, os, sys, statistics
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import configs as S
from paper_2411_17729_b200 import api as pk
cfg = sys.argv[1]
wl = {"E2": S.make_E2, "E3": S.make_E3, "E4": S.make_E4, "E5": S.make_E5}[cfg]()
from paper_2411_17729_b200.runner import DeviceWorkload
f = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
chans = list(range(wl.n_ch))
n = len(chans)
dw = DeviceWorkload(wl)
Ab_h, Bb_h, C_h = f(wl.Abar[chans]), f(wl.Bbar[chans]), f(wl.C[chans])
D_h = f(wl.D[chans]) if np.any(wl.D[chans]) else None
u_h = dw.u.cpu().reshape(n, wl.batch, wl.L, wl.p).pin_memory()
y_h = torch.empty((n, wl.batch, wl.L, wl.q), dtype=u_h.dtype).pin_memory()
del dw
torch.cuda.empty_cache()
Ns = [int(wl.N[c]) for c in chans]
need = pk.run_host_bytes(n, wl.m, wl.p, wl.q, wl.L, wl.batch, max(Ns), wl.mode)
ws = torch.empty(min(need, int(0.8 * torch.cuda.mem_get_info()[0])), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
ts = []
for i in range(int(os.environ.get("REPS", "8"))):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); pk.run_host(Ab_h, Bb_h, C_h, D_h, u_h, y_h, Ns, wl.mode, ws); b.record(st); torch.cuda.synchronize()
    if i >= min(2, int(os.environ.get("REPS", "8")) - 1): ts.append(a.elapsed_time(b))
print(json.dumps({"median_ms": statistics.median(ts), "min_ms": min(ts)}))
if cfg != "E2": sys.exit(0)
ud = torch.empty(u_h.shape, dtype=u_h.dtype, device="cuda")
def tm(fn):
    r = []
    for i in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); torch.cuda.synchronize(); r.append(a.elapsed_time(b))
    return round(statistics.median(r[1:]), 3)
s2 = torch.cuda.Stream()
def both():
    s2.wait_stream(st)
    ud.copy_(u_h, non_blocking=True)
    with torch.cuda.stream(s2): y_h.copy_(ud, non_blocking=True)
    st.wait_stream(s2)
print(json.dumps({"h2d_ms": tm(lambda: ud.copy_(u_h, non_blocking=True)), "d2h_ms": tm(lambda: y_h.copy_(ud, non_blocking=True)),
                  "both_ms": tm(both), "bytes": u_h.numel() * u_h.element_size()}))
row = wl.batch * wl.L * 4
yd = torch.empty(u_h.shape, dtype=u_h.dtype, device="cuda")
perm = np.random.default_rng(0).permutation(n)[:86]
def scattered():
    for c in perm:
        y_h[c].copy_(yd[c], non_blocking=True)
def contiguous():
    y_h[:86].copy_(yd[:86], non_blocking=True)
def tm_hidden(fn):
    r = []
    for i in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000); a.record(st); fn(); b.record(st); torch.cuda.synchronize(); r.append(a.elapsed_time(b))
    return round(statistics.median(r[1:]), 3)
ss = [torch.cuda.Stream() for _ in range(4)]
def scattered_k(k):
    def f():
        for s_ in ss[:k]: s_.wait_stream(st)
        for i, c in enumerate(perm):
            with torch.cuda.stream(ss[i % k]): y_h[c].copy_(yd[c], non_blocking=True)
        for s_ in ss[:k]: st.wait_stream(s_)
    return f
print(json.dumps({"d2h_86_scattered_ms": tm_hidden(scattered), "d2h_86_one_ms": tm_hidden(contiguous),
                  "2 streams": tm_hidden(scattered_k(2)), "4 streams": tm_hidden(scattered_k(4))}))
