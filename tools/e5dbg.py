import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2411_17729_b200 as pk
from synth import configs as S
wl = S.make_E2(n_ch=64, L=16384, batch=4)
n = wl.n_ch; Ns=[int(x) for x in wl.N]
need = pk.run_host_bytes(n, wl.m, 1, 1, wl.L, wl.batch, max(Ns), 'fp32')
one = pk.bank_workspace_bytes(1, wl.m, wl.L, wl.batch, max(Ns), 'fp32')
print('need', need/1e9, 'one', one/1e9, 'free', torch.cuda.mem_get_info()[0]/1e9)
f = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
u_h = torch.from_numpy(wl.u_storage()).reshape(n, wl.batch, wl.L, 1).pin_memory(); y_h = torch.empty_like(u_h).pin_memory()
for frac in (1.0, 0.5, 0.2):
    ws = torch.empty(int(need*frac), dtype=torch.uint8, device='cuda')
    try:
        pk.run_host(f(wl.Abar), f(wl.Bbar), f(wl.C), f(wl.D), u_h, y_h, Ns, 'fp32', ws); print(frac, 'ok', float(y_h.float().abs().sum()))
    except Exception as e: print(frac, e)
