"""PLR evidence for the bank workloads: for every channel of E2
(and a channel sample of E5) build the PLR trees of its powers P_k with the float64 oracle
(oracle/plr.py, leaf 16, eps = 1e-7: the fp32 target) and report, per stage k, the largest
off-diagonal rank and the PLR matvec's flops relative to the dense lower-triangular matvec the GPU
bank pass executes (m (m + 1) flops per row and source; 2 m^2 dense). Diagnostics; calls only
oracle/ and synth/.   usage: python tools/plr_ranks.py > profiles/r02_plr_ranks.txt"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import plr as R  # noqa: E402
from synth import configs as S  # noqa: E402


def table(name, wl, chans, eps=1e-7):
    m = wl.Abar[0].shape[0]
    kmax = max(int(wl.N[c]) for c in chans) + 1
    ranks = [[] for _ in range(kmax)]
    ratio = [[] for _ in range(kmax)]
    for c in chans:
        N = int(wl.N[c])
        for k, t in enumerate(R.plr_power_build(wl.Abar[c], N + 1, eps)):
            ranks[k].append(max(R.plr_ranks(t)))
            ratio[k].append(R.plr_matvec(t, np.ones(m))[1] / (m * (m + 1)))
    print(f"{name}: {len(chans)} channels, m = {m}, leaf 16, eps = {eps:g}")
    print(" k  channels  max-rank(median/max)  PLR flops / dense-triangular (mean, min, max)")
    tot_plr = tot_tri = 0.0
    for k in range(kmax):
        if not ranks[k]:
            continue
        r, q = np.array(ranks[k]), np.array(ratio[k])
        tot_plr += q.sum()
        tot_tri += len(q)
        print(f"{k:2d}  {len(r):8d}  {int(np.median(r)):3d} / {r.max():3d}            "
              f"{q.mean():.2f}  {q.min():.2f}  {q.max():.2f}")
    print(f"all stages: PLR / dense-triangular flops = {tot_plr / tot_tri:.3f} "
          f"(dense-triangular / dense = {(m + 1) / (2 * m):.3f})\n")


if __name__ == "__main__":
    wl2 = S.make_E2()
    table("E2", wl2, range(wl2.n_ch))
    wl5 = S.make_E5()
    table("E5 (every 16th channel)", wl5, range(0, wl5.n_ch, 16))
