"""GPU parity of the fused persistent bank kernel (bank_fused.cu: m = 64, every channel with
Ne >= 7; one launch, states in TMEM, levels exchanged through L2 with per-tile flags) against the
float64 oracle, plus the properties its schedule must keep: results independent of the number
of sequence slots (slot reuse waits), of the L2 discard, and of how many chunks a sequence has
relative to the grid (a sequence longer than all CTAs together)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
from synth import configs as S

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2411_17729_b200 as pk
    pk.lib()
    os.environ["CASC_BANK_FUSED"] = "1"          # opt-in path, read by the library per call
    yield
    del os.environ["CASC_BANK_FUSED"]


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def run(wl, ws_budget=None):
    from paper_2411_17729_b200.runner import DeviceWorkload
    dw = DeviceWorkload(wl, ws_budget=ws_budget)
    dw.step()
    torch.cuda.synchronize()
    return dw.y_f64()


def check(wl, y, chans=None):
    chans = list(range(wl.n_ch)) if chans is None else list(chans)
    u = wl.u_all()
    ref = oracle.apply_workload(wl, u=u, channels=chans)
    Du = np.stack([u[c] @ wl.D[c].T for c in chans])
    yy = y[chans] if len(chans) != y.shape[0] else y
    e, es = rel(yy, ref), rel(yy - Du, ref - Du)
    assert np.all(np.isfinite(yy))
    print(f"{wl.name}: rel {e:.3e} state {es:.3e}")
    assert e <= 1e-5 and es <= 1e-5, (e, es)
    return e, es


@pytest.mark.parametrize("L,batch,N", [(129, 1, 7), (256, 2, 7), (300, 3, 8), (1000, 2, 9),
                                       (2049, 2, 11), (4096, 1, 12), (5000, 3, 12)])
def test_fused_single_system_shapes(L, batch, N):
    """Ne = 7 (head + tail only), ragged last tiles, chunks of fewer than 4 tiles."""
    wl = S.make_random_mimo(64, 1, 1, L=L, batch=batch, N=N, rho=0.97, mode="fp32")
    check(wl, run(wl))


def test_fused_bank_mixed_orders():
    """Channels with N from 7 to 13 (Ne from 7 to 12 at L = 3000) in one launch."""
    wl = S.make_E2(n_ch=14, L=3000, batch=3)
    wl.N[:] = 7 + (np.arange(14) % 7)
    check(wl, run(wl))


def test_fused_slot_reuse_bitwise():
    """One sequence slot (CASC_FUSED_SLOTS=1, read per call) forces every chunk of sequence q to
    wait for sequence q-1 to complete; the result must be bitwise the many-slot result."""
    wl = S.make_E2(n_ch=6, L=3000, batch=2)
    wl.N[:] = np.maximum(wl.N, 7)
    y_full = run(wl)
    os.environ["CASC_FUSED_SLOTS"] = "1"
    try:
        y_one = run(wl)
    finally:
        del os.environ["CASC_FUSED_SLOTS"]
    assert np.array_equal(y_one, y_full)
    check(wl, y_full)


def test_fused_sequence_longer_than_grid():
    """L = 2^17: 1024 tiles = 256 chunks per sequence, more than one chunk per SM, so a sequence's
    chunks wait on chunks dealt to the same CTAs in earlier rounds."""
    wl = S.make_random_mimo(64, 1, 1, L=1 << 17, batch=1, N=15, rho=0.995, mode="fp32")
    check(wl, run(wl))


def test_fused_discard_off_bitwise(tmp_path):
    """discard.global.L2 only drops dead lines: a run without it is bitwise identical."""
    wl = S.make_E2(n_ch=4, L=4096, batch=2)
    y = run(wl)
    out = tmp_path / "y.npy"
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import numpy as np, torch\n"
            "from synth import configs as S\n"
            "from paper_2411_17729_b200.runner import DeviceWorkload\n"
            "wl = S.make_E2(n_ch=4, L=4096, batch=2)\n"
            "dw = DeviceWorkload(wl); dw.step(); torch.cuda.synchronize()\n"
            "np.save(%r, dw.y_f64())\n") % (ROOT, str(out))
    env = dict(os.environ, CASC_DISCARD="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)
    assert np.array_equal(np.load(out), y)


def test_fused_matches_multikernel_path(tmp_path):
    """The fused kernel and the multi-kernel path (CASC_BANK_FUSED unset) compute the same cascade:
    both within tolerance of the oracle and of each other."""
    wl = S.make_E2(n_ch=6, L=4096, batch=2)
    y = run(wl)
    out = tmp_path / "y.npy"
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import numpy as np, torch\n"
            "from synth import configs as S\n"
            "from paper_2411_17729_b200.runner import DeviceWorkload\n"
            "wl = S.make_E2(n_ch=6, L=4096, batch=2)\n"
            "dw = DeviceWorkload(wl); dw.step(); torch.cuda.synchronize()\n"
            "np.save(%r, dw.y_f64())\n") % (ROOT, str(out))
    env = {k: v for k, v in os.environ.items() if k != "CASC_BANK_FUSED"}
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)
    y_mk = np.load(out)
    assert rel(y, y_mk) < 2e-6
    check(wl, y)


def test_fused_chunk_size_invariance_bitwise():
    """Every tile sees the same arithmetic whatever the chunking: T = 1..6 tiles per chunk
    (CASC_FUSED_T, read per call) must give bitwise identical outputs. Many chunks per CTA and
    ragged last chunks exercise the ring bookkeeping across chunk boundaries."""
    wl = S.make_E2(n_ch=40, L=5000, batch=3)
    wl.N[:] = np.maximum(wl.N, 7)
    ys = []
    for T in range(1, 7):
        os.environ["CASC_FUSED_T"] = str(T)
        try:
            ys.append(run(wl))
        finally:
            del os.environ["CASC_FUSED_T"]
    for T, y in enumerate(ys[1:], start=2):
        assert np.array_equal(y, ys[0]), T
    check(wl, ys[-1], chans=[0, 7, 19, 39])


def test_fused_many_chunks_per_cta():
    """64 channels x 4 sequences x 22 chunks: ~38 chunks per CTA, sequence slots reused."""
    wl = S.make_E2(n_ch=64, L=16384, batch=4)
    y = run(wl)
    order = np.argsort(wl.N, kind="stable")
    check(wl, y, chans=sorted({int(order[0]), int(order[32]), int(order[-1]), 5}))
