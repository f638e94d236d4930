"""Seeded synthetic workloads E1..E5 of BASELINE.json `configs` (input generation only).

This module builds the *inputs* of the method -- the discrete LTI systems
(Abar, Bbar, C, D), the truncation order N and the input signal u -- and
nothing of the cascade itself. It is shared by the oracle side and the
product side; neither side's arithmetic lives here.

Paper anchors for the input construction:
  * HiPPO-LegS generator, 1 <= n,k <= m       PAPER.md:253-262 (Eq. 9)
  * trapezoidal discretisation                 PAPER.md:51-53, :266 (Eq. 10)
  * stability assumption |lambda(Abar)| < 1
  * N chosen so the dropped factor is small    PAPER.md:143-159 (Lemma 1), :270-273
The planner `plan_N` (a0 in SURVEY §8a) measures ||Abar^(2^(N+1))||_2 with
numpy's own matrix_power/svd: N is an input to both implementations
(reading R5), never computed by the GPU path.

Draw order (numpy default_rng(seed), PCG64, all seeds 0 -- DESIGN.md R14):
  E1: G(16x16), Bbar(16x1), C(1x16)
  E2/E5: Delta(n_ch) log-uniform, C(n_ch x m), D(n_ch)
  E3: G(256x256), r(128), theta(128), Bbar(256x64), C(64x256), D(64x64)
  E4: G(1024x1024), Bbar(1024x256), C(256x1024)
The signal u is drawn by the counter-based generator in synth.rng
(stream = 100 + config index), flat index ((c*batch + b)*L + l)*p + j.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import rng as _rng


# ----------------------------------------------------------------------------------------------
# system construction (inputs)
# ----------------------------------------------------------------------------------------------
def hippo(m: int, base: int = 1) -> np.ndarray:
    """HiPPO-LegS matrix of PAPER.md:253-262 (Eq. 9); indices n,k run base..base+m-1.

    A_nk = -sqrt(2n+1) sqrt(2k+1) (n>k), -(n+1) (n=k), 0 (n<k). The paper's 1 <= n,k <= m
    (base=1) is the only choice that reproduces its d_1 and d_100 (R9).
    """
    n = np.arange(base, base + m, dtype=np.float64)
    s = np.sqrt(2.0 * n + 1.0)
    A = -np.tril(np.outer(s, s), -1)
    A[np.diag_indices(m)] = -(n + 1.0)
    return A


def hippo_B(m: int, base: int = 1) -> np.ndarray:
    """B_n = sqrt(2n+1) (BASELINE.json configs[1]), as an m x 1 column."""
    n = np.arange(base, base + m, dtype=np.float64)
    return np.sqrt(2.0 * n + 1.0).reshape(m, 1)


def trapezoid(A: np.ndarray, B: np.ndarray | None, delta: float):
    """Abar = (I - D/2 A)^-1 (I + D/2 A), Bbar = D (I - D/2 A)^-1 B   (Eq. 10).
    Done as linear solves, never an explicit inverse."""
    m = A.shape[0]
    I = np.eye(m)
    M = I - 0.5 * delta * A
    Abar = np.linalg.solve(M, I + 0.5 * delta * A)
    Bbar = None if B is None else delta * np.linalg.solve(M, B)
    return Abar, Bbar


def exponential(A: np.ndarray, B: np.ndarray | None, delta: float):
    """Exponential (zero-order-hold) discretisation of PAPER.md:306-311 (§5):
    Abar = exp(D A), Bbar = (D A)^-1 [exp(D A) - I] D B  (= int_0^D exp(A s) ds B).

    Reading (R27): the paper prints Bbar = (DA)^-1[exp(DA) - I] DA, which is m x m and
    has no B; the dimensionally consistent zero-order hold ends in D B.
    Both blocks come from ONE matrix exponential of the augmented generator (Van Loan's identity):
        exp(D [[A, B], [0, 0]]) = [[exp(D A), int_0^D exp(A s) ds B], [0, I]],
    computed by scipy.linalg.expm (scaling and squaring with Pade; a library primitive). No
    inverse of A is formed, so the recipe holds for singular A too."""
    from scipy.linalg import expm
    m = A.shape[0]
    p = 0 if B is None else B.shape[1]
    G = np.zeros((m + p, m + p))
    G[:m, :m] = A
    if p:
        G[:m, m:] = B
    E = expm(delta * G)
    Abar = E[:m, :m].copy()
    if not np.any(np.triu(A, 1)):
        # exp of a lower-triangular matrix is lower triangular; Pade's pivoted solves can leave
        # rounding-level entries above the diagonal, which are zero in exact arithmetic
        Abar = np.tril(Abar)
    Bbar = None if B is None else E[:m, m:].copy()
    return Abar, Bbar


def discretize(A: np.ndarray, B: np.ndarray | None, delta: float, scheme: str = "trapezoid"):
    """Abar, Bbar by the bilinear/trapezoidal rule (Eq. 10, the paper's examples) or the
    exponential zero-order hold."""
    if scheme == "trapezoid":
        return trapezoid(A, B, delta)
    if scheme == "exponential":
        return exponential(A, B, delta)
    raise ValueError(scheme)


def spectral_radius(A: np.ndarray) -> float:
    return float(np.max(np.abs(np.linalg.eigvals(A))))


def n_cap_for_length(L: int) -> int:
    """Largest useful N: 2^(N+1) >= L makes the cascade exact (stages with 2^k >= L are identities)."""
    return max(0, (max(L, 2) - 1).bit_length() - 1)      # ceil(log2 L) - 1 in exact integer arithmetic


def plan_N(Abar: np.ndarray, tol: float, N_cap: int) -> int:
    """Smallest N with ||Abar^(2^(N+1))||_2 <= tol, capped at N_cap (A5, A6).

    The spectral norm is used (R5); numpy's matrix product and SVD are used as
    library primitives. Returns N_cap if the criterion is never met below the cap.
    """
    P = np.array(Abar, dtype=np.float64)
    for N in range(0, N_cap + 1):
        P = P @ P                     # now Abar^(2^(N+1))
        if np.linalg.norm(P, 2) <= tol:
            return N
    return N_cap


# ----------------------------------------------------------------------------------------------
# storage rounding (the arrays the GPU reads; the oracle reads them upcast exactly, R16)
# ----------------------------------------------------------------------------------------------
def bf16_bits_from_f32(x32: np.ndarray) -> np.ndarray:
    """IEEE round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns."""
    b = np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32)
    rounding = np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))
    out = ((b + rounding) >> np.uint32(16)).astype(np.uint16)
    nan = np.isnan(x32)
    if nan.any():
        out[nan] = np.uint16(0x7FC0)
    return out


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def round_to_storage(x: np.ndarray, mode: str) -> np.ndarray:
    """float64 values exactly representable in the storage dtype of `mode` ('fp32' | 'bf16')."""
    x32 = np.asarray(x, dtype=np.float32)
    if mode == "fp32":
        return x32.astype(np.float64)
    if mode == "bf16":
        return bf16_bits_to_f64(bf16_bits_from_f32(x32))
    raise ValueError(mode)


# ----------------------------------------------------------------------------------------------
# workloads
# ----------------------------------------------------------------------------------------------
@dataclass
class Workload:
    """n_ch independent LTI systems sharing (m, p, q); each is applied to `batch` sequences.

    Abar [n_ch][m][m], Bbar [n_ch][m][p], C [n_ch][q][m], D [n_ch][q][p] (float64; the model
    parameters are passed to both implementations in float64), N [n_ch] (int).
    Signals: u, y are [n_ch][batch][L][p|q]. kind='mimo' has n_ch == 1; kind='bank' has p=q=1.
    mode: 'fp32' (fp32 storage, fp32-accurate arithmetic) or 'bf16' (bf16 storage, fp32 accumulate).
    """
    name: str
    kind: str
    mode: str
    m: int
    p: int
    q: int
    L: int
    batch: int
    Abar: np.ndarray
    Bbar: np.ndarray
    C: np.ndarray
    D: np.ndarray
    N: np.ndarray
    u_seed: int = 0
    u_stream: int = 100
    meta: dict = field(default_factory=dict)

    @property
    def n_ch(self) -> int:
        return self.Abar.shape[0]

    def u_window(self, c: int, b: int, l0: int, l1: int) -> np.ndarray:
        """Storage-rounded u[c][b][l0:l1][:] as float64 (l0 may be negative: zeros before t=0)."""
        lo = max(l0, 0)
        out = np.zeros((l1 - l0, self.p), dtype=np.float64)
        if l1 > lo:
            start = ((c * self.batch + b) * self.L + lo) * self.p
            vals = _rng.normal(self.u_seed, self.u_stream, start, (l1 - lo) * self.p)
            out[lo - l0:] = round_to_storage(vals, self.mode).reshape(l1 - lo, self.p)
        return out

    def u_all(self) -> np.ndarray:
        """The whole storage-rounded input, float64 [n_ch][batch][L][p] (small workloads only)."""
        n = self.n_ch * self.batch * self.L * self.p
        vals = _rng.normal(self.u_seed, self.u_stream, 0, n)
        return round_to_storage(vals, self.mode).reshape(self.n_ch, self.batch, self.L, self.p)

    def u_storage(self, c0: int = 0, c1: int | None = None) -> np.ndarray:
        """u for channels [c0, c1) in its storage dtype (float32 array, or uint16 bf16 bits)."""
        c1 = self.n_ch if c1 is None else c1
        per_ch = self.batch * self.L * self.p
        n = (c1 - c0) * per_ch
        shape = (c1 - c0, self.batch, self.L, self.p)
        if self.mode == "fp32":
            buf = np.empty(n, dtype=np.float32)
            _rng.normal_chunked(self.u_seed, self.u_stream, c0 * per_ch, n, buf)
            return buf.reshape(shape)
        out = np.empty(n, dtype=np.uint16)
        chunk = 1 << 22
        start = c0 * per_ch

        def work(o):
            c = min(chunk, n - o)
            out[o:o + c] = bf16_bits_from_f32(_rng.normal32(self.u_seed, self.u_stream, start + o, c))

        from concurrent.futures import ThreadPoolExecutor
        import os
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
            list(ex.map(work, range(0, n, chunk)))
        return out.reshape(shape)

    def flops_ns(self) -> float:
        """BASELINE north_star count F = sum_c 2 m^2 L batch (N_c + 1)."""
        return float(2.0 * self.m * self.m * self.L * self.batch * np.sum(self.N + 1))

    def flops_exact(self) -> float:
        """Dense stage flops actually required: sum_c sum_{k<=N_c} 2 m^2 batch (L - 2^k)^+ (A4)."""
        tot = 0.0
        for Nc in self.N:
            for k in range(int(Nc) + 1):
                tot += 2.0 * self.m * self.m * self.batch * max(self.L - (1 << k), 0)
        return tot

    def samples(self) -> int:
        return self.n_ch * self.batch * self.L


def _stack(systems):
    Ab = np.stack([s[0] for s in systems])
    Bb = np.stack([s[1] for s in systems])
    C = np.stack([s[2] for s in systems])
    D = np.stack([s[3] for s in systems])
    return Ab, Bb, C, D


def make_E1(L: int = 4096, batch: int = 1, N: int = 11, seed: int = 0, mode: str = "fp32") -> Workload:
    """configs[0]: SISO m=16; A = -I + 0.5 G/sqrt(m), trapezoid Delta=0.05, rho(Abar) <= 0.99."""
    m = 16
    g = np.random.default_rng(seed)
    G = g.standard_normal((m, m))
    A = -np.eye(m) + 0.5 * G / math.sqrt(m)
    Abar, _ = trapezoid(A, None, 0.05)
    Abar = Abar * min(1.0, 0.99 / spectral_radius(Abar))
    Bbar = g.normal(0.0, 1.0 / math.sqrt(m), (m, 1))
    C = g.normal(0.0, 1.0 / math.sqrt(m), (1, m))
    D = np.zeros((1, 1))
    Ab, Bb, Cs, Ds = _stack([(Abar, Bbar, C, D)])
    return Workload("E1", "bank", mode, m, 1, 1, L, batch, Ab, Bb, Cs, Ds,
                    np.array([N]), u_seed=seed, u_stream=101)


def make_hippo_bank(name: str, n_ch: int, L: int, batch: int, dmin: float, dmax: float,
                    tol: float, N_cap: int | None, m: int = 64, seed: int = 0,
                    stream: int = 102, mode: str = "fp32", scheme: str = "trapezoid") -> Workload:
    """configs[1] / configs[4]: HiPPO-LegS SISO channels, Delta_c log-uniform, trapezoid Abar/Bbar
    (scheme='exponential': the zero-order hold of PAPER.md:306-311, NEXT-4), B_n = sqrt(2n+1),
    C ~ N(0,1/m), D ~ N(0,1); N_c from ||Abar^(2^(N+1))||_2 <= tol."""
    g = np.random.default_rng(seed)
    deltas = 10.0 ** g.uniform(math.log10(dmin), math.log10(dmax), n_ch)
    Cs = g.normal(0.0, 1.0 / math.sqrt(m), (n_ch, 1, m))
    Ds = g.normal(0.0, 1.0, (n_ch, 1, 1))
    A = hippo(m)
    B = hippo_B(m)
    cap = n_cap_for_length(L) if N_cap is None else min(N_cap, n_cap_for_length(L))
    Abars, Bbars, Ns = [], [], []
    for c in range(n_ch):
        Abar, Bbar = discretize(A, B, float(deltas[c]), scheme)
        Abars.append(Abar)
        Bbars.append(Bbar)
        Ns.append(plan_N(Abar, tol, cap))
    return Workload(name, "bank", mode, m, 1, 1, L, batch, np.stack(Abars), np.stack(Bbars),
                    Cs, Ds, np.array(Ns), u_seed=seed, u_stream=stream,
                    meta={"delta": deltas, "tol": tol, "N_cap": cap, "scheme": scheme})


def make_E2(n_ch: int = 256, L: int = 16384, batch: int = 4, seed: int = 0, mode: str = "fp32",
            scheme: str = "trapezoid") -> Workload:
    name = "E2" if scheme == "trapezoid" else "E2x"
    return make_hippo_bank(name, n_ch, L, batch, 1e-3, 1e-1, 1e-6, None, seed=seed, stream=102, mode=mode,
                           scheme=scheme)


def make_E5(n_ch: int = 4096, L: int = 65536, batch: int = 8, seed: int = 0, mode: str = "fp32",
            scheme: str = "trapezoid") -> Workload:
    name = "E5" if scheme == "trapezoid" else "E5x"
    return make_hippo_bank(name, n_ch, L, batch, 1e-4, 1e-1, 1e-6, 15, seed=seed, stream=105, mode=mode,
                           scheme=scheme)


def make_E3(L: int = 65536, batch: int = 16, N: int = 13, m: int = 256, p: int = 64,
            seed: int = 0, mode: str = "fp32") -> Workload:
    """configs[2]: Abar = Q Lambda Q^-1, Q = I + 0.1 G/sqrt(m); Lambda real block-diagonal with
    m/2 blocks r [[cos t, -sin t], [sin t, cos t]], r ~ U[0.5, 0.999], t ~ U[0, pi] (R11)."""
    q = p
    g = np.random.default_rng(seed)
    G = g.standard_normal((m, m))
    Q = np.eye(m) + 0.1 * G / math.sqrt(m)
    r = g.uniform(0.5, 0.999, m // 2)
    th = g.uniform(0.0, math.pi, m // 2)
    Lam = np.zeros((m, m))
    for i in range(m // 2):
        c, s = math.cos(th[i]), math.sin(th[i])
        Lam[2 * i:2 * i + 2, 2 * i:2 * i + 2] = r[i] * np.array([[c, -s], [s, c]])
    X = Q @ Lam
    Abar = np.linalg.solve(Q.T, X.T).T          # Q Lambda Q^-1
    Bbar = g.normal(0.0, 1.0 / math.sqrt(m), (m, p))
    C = g.normal(0.0, 1.0 / math.sqrt(m), (q, m))
    D = g.normal(0.0, 1.0 / math.sqrt(p), (q, p))
    Ab, Bb, Cs, Ds = _stack([(Abar, Bbar, C, D)])
    return Workload("E3", "mimo", mode, m, p, q, L, batch, Ab, Bb, Cs, Ds, np.array([N]),
                    u_seed=seed, u_stream=103)


def make_E4(L: int = 1 << 20, batch: int = 8, m: int = 1024, p: int = 256, tol: float = 1e-4,
            seed: int = 0, mode: str = "bf16", N: int | None = None) -> Workload:
    """configs[3]: A = -I + 0.9 G/sqrt(m), trapezoid Delta = 0.05 (R12), Abar <- 0.995 Abar / rho(Abar);
    Bbar, C ~ N(0, 1/m), D = 0; N from ||Abar^(2^(N+1))||_2 <= 1e-4."""
    q = p
    g = np.random.default_rng(seed)
    G = g.standard_normal((m, m))
    A = -np.eye(m) + 0.9 * G / math.sqrt(m)
    Abar, _ = trapezoid(A, None, 0.05)
    Abar = 0.995 * Abar / spectral_radius(Abar)
    Bbar = g.normal(0.0, 1.0 / math.sqrt(m), (m, p))
    C = g.normal(0.0, 1.0 / math.sqrt(m), (q, m))
    D = np.zeros((q, p))
    if N is None:
        N = plan_N(Abar, tol, n_cap_for_length(L))
    Ab, Bb, Cs, Ds = _stack([(Abar, Bbar, C, D)])
    return Workload("E4", "mimo", mode, m, p, q, L, batch, Ab, Bb, Cs, Ds, np.array([N]),
                    u_seed=seed, u_stream=104)


def make_random_mimo(m: int, p: int, q: int, L: int, batch: int, N: int, rho: float = 0.95,
                     seed: int = 7, mode: str = "fp32", zero_D: bool = False) -> Workload:
    """Generic random stable system for edge-case tests: Abar = rho * G / rho(G)."""
    g = np.random.default_rng(seed)
    G = g.standard_normal((m, m))
    Abar = rho * G / spectral_radius(G)
    Bbar = g.normal(0.0, 1.0 / math.sqrt(m), (m, p))
    C = g.normal(0.0, 1.0 / math.sqrt(m), (q, m))
    D = np.zeros((q, p)) if zero_D else g.normal(0.0, 1.0 / math.sqrt(p), (q, p))
    Ab, Bb, Cs, Ds = _stack([(Abar, Bbar, C, D)])
    kind = "bank" if (p == 1 and q == 1) else "mimo"
    return Workload(f"rand_m{m}", kind, mode, m, p, q, L, batch, Ab, Bb, Cs, Ds, np.array([N]),
                    u_seed=seed, u_stream=200)


CONFIGS = {"E1": make_E1, "E2": make_E2, "E3": make_E3, "E4": make_E4, "E5": make_E5}
