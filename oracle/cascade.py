"""Float64 CPU oracle for the fast cascade algorithm of G. Beylkin, arXiv 2411.17729.

TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT. Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs may import this module. It shares no code
with paper_2411_17729_b200/ (the CUDA path); both read their inputs from synth/.

Plain, slow, obviously-correct float64 implementations, each citing PAPER.md (reference
path /root/reference/PAPER.md; line numbers of that file):

  powers          Abar^(2^k) by repeated squaring              PAPER.md:164-166 (§2 end)
  recurrence      x_n = Abar x_{n-1} + Bbar u_n, y = Cx + Du    PAPER.md:47-50 (Eq. 2), x_{-1}=0 :109
  cascade         v^(0) = Bbar u; N+1 shifted stages; y=Cv+Du   PAPER.md:185-229 (§3, eq:step1-3)
  cascade_window  the same on an input window (exact, R20)      derived from PAPER.md:126 + §3
  kernel_taps     h_j = C Abar^j Bbar by iterated application   PAPER.md:176-178 (Eq. 8)
  convolution     y_l = sum_j h_j u_{l-j} + D u_l               PAPER.md:176-178 (Eq. 8, reading R2)
  transfer        H(z) = C (I - z^-1 Abar)^-1 Bbar + D          PAPER.md:69-71 (Eq. 3)
  transfer_N      H_N(z) = C prod_{n=0..N} (I + (z^-1 Abar)^(2^n)) Bbar + D   PAPER.md:132-135 (Eq. 5)
  lemma1_bound    gamma^(2^(N+1)) / (1-gamma) ||C|| ||Bbar||    PAPER.md:143-153 (Lemma 1)

Readings of the paper taken here (all listed in DESIGN.md §readings):
  R1  N+1 stages k = 0..N with shifts 2^k (product n=0..N; the §3 narration's
      n=1..N with Abar^(2^(n-1)) is the same set of stages, off by one in its labels).
  R2  Eq. 8's "+ D u_k" inside the sum is read as "+ D u_l" outside it (Eq. 2/3 require it).
  R3  "At each step l=0,2,...,L-1" is the stage loop.
  R19 stages applied in the ascending order of PAPER.md:193-225, each out of place.
  R20 stages with 2^k >= L are the identity on a length-L block and are skipped.

Signal layout: u [batch][L][p], y [batch][L][q] (time along axis 1); the shift is
within each sequence, never across batch entries (column l - 2^k < 0 gets "no update").
"""
from __future__ import annotations

import numpy as np


# ---------------------------------------------------------------------------------------------
# a1: powers by repeated squaring -- PAPER.md:164-166 ("compute the powers of the matrix
#     Abar, Abar^2, Abar^4, Abar^8, ..."), accuracy remark PAPER.md:274-277
# ---------------------------------------------------------------------------------------------
def powers(Abar: np.ndarray, N: int) -> list[np.ndarray]:
    """[P_0, ..., P_N] with P_0 = Abar and P_{k+1} = P_k P_k, so P_k = Abar^(2^k)."""
    P = [np.array(Abar, dtype=np.float64)]
    for _ in range(N):
        P.append(P[-1] @ P[-1])
    return P


# ---------------------------------------------------------------------------------------------
# the direct recurrence -- PAPER.md:47-50 (Eq. 2), with x_{-1} = 0
# ---------------------------------------------------------------------------------------------
def recurrence(Abar, Bbar, C, D, u: np.ndarray, return_states: bool = False):
    """y_n = C x_n + D u_n with x_n = Abar x_{n-1} + Bbar u_n, x_{-1} = 0.  u: [batch][L][p]."""
    u = np.asarray(u, dtype=np.float64)
    batch, L, _ = u.shape
    m = Abar.shape[0]
    x = np.zeros((batch, m))
    xs = np.zeros((batch, L, m)) if return_states else None
    y = np.zeros((batch, L, C.shape[0]))
    for n in range(L):
        x = x @ Abar.T + u[:, n, :] @ Bbar.T          # x_n = Abar x_{n-1} + Bbar u_n
        y[:, n, :] = x @ C.T + u[:, n, :] @ D.T       # y_n = C x_n + D u_n
        if return_states:
            xs[:, n, :] = x
    return (y, xs) if return_states else y


# ---------------------------------------------------------------------------------------------
# the cascade -- PAPER.md:185-229 (§3), stage k adds Abar^(2^k) v_{l-2^k} for l >= 2^k
# ---------------------------------------------------------------------------------------------
def effective_stages(L: int, N: int) -> int:
    """#{k in 0..N : 2^k < L}  (R20)."""
    return sum(1 for k in range(N + 1) if (1 << k) < L)


def cascade_states(P: list[np.ndarray], Bbar, u: np.ndarray, N: int) -> np.ndarray:
    """v^(N+1) for every column: [batch][L][m].  P must hold P_0..P_N (at least)."""
    u = np.asarray(u, dtype=np.float64)
    L = u.shape[1]
    V = u @ Bbar.T                                     # v_l^(0) = Bbar u_l
    for k in range(N + 1):                             # N+1 stages (R1)
        s = 1 << k
        if s >= L:                                     # identity on the block (R20)
            break
        Vn = V.copy()                                  # out of place
        Vn[:, s:, :] = V[:, s:, :] + V[:, :L - s, :] @ P[k].T   # v_l <- Abar^(2^k) v_{l-2^k} + v_l
        V = Vn                                         # columns l < 2^k unchanged
    return V


def cascade(P: list[np.ndarray], Bbar, C, D, u: np.ndarray, N: int) -> np.ndarray:
    """y_l = C v_l^(N+1) + D u_l."""
    u = np.asarray(u, dtype=np.float64)
    V = cascade_states(P, Bbar, u, N)
    return V @ C.T + u @ D.T


def cascade_window(P, Bbar, C, D, u_window: np.ndarray, N: int, l0: int, lo: int) -> np.ndarray:
    """y on [l0, l0+W) from the input window u[lo : l0+W) with lo = max(0, l0 - 2^(N+1) + 1).

    Exact (not approximate): y_l of the truncated cascade depends only on u_{l-2^(N+1)+1..l},
    because the product of the N+1 factors is a polynomial of degree 2^(N+1)-1 in the shift
    (PAPER.md:137-141). Padding the window on the left with the zeros of x_{-1} = 0 when
    lo = 0 keeps the time origin. Returns [batch][W][q].
    """
    y = cascade(P, Bbar, C, D, u_window, N)
    return y[:, l0 - lo:, :]


def window_start(l0: int, N: int) -> int:
    return max(0, l0 - (1 << (N + 1)) + 1)


# ---------------------------------------------------------------------------------------------
# Eq. 8: the convolution-sum form, used as a brute-force check on small sizes
# ---------------------------------------------------------------------------------------------
def kernel_taps(Abar, Bbar, C, K: int) -> np.ndarray:
    """h_j = C Abar^j Bbar for j = 0..K-1 by iterated application of Abar (never a dense power)."""
    taps = np.zeros((K, C.shape[0], Bbar.shape[1]))
    W = np.array(Bbar, dtype=np.float64)
    for j in range(K):
        taps[j] = C @ W
        W = Abar @ W
    return taps


def convolution(taps: np.ndarray, D, u: np.ndarray) -> np.ndarray:
    """y_l = sum_{j=0}^{min(l, K-1)} h_j u_{l-j} + D u_l  (Eq. 8 with reading R2)."""
    u = np.asarray(u, dtype=np.float64)
    batch, L, _ = u.shape
    K = taps.shape[0]
    y = u @ D.T
    for j in range(min(K, L)):
        y[:, j:, :] += u[:, :L - j, :] @ taps[j].T
    return y


# ---------------------------------------------------------------------------------------------
# z-domain (test helpers): Eq. 3, Eq. 5, Lemma 1
# ---------------------------------------------------------------------------------------------
def transfer(Abar, Bbar, C, D, z: complex) -> np.ndarray:
    """H(z) = C (I - z^-1 Abar)^-1 Bbar + D, by one complex solve."""
    m = Abar.shape[0]
    return C @ np.linalg.solve(np.eye(m) - Abar / z, Bbar.astype(complex)) + D


def transfer_N(P: list[np.ndarray], Bbar, C, D, z: complex, N: int) -> np.ndarray:
    """H_N(z) = C prod_{n=0}^{N} [I + (z^-1 Abar)^(2^n)] Bbar + D  (Eq. 5),
    with (z^-1 Abar)^(2^n) = z^-(2^n) P_n (powers of PAPER.md:164-166)."""
    W = Bbar.astype(complex)
    for n in range(N + 1):
        W = W + (z ** -(1 << n)) * (P[n] @ W)
    return C @ W + D


def lemma1_bound(Abar, Bbar, C, N: int) -> float:
    """gamma^(2^(N+1)) / (1 - gamma) ||C||_2 ||Bbar||_2, gamma = sigma_max(Abar) < 1 (Lemma 1)."""
    gamma = np.linalg.norm(Abar, 2)
    if gamma >= 1.0:
        return float("inf")
    return float(gamma ** (2 ** (N + 1)) / (1.0 - gamma) * np.linalg.norm(C, 2) * np.linalg.norm(Bbar, 2))


# ---------------------------------------------------------------------------------------------
# workload-level drivers (banks of independent channels; the same maps per channel)
# ---------------------------------------------------------------------------------------------
def apply_workload(wl, u: np.ndarray | None = None, channels=None, method: str = "cascade") -> np.ndarray:
    """y [n_sel][batch][L][q] for the selected channels of a synth Workload (float64)."""
    chans = range(wl.n_ch) if channels is None else channels
    u = wl.u_all() if u is None else u
    out = []
    for c in chans:
        Ab, Bb, C, D, N = wl.Abar[c], wl.Bbar[c], wl.C[c], wl.D[c], int(wl.N[c])
        if method == "cascade":
            out.append(cascade(powers(Ab, N), Bb, C, D, u[c], N))
        elif method == "recurrence":
            out.append(recurrence(Ab, Bb, C, D, u[c]))
        else:
            raise ValueError(method)
    return np.stack(out)


def workload_window(wl, c: int, b: int, l0: int, W: int, P=None) -> np.ndarray:
    """Exact cascade output y[c][b][l0:l0+W][:] from the minimal input window (R20 / T14)."""
    N = int(wl.N[c])
    lo = window_start(l0, N)
    uw = wl.u_window(c, b, lo, l0 + W)[None]
    P = powers(wl.Abar[c], N) if P is None else P
    return cascade_window(P, wl.Bbar[c], wl.C[c], wl.D[c], uw, N, l0, lo)[0]
