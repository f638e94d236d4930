"""Float64 CPU oracle: partitioned low rank (PLR) representation of Abar and its powers.

TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT (same import rule as oracle/cascade.py). Shares
no code with paper_2411_17729_b200/.

PAPER.md:292-298 (§5 "Structured representation of matrices"): "the matrix in (eq:hippo-discrete)
admits the so-called partitioned low rank representation (PLR) ..., where the rank of the
off-diagonal blocks is equal to 1. The cost of applying the m x m matrix (10) and its powers in
PLR representation does not exceed O(m log m)." The paper gives no construction; the readings
(R32) follow SPEC.md:338-396:

  plr_build        dyadic midpoint split (ceil(n/2) / floor(n/2)) down to leaves of <= leaf
                   rows, dense leaves, every off-diagonal block truncated by its SVD keeping the
                   singular values sigma_i > eps * ||a||_2 (the threshold is
                   relative to the whole matrix, not to the block's sigma_1 as SPEC.md:392 has it:
                   a block of pure round-off, e.g. the upper part of a computed lower-triangular
                   Abar, would otherwise keep full rank -- reading R32)
  plr_matvec       recursive apply: leaves dense, off-diagonal blocks as U (V^T x); flop count
                   recorded
  plr_dense        the dense matrix a PLR tree stands for (reconstruction)
  plr_power_build  each power Abar^(2^k) computed densely by repeated squaring, then compressed
                   independently
  cascade_plr      the cascade of PAPER.md:185-229 with every stage's P_k v applied through its
                   PLR tree (the map of oracle.cascade.cascade with P_k replaced by the
                   compressed P_k)

Node encoding: ("leaf", dense block) or ("split", n1, child_11, child_22, (U12, V12), (U21, V21))
with A[:n1, n1:] ~ U12 V12^T and A[n1:, :n1] ~ U21 V21^T (U: rows x r, V: cols x r).
"""
from __future__ import annotations

import numpy as np

from .cascade import powers


def _compress(block: np.ndarray, tol: float):
    """Truncated SVD of one off-diagonal block: keep the singular values sigma_i > tol."""
    if block.size == 0 or not np.any(block):
        return np.zeros((block.shape[0], 0)), np.zeros((block.shape[1], 0))
    U, s, Vt = np.linalg.svd(block, full_matrices=False)
    r = int(np.sum(s > tol)) if tol > 0 else int(np.sum(s > 0))
    return U[:, :r] * s[:r], Vt[:r, :].T


def plr_build(a: np.ndarray, eps: float, leaf_size: int = 16, _tol: float | None = None):
    """PLR tree of the square matrix a; off-diagonal singular values at or
    below eps * ||a||_2 are dropped (R32)."""
    a = np.asarray(a, dtype=np.float64)
    tol = eps * (np.linalg.norm(a, 2) if a.size else 0.0) if _tol is None else _tol
    n = a.shape[0]
    if n <= leaf_size:
        return ("leaf", a.copy())
    n1 = (n + 1) // 2                                  # midpoint split, ceil / floor
    return ("split", n1, plr_build(a[:n1, :n1], eps, leaf_size, tol), plr_build(a[n1:, n1:], eps, leaf_size, tol),
            _compress(a[:n1, n1:], tol), _compress(a[n1:, :n1], tol))


def plr_dense(node) -> np.ndarray:
    if node[0] == "leaf":
        return node[1].copy()
    _, n1, c11, c22, (U12, V12), (U21, V21) = node
    a11, a22 = plr_dense(c11), plr_dense(c22)
    n = n1 + a22.shape[0]
    a = np.zeros((n, n))
    a[:n1, :n1] = a11
    a[n1:, n1:] = a22
    a[:n1, n1:] = U12 @ V12.T
    a[n1:, :n1] = U21 @ V21.T
    return a


def plr_ranks(node) -> list[int]:
    """Ranks of every off-diagonal block, pre-order."""
    if node[0] == "leaf":
        return []
    _, _, c11, c22, (U12, _), (U21, _) = node
    return [U12.shape[1], U21.shape[1]] + plr_ranks(c11) + plr_ranks(c22)


def plr_matvec(node, x: np.ndarray):
    """(PLR a) x for x of shape (n,) or (n, k); returns (result, flops)."""
    x = np.asarray(x, dtype=np.float64)
    k = 1 if x.ndim == 1 else x.shape[1]
    if node[0] == "leaf":
        a = node[1]
        return a @ x, 2 * a.shape[0] * a.shape[1] * k
    _, n1, c11, c22, (U12, V12), (U21, V21) = node
    x1, x2 = x[:n1], x[n1:]
    y1, f1 = plr_matvec(c11, x1)                       # A11 x1
    y2, f2 = plr_matvec(c22, x2)                       # A22 x2
    y1 = y1 + U12 @ (V12.T @ x2)                       # + A12 x2 = U12 (V12^T x2)
    y2 = y2 + U21 @ (V21.T @ x1)                       # + A21 x1 = U21 (V21^T x1)
    f = f1 + f2 + 2 * k * (U12.shape[1] * (U12.shape[0] + V12.shape[0]) + U21.shape[1] * (U21.shape[0] + V21.shape[0]))
    return np.concatenate([y1, y2], axis=0), f


def plr_power_build(Abar: np.ndarray, stages: int, eps: float, leaf_size: int = 16):
    """PLR trees of P_k = Abar^(2^k), k = 0..stages-1, each compressed on its own."""
    return [plr_build(P, eps, leaf_size) for P in powers(Abar, stages - 1)]


def cascade_plr(trees: list, Bbar, C, D, u: np.ndarray, N: int) -> np.ndarray:
    """The cascade of PAPER.md:185-229 with the stage products P_k v_{l-2^k} applied through the
    PLR trees (trees[k] for P_k): v^(0) = Bbar u; for k = 0..N with 2^k < L (R20):
    v_l <- v_l + P_k v_{l-2^k} (l >= 2^k), out of place; y = C v + D u. u: [batch][L][p]."""
    u = np.asarray(u, dtype=np.float64)
    batch, L, _ = u.shape
    V = u @ Bbar.T                                     # [batch][L][m]
    m = V.shape[2]
    for k in range(N + 1):
        s = 1 << k
        if s >= L:
            break
        Vn = V.copy()
        src = V[:, :L - s, :].reshape(-1, m).T         # columns = the shifted state vectors
        Vn[:, s:, :] = V[:, s:, :] + plr_matvec(trees[k], src)[0].T.reshape(batch, L - s, m)
        V = Vn
    return V @ C.T + u @ D.T
