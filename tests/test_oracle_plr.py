"""Pins of the PLR oracle (oracle/plr.py, R32).

Each check compares with something the oracle does not compute itself: the input matrix, a
closed form, a rank fixed by linear algebra (sub-blocks of an outer product; the nullity theorem
for the inverse of a triangular matrix), or the dense cascade of oracle/cascade.py, which is
pinned on its own (tests/test_oracle_pins.py)."""
import numpy as np
import pytest

import oracle as O
from oracle import plr as R
from synth import configs as S


def _hippo_abar(m, delta):
    return S.trapezoid(S.hippo(m), None, delta)[0]


def test_identity_has_rank_zero_blocks():
    """SPEC.md:357 identity -> all off-diagonal ranks 0; the tree is I exactly."""
    for m in (64, 100):
        t = R.plr_build(np.eye(m), 1e-10)
        assert max(R.plr_ranks(t)) == 0
        assert np.array_equal(R.plr_dense(t), np.eye(m))
        x = np.random.default_rng(0).standard_normal(m)
        assert np.array_equal(R.plr_matvec(t, x)[0], x)


@pytest.mark.parametrize("m", [64, 100])
def test_strictly_lower_outer_product(m):
    """A = -tril(u v^T, -1). Every lower off-diagonal block of the dyadic tree is a
    whole sub-block of u v^T (rank exactly 1 for u, v without zeros); every upper block is zero.
    A x for x = ones has the closed form y_i = -u_i sum_{j<i} v_j (a prefix sum, no matrix)."""
    rng = np.random.default_rng(1)
    u, v = 1.0 + rng.random(m), 1.0 + rng.random(m)
    A = -np.tril(np.outer(u, v), -1)
    t = R.plr_build(A, 1e-12)
    ranks = R.plr_ranks(t)
    assert ranks[0::2] == [0] * (len(ranks) // 2)       # upper blocks (pre-order: 12 then 21)
    assert ranks[1::2] == [1] * (len(ranks) // 2)       # lower blocks
    y, flops = R.plr_matvec(t, np.ones(m))
    closed = -u * np.concatenate([[0.0], np.cumsum(v)[:-1]])
    assert np.allclose(y, closed, rtol=1e-12, atol=1e-12 * np.abs(closed).max())
    assert flops < 2 * m * m


def test_eps_zero_reproduces_the_matrix():
    """eps = 0 keeps every non-zero singular value: the input to machine precision."""
    A = np.random.default_rng(2).standard_normal((100, 100))
    t = R.plr_build(A, 0.0)
    assert np.linalg.norm(R.plr_dense(t) - A, 2) <= 1e-13 * np.linalg.norm(A, 2)


def test_exact_low_rank_structure():
    """diag + X Y^T with X, Y of 3 generic columns: every off-diagonal block is a sub-block of X Y^T,
    rank exactly 3 (generic), and the reconstruction is exact to rounding."""
    rng = np.random.default_rng(3)
    m = 64
    X, Y = rng.standard_normal((m, 3)), rng.standard_normal((m, 3))
    A = np.diag(rng.standard_normal(m)) + X @ Y.T
    t = R.plr_build(A, 1e-12)
    assert set(R.plr_ranks(t)) == {3}
    assert np.linalg.norm(R.plr_dense(t) - A, 2) <= 1e-12 * np.linalg.norm(A, 2)


def test_zero_and_diagonal_powers():
    """Abar = 0 and diagonal Abar -> every power has off-diagonal rank 0."""
    for Ab in (np.zeros((64, 64)), np.diag(np.linspace(0.1, 0.9, 64))):
        for t in R.plr_power_build(Ab, 6, 1e-10):
            assert max(R.plr_ranks(t)) == 0
        d = np.diag(Ab)
        t = R.plr_power_build(Ab, 4, 1e-10)[3]           # P_3 = Abar^8: closed form d^8 on the diagonal
        assert np.allclose(np.diag(R.plr_dense(t)), d ** 8, rtol=1e-13, atol=0)


def test_paper_hippo_abar_off_diagonal_rank_one():
    """the HiPPO Abar of Eq. 10 (the worked example's m = 100, Delta = 0.5e-3,
    PAPER.md:264-266) has off-diagonal blocks of rank 1. Linear algebra fixes it: Abar =
    -I + 2 M^-1 with M = I - Delta/2 A lower triangular whose strictly lower part is rank 1, and by the
    nullity theorem an off-diagonal block of M^-1 has the rank of the matching block of M (lower:
    1, upper: 0). The reconstruction error is within the eps of SPEC.md:359."""
    Ab = _hippo_abar(100, 0.5e-3)
    t = R.plr_build(Ab, 1e-10)
    ranks = R.plr_ranks(t)
    assert ranks[0::2] == [0] * (len(ranks) // 2) and ranks[1::2] == [1] * (len(ranks) // 2)
    assert np.linalg.norm(R.plr_dense(t) - Ab, 2) <= 1e-9 * np.linalg.norm(Ab, 2)
    _, flops = R.plr_matvec(t, np.ones(100))
    assert flops < 2 * 100 * 100


@pytest.mark.parametrize("delta", [1e-4, 1e-2, 1e-1])
def test_powers_matvec_within_bound(delta):
    """through every compressed power, ||PLR x - P_k x|| <= c_tree eps ||P_k|| ||x||,
    c_tree = 2 log2(m / leaf) + 1, against the dense powers of oracle/cascade.py (pinned T3/T4)."""
    m, eps = 64, 1e-10
    Ab = _hippo_abar(m, delta)
    P = O.powers(Ab, 14)
    trees = R.plr_power_build(Ab, 15, eps)
    c_tree = 2 * np.log2(m / 16) + 1
    X = np.random.default_rng(4).standard_normal((m, 100))
    X /= np.linalg.norm(X, axis=0)
    for k, t in enumerate(trees):
        err = np.linalg.norm(R.plr_matvec(t, X)[0] - P[k] @ X, axis=0).max()
        assert err <= c_tree * eps * np.linalg.norm(P[k], 2) + 1e-15, (k, err)


def test_cascade_plr_matches_dense_cascade():
    """eps = 0: the PLR cascade is the dense cascade (pinned against the recurrence and brute force in
    test_oracle_pins.py) to rounding; eps = 1e-10: within the eps-scaled bound."""
    rng = np.random.default_rng(5)
    m, L, N = 64, 300, 8
    A = S.hippo(m)
    Ab, Bb = S.trapezoid(A, S.hippo_B(m), 1e-2)
    C = rng.standard_normal((1, m))
    D = rng.standard_normal((1, 1))
    u = rng.standard_normal((2, L, 1))
    y_dense = O.cascade(O.powers(Ab, N), Bb, C, D, u, N)
    for eps, tol in ((0.0, 1e-12), (1e-10, 1e-8)):
        y = R.cascade_plr(R.plr_power_build(Ab, N + 1, eps), Bb, C, D, u, N)
        assert np.linalg.norm(y - y_dense) <= tol * np.linalg.norm(y_dense)


def test_rank_growth_of_the_powers_is_recorded():
    """The measurement behind DESIGN.md §9 (PLR not built on the GPU): at m = 64 and the fp32 target
    (eps = 1e-7) the off-diagonal rank of P_k grows with k before the powers decay (SPEC.md:369 'ranks
    may grow with s'); Abar itself stays rank 1 (the paper's claim)."""
    ranks = [max(R.plr_ranks(t)) for t in R.plr_power_build(_hippo_abar(64, 1e-2), 15, 1e-7)]
    assert ranks[0] == 1
    assert max(ranks) >= 16                             # half the 32 x 32 block's full rank or more
