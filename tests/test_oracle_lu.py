"""Pins of the tiled-LU oracle (oracle/oracle_lu.c, LU1-LU7)
against things other than itself:

* LAPACK's dgetrf (scipy.linalg.lu_factor, partial pivoting) where the tiled kernels reduce to
  it: GETRF of one tile at s = b; TSTRF at s = b, which is LU with partial pivoting of the
  stacked [U; A]; one tile row (GETRF + GESSM = dgetrf of the wide matrix);
* at s < b the same pivots, and LAPACK's L recovered by applying the later blocks'
  interchanges to each block's multipliers (the incremental storage of LU3);
* the defining identity of the whole factorization: the recorded transformation M (every
  interchange and elimination, replayed by oracle_lu_apply) maps A to the oracle's own U,
  with zeros below it; solves; the determinant's sign and magnitude (numpy slogdet);
* partial-pivoting invariants (|multipliers| <= 1), degenerate inputs, the flop count's
  limits (the paper's "50% higher" at s = b).
"""
import numpy as np
import pytest
import scipy.linalg as sl

import oracle
import tqr_inputs


def _rand(m, n, seed, dist="uniform"):
    return tqr_inputs.make(m, n, dist, seed)


# ---- GETRF (LU1) -------------------------------------------------------------------------------
@pytest.mark.parametrize("b,seed", [(8, 1), (16, 2), (32, 3), (64, 4)])
def test_getrf_s_eq_b_is_lapack_dgetrf(b, seed):
    A = _rand(b, b, seed)
    LU, piv = oracle.lu_getrf(A, b)
    lu, pv = sl.lu_factor(A)
    assert np.array_equal(piv, pv.astype(np.int32))
    assert np.max(np.abs(LU - lu)) <= 1e-13 * b


def _later_swaps(Lc, piv, c_from):
    """apply row interchanges c <-> piv[c], c >= c_from, to the rows of Lc (in place)"""
    for c in range(c_from, len(piv)):
        r = piv[c]
        if r != c:
            Lc[[c, r], :] = Lc[[r, c], :]
    return Lc


@pytest.mark.parametrize("b,s,seed", [(16, 4, 5), (32, 8, 6), (64, 16, 7), (64, 8, 8)])
def test_getrf_inner_blocking_same_pivots_and_lapack_l(b, s, seed):
    A = _rand(b, b, seed)
    LU, piv = oracle.lu_getrf(A, s)
    lu, pv = sl.lu_factor(A)
    assert np.array_equal(piv, pv.astype(np.int32))
    assert np.max(np.abs(np.triu(LU) - np.triu(lu))) <= 1e-13 * b
    Lref = np.tril(lu, -1)
    for c0 in range(0, b, s):
        blk = np.tril(LU, -1)[:, c0:c0 + s].copy()
        blk = _later_swaps(blk, piv, c0 + s)
        assert np.max(np.abs(blk - Lref[:, c0:c0 + s])) <= 1e-13 * b, c0
    # (the storage really is incremental: without the later swaps the columns differ)
    if b // s > 1:
        assert np.max(np.abs(np.tril(LU, -1) - Lref)) > 1e-3


# ---- TSTRF (LU3) ---------------------------------------------------------------------------------
def _u_and_a(b, seed):
    U = np.triu(_rand(b, b, seed)) + np.diag(np.full(b, 0.25))
    A = _rand(b, b, seed + 100)
    return U, A


@pytest.mark.parametrize("b,seed", [(8, 11), (16, 12), (32, 13)])
def test_tstrf_s_eq_b_is_lapack_on_the_stacked_matrix(b, seed):
    U, A = _u_and_a(b, seed)
    # GETRF's multipliers in U's strict lower part must survive untouched
    Ukk = U + np.tril(np.full((b, b), 7.0), -1)
    U2, A2, Lt, piv = oracle.lu_tstrf(Ukk, A, b)
    lu, pv = sl.lu_factor(np.vstack([U, A]))
    assert np.array_equal(np.tril(U2, -1), np.tril(Ukk, -1))
    exp = np.where(piv < 0, np.arange(b), b + piv)
    assert np.array_equal(exp, pv)
    assert np.max(np.abs(np.triu(U2) - np.triu(lu[:b]))) <= 1e-13 * b
    assert np.max(np.abs(Lt.reshape(b, b, order="F") - np.tril(lu[:b], -1))) <= 1e-13 * b
    assert np.max(np.abs(A2 - lu[b:])) <= 1e-13 * b


@pytest.mark.parametrize("b,s,seed", [(16, 4, 21), (32, 8, 22), (64, 16, 23), (32, 4, 24)])
def test_tstrf_inner_blocking_same_pivots_and_lapack_l(b, s, seed):
    U, A = _u_and_a(b, seed)
    U2, A2, Lt, piv = oracle.lu_tstrf(U, A, s)
    _, _, _, piv_b = oracle.lu_tstrf(U, A, b)
    assert np.array_equal(piv, piv_b)
    lu, pv = sl.lu_factor(np.vstack([U, A]))
    assert np.max(np.abs(np.triu(U2) - np.triu(lu[:b]))) <= 1e-13 * b
    Lref = np.vstack([np.tril(lu[:b], -1), lu[b:]])
    Lts = Lt.reshape(s, b, order="F")
    for c0 in range(0, b, s):
        blk = np.zeros((2 * b, s))
        blk[c0:c0 + s, :] = Lts[:, c0:c0 + s]
        blk[b:, :] = A2[:, c0:c0 + s]
        for c in range(c0 + s, b):   # the later blocks' interchanges (stacked rows c <-> b + r)
            if piv[c] >= 0:
                blk[[c, b + piv[c]], :] = blk[[b + piv[c], c], :]
        assert np.max(np.abs(blk - Lref[:, c0:c0 + s])) <= 1e-13 * b, c0
    for c0 in range(0, b, s):   # Ltilde_l is strictly lower triangular
        assert np.all(np.triu(Lts[:, c0:c0 + s]) == 0)


def test_tstrf_zero_lower_block_keeps_u():
    b, s = 16, 4
    U, _ = _u_and_a(b, 31)
    U2, A2, Lt, piv = oracle.lu_tstrf(U, np.zeros((b, b)), s)
    assert np.array_equal(np.triu(U2), np.triu(U)) and np.all(A2 == 0) and np.all(Lt == 0) and np.all(piv == -1)


# ---- GESSM / SSSSM = the recorded transformation ---------------------------------------------------
@pytest.mark.parametrize("b,s", [(16, 4), (32, 32)])
def test_gessm_applies_getrf_transformation(b, s):
    A = _rand(b, b, 41)
    C = _rand(b, b, 42)
    LU, piv = oracle.lu_getrf(A, s)
    # the GETRF of the augmented [A C] (one tile row, two tile columns) computes GESSM on C
    At, Lt, pv = oracle.lu_getrf_tiles(np.hstack([A, C]), b, s)
    C2 = oracle.lu_gessm(LU, piv, C, s)
    assert np.array_equal(oracle.unpack(At, b, 2 * b, b)[:, b:], C2)
    # and at s = b it is L^{-1} P C with LAPACK's factors
    if s == b:
        lu, pv2 = sl.lu_factor(A)
        ref = sl.lu_solve((lu, pv2), np.eye(b))  # (PLU)^{-1}
        assert np.max(np.abs(C2 - np.triu(lu) @ ref @ C)) <= 1e-11 * b


def test_ssssm_equals_explicit_elimination_matrix():
    b, s = 16, 4
    U, A = _u_and_a(b, 51)
    U2, A2, Lt, piv = oracle.lu_tstrf(U, A, s)
    # M: replay on the identity (2b x 2b) in the stacked space; M [U; A] = [U2; 0]
    I1, I2 = np.eye(2 * b)[:b], np.eye(2 * b)[b:]
    M = np.zeros((2 * b, 2 * b))
    for c in range(2 * b):
        c1, c2 = oracle.lu_ssssm(A2, Lt, piv, I1[:, c:c + 1].repeat(b, 1), I2[:, c:c + 1].repeat(b, 1), s)
        M[:b, c], M[b:, c] = c1[:, 0], c2[:, 0]
    S = np.vstack([U, A])
    R = M @ S
    assert np.max(np.abs(R[:b] - np.triu(U2))) <= 1e-12 * b
    assert np.max(np.abs(R[b:])) <= 1e-12 * b
    assert abs(abs(np.linalg.det(M)) - 1.0) <= 1e-10   # interchanges and unit-lower eliminations


# ---- the tiled factorization --------------------------------------------------------------------
_SHAPES = [(64, 64, 16, 4), (67, 41, 16, 8), (41, 67, 16, 16), (96, 96, 32, 32), (128, 80, 32, 8),
           (200, 200, 64, 16), (256, 256, 64, 16), (130, 64, 32, 8), (300, 120, 32, 32)]


@pytest.mark.parametrize("m,n,b,s", _SHAPES)
def test_transformation_maps_a_to_u(m, n, b, s):
    A = _rand(m, n, 61 + m + n)
    At, Lt, piv = oracle.lu_getrf_tiles(A, b, s, nthreads=2)
    U = oracle.get_r(At, m, n, b)        # upper trapezoid of the tiles
    MA = oracle.lu_apply(At, Lt, piv, m, n, b, s, A)
    k = min(m, n)
    nA = np.linalg.norm(A)
    assert np.max(np.abs(MA[:k] - U)) <= 1e-12 * nA
    assert np.max(np.abs(MA[k:])) <= 1e-12 * nA if m > k else True
    assert np.max(np.abs(np.tril(MA[:k], -1))) <= 1e-12 * nA


@pytest.mark.parametrize("m,n,b,s", _SHAPES)
def test_multipliers_bounded_by_one(m, n, b, s):
    A = _rand(m, n, 71 + m)
    At, Lt, piv = oracle.lu_getrf_tiles(A, b, s)
    p, q = oracle.dims(m, n, b)
    T = At.reshape(q, p, b, b).transpose(1, 0, 3, 2)   # T[i, j] = tile (i, j), row-major view
    for k in range(min(p, q)):
        assert np.max(np.abs(np.tril(T[k, k], -1))) <= 1.0
        for i in range(k + 1, p):
            assert np.max(np.abs(T[i, k])) <= 1.0
    assert np.max(np.abs(Lt)) <= 1.0


@pytest.mark.parametrize("n,b,s", [(64, 16, 4), (128, 32, 8), (192, 64, 16), (96, 32, 32)])
def test_solve_and_determinant(n, b, s):
    A = _rand(n, n, 81 + n)
    At, Lt, piv = oracle.lu_getrf_tiles(A, b, s)
    X0 = _rand(n, 3, 82)
    B = A @ X0
    X = oracle.lu_solve(At, Lt, piv, n, b, s, B)
    assert np.linalg.norm(A @ X - B) <= 1e-12 * np.linalg.norm(A) * np.linalg.norm(X) * n
    # det(A) = (-1)^(#interchanges) prod diag(U)  (every GETRF piv[c] != c and TSTRF piv >= 0 is one)
    p = n // b
    U = oracle.get_r(At, n, n, b)
    nswap = 0
    P = piv.reshape(p, p, b)   # slot (i, k) at (i + k p) b: P[k, i]
    for k in range(p):
        nswap += int(np.sum(P[k, k] != np.arange(b)))
        for i in range(k + 1, p):
            nswap += int(np.sum(P[k, i] >= 0))
    sign, logdet = np.linalg.slogdet(A)
    d = np.diag(U)
    assert np.isclose(np.sum(np.log(np.abs(d))), logdet, rtol=1e-10, atol=1e-9)
    assert sign == (-1) ** nswap * np.prod(np.sign(d))


def test_one_tile_row_is_lapack_dgetrf_of_the_wide_matrix():
    for b, s, n in [(16, 16, 64), (32, 8, 96)]:
        A = _rand(b, n, 91 + n)
        At, Lt, piv = oracle.lu_getrf_tiles(A, b, s)
        lu, pv = sl.lu_factor(A)
        assert np.array_equal(piv[:b], pv.astype(np.int32))
        U = oracle.get_r(At, b, n, b)
        assert np.max(np.abs(U - np.triu(lu))) <= 1e-12 * n


@pytest.mark.parametrize("nthreads", [2, 4])
def test_threaded_bitwise_equals_sequential(nthreads):
    A = _rand(320, 256, 101)
    r1 = oracle.lu_getrf_tiles(A, 32, 8, nthreads=1)
    r2 = oracle.lu_getrf_tiles(A, 32, 8, nthreads=nthreads)
    assert all(np.array_equal(x, y) for x, y in zip(r1, r2))


def test_degenerate_inputs():
    # zero matrix: no interchanges, no NaN, U = 0
    At, Lt, piv = oracle.lu_getrf_tiles(np.zeros((48, 40)), 16, 4)
    assert np.all(At == 0) and np.all(Lt == 0)
    P = piv.reshape(3, 3, 16)
    assert all(np.array_equal(P[k, k], np.arange(16)) for k in range(3))
    assert all(np.all(P[k, i] == -1) for k in range(3) for i in range(k + 1, 3))
    # identity: no interchanges, U = I, no multipliers
    At, Lt, piv = oracle.lu_getrf_tiles(np.eye(48), 16, 4)
    assert np.array_equal(oracle.unpack(At, 48, 48, 16), np.eye(48)) and np.all(Lt == 0)
    # 1 x 1
    At, Lt, piv = oracle.lu_getrf_tiles(np.array([[-3.0]]), 16, 8)
    assert oracle.get_r(At, 1, 1, 16)[0, 0] == -3.0
    # one column: pairwise pivoting carries the column's largest |entry| up, unchanged (no arithmetic)
    A = _rand(50, 1, 5)
    At, Lt, piv = oracle.lu_getrf_tiles(A, 16, 8)
    assert oracle.get_r(At, 50, 1, 16)[0, 0] == A[np.argmax(np.abs(A[:, 0])), 0]


def test_invalid_args():
    with pytest.raises(ValueError):
        oracle.lu_getrf(np.zeros((16, 16)), 5)   # s does not divide b
    with pytest.raises(ValueError):
        oracle.lu_getrf_tiles(np.zeros((16, 16)), 16, 0)


def test_flop_counts():
    # standard count (LAPACK dgetrf): 2/3 n^3 for square, mn^2 - n^3/3 for m >= n
    assert oracle.lu_flops_standard(3000, 3000) == pytest.approx(2.0 / 3.0 * 3000 ** 3)
    assert oracle.lu_flops_standard(4000, 1000) == pytest.approx(4000 * 1000 ** 2 - 1000 ** 3 / 3)
    # s = b: the tiled algorithm costs 50% more than LAPACK's as p grows
    r = oracle.lu_flops_tiled(64 * 64, 64 * 64, 64, 64) / oracle.lu_flops_standard(64 * 64, 64 * 64)
    assert 1.45 < r < 1.51
    # inner blocking removes most of it: overhead ~ s / 2b
    r2 = oracle.lu_flops_tiled(64 * 256, 64 * 256, 256, 32) / oracle.lu_flops_standard(64 * 256, 64 * 256)
    assert 1.0 < r2 < 1.0 + 32 / 256
    # one tile, s = b: GETRF alone = 2/3 b^3 to leading order (exact: sum of the dgetf2 loop)
    b = 64
    exact = sum((b - c - 1) + 2 * (b - c - 1) ** 2 for c in range(b))
    assert oracle.lu_flops_tiled(b, b, b, b) == exact


def test_forced_pivot_mode():
    """DESIGN.md LU10: forcing the oracle's own pivots reproduces it bit for bit; an exact tie
    forced the other way is a near-tie (valid), a non-maximal pivot is invalid."""
    A = _rand(96, 96, 123)
    At, Lt, piv = oracle.lu_getrf_tiles(A, 32, 8)
    At2, Lt2, piv2, nt, ni = oracle.lu_getrf_tiles_forced(A, 32, 8, piv)
    assert np.array_equal(At, At2) and np.array_equal(Lt, Lt2) and np.array_equal(piv, piv2) and nt == ni == 0
    T = np.array(A)
    amax = int(np.argmax(np.abs(T[:32, 0])))
    other = 5 if amax != 5 else 6
    T[other, 0] = -T[amax, 0]                          # an exact tie in the first column of tile 0
    _, _, pt = oracle.lu_getrf_tiles(T, 32, 8)
    assert pt[0] == min(amax, other)
    f = pt.copy()
    f[0] = max(amax, other)
    _, _, _, nt, ni = oracle.lu_getrf_tiles_forced(T, 32, 8, f)
    assert nt >= 1
    bad = piv.copy()
    bad[1] = (bad[1] + 3) % 32 if (bad[1] + 3) % 32 >= 1 else 2
    _, _, _, nt, ni = oracle.lu_getrf_tiles_forced(A, 32, 8, bad)
    assert ni >= 1
