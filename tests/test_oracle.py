"""Pins for the CPU oracle (oracle/oracle.c) against what the paper and the mathematics fix.

Each test pins the oracle to something other than itself: worked examples
(tests/golden, cited), closed-form identities, special cases that reduce to a
textbook routine, brute force on tiny inputs, LAPACK (numpy) up to row signs,
and invariants (R^T R = A^T A, backward error, orthogonality).
"""
import json
import os

import numpy as np
import pytest

import oracle
import tqr_inputs
from conftest import GOLDEN

EPS = np.finfo(np.float64).eps


# ----------------------------------------------------------------------------------------
# independent dense helpers (textbook Householder, no tiles, no T, no blocking)
# ----------------------------------------------------------------------------------------

def dense_house(alpha, x):
    """Textbook Householder generator with the DESIGN.md R2/R3 sign/zero conventions."""
    sigma = float(np.dot(x, x))
    if sigma == 0.0:
        return alpha, 0.0, np.zeros_like(x)
    nu = np.sqrt(alpha * alpha + sigma)
    beta = -nu if alpha >= 0 else nu
    return beta, (beta - alpha) / beta, x / (alpha - beta)


def reflector(n, rows, tau, vals):
    """Dense n x n H = I - tau u u^T with u[rows] = vals."""
    u = np.zeros(n)
    u[rows] = vals
    return np.eye(n) - tau * np.outer(u, u)


def brute_force_tiled_qr(A, b):
    """Flat-tree tiled Householder QR written densely (Algorithm 1):
    every reflector is built as an explicit m x m matrix and applied eagerly to the
    whole matrix in creation order.  Returns (R_dense, Q, list of (rows, tau, v))."""
    A = np.array(A, dtype=np.float64)
    m, n = A.shape
    p, q = -(-m // b), -(-n // b)
    M = np.zeros((p * b, q * b))
    M[:m, :n] = A
    Q = np.eye(p * b)
    refl = []
    for k in range(min(p, q)):
        # GEQRT(k): column c of the diagonal tile, reflector confined to tile-row k
        for c in range(b):
            col = k * b + c
            lo, hi = col + 1, (k + 1) * b
            beta, tau, v = dense_house(M[col, col], M[lo:hi, col].copy())
            rows = list(range(col, hi))
            H = reflector(p * b, rows, tau, np.concatenate([[1.0], v]))
            M = H @ M
            M[col, col] = beta
            M[lo:hi, col] = 0.0
            Q = Q @ H
            refl.append(("G", k, k, c, tau, v))
        # TSQRT(k,i): column c, reflector = e_{kb+c} on top of tile-row i
        for i in range(k + 1, p):
            for c in range(b):
                col = k * b + c
                beta, tau, v = dense_house(M[col, col], M[i * b:(i + 1) * b, col].copy())
                rows = [col] + list(range(i * b, (i + 1) * b))
                H = reflector(p * b, rows, tau, np.concatenate([[1.0], v]))
                M = H @ M
                M[col, col] = beta
                M[i * b:(i + 1) * b, col] = 0.0
                Q = Q @ H
                refl.append(("T", k, i, c, tau, v))
    return M, Q, refl


def tile_of(At, i, j, p, b):
    off = (i + j * p) * b * b
    return At[off:off + b * b].reshape((b, b), order="F")


def tslot(T, i, k, p, s, b):
    off = (i + k * p) * s * b
    return T[off:off + s * b].reshape((s, b), order="F")


def rand(m, n, seed):
    return tqr_inputs.uniform(m, n, seed)


# ----------------------------------------------------------------------------------------
# house (SPEC.md:116-121 worked examples)
# ----------------------------------------------------------------------------------------

def test_house_golden():
    cases = json.load(open(os.path.join(GOLDEN, "house_examples.json")))["cases"]
    for c in cases:
        beta, tau, v = oracle.house(c["x"])
        assert beta == c["beta"], c["cite"]
        assert tau == c["tau"], c["cite"]
        np.testing.assert_array_equal(v, c["v"], err_msg=c["cite"])


def test_house_reflects():
    rng = np.random.default_rng(1)
    for L in (1, 2, 5, 33):
        x = rng.standard_normal(L)
        beta, tau, v = oracle.house(x)
        H = np.eye(L) - tau * np.outer(v, v)
        y = H @ x
        assert abs(y[0] - beta) <= 16 * L * EPS * np.linalg.norm(x)
        assert np.all(np.abs(y[1:]) <= 16 * L * EPS * np.linalg.norm(x))
        assert np.linalg.norm(H.T @ H - np.eye(L)) <= 16 * L * EPS
        assert 1.0 <= tau <= 2.0 or L == 1


def test_house_negative_zero_alpha():
    # DESIGN.md R2: alpha = -0.0 counts as >= 0, so beta = -nu.
    beta, tau, v = oracle.house([-0.0, 3.0])
    assert beta == -3.0 and tau == 1.0


# ----------------------------------------------------------------------------------------
# tile kernels
# ----------------------------------------------------------------------------------------

def reflectors_from_geqrt(Af, T, s):
    """Reflectors of a GEQRT output: u_c = e_c + strict-lower column c; tau_c = diag of T_l."""
    b = Af.shape[0]
    out = []
    for c in range(b):
        l, j = divmod(c, s)
        tau = T[j, l * s + j]
        u = np.zeros(b)
        u[c] = 1.0
        u[c + 1:] = Af[c + 1:, c]
        out.append((tau, u))
    return out


@pytest.mark.parametrize("b,s", [(1, 1), (4, 1), (4, 2), (4, 4), (8, 2), (16, 4), (16, 16), (12, 3)])
def test_geqrt_equals_textbook_qr(b, s):
    """s == b or s < b: GEQRT equals textbook unblocked Householder QR of the tile
    (same reflectors, same signs); T_l is the forward column-wise T."""
    A = rand(b, b, 100 + b + s)
    Af, T = oracle.geqrt(A, s)
    # textbook: dense Householder, one column at a time
    M = A.copy()
    taus, vs = [], []
    for c in range(b):
        beta, tau, v = dense_house(M[c, c], M[c + 1:, c].copy())
        u = np.concatenate([np.zeros(c), [1.0], v])
        M = M - tau * np.outer(u, u @ M)
        M[c, c] = beta
        M[c + 1:, c] = 0.0
        taus.append(tau); vs.append(v)
    tol = 100 * b * EPS * max(1.0, np.linalg.norm(A))
    np.testing.assert_allclose(np.triu(Af), np.triu(M), atol=tol, rtol=0)
    for c in range(b):
        np.testing.assert_allclose(Af[c + 1:, c], vs[c], atol=tol, rtol=0)
        l, j = divmod(c, s)
        assert abs(T[j, l * s + j] - taus[c]) <= tol
    # T_l identity: I - U_l T_l U_l^T == H_{c0} ... H_{c0+s-1}
    refl = reflectors_from_geqrt(Af, T, s)
    for l in range(b // s):
        Tl = T[:, l * s:(l + 1) * s]
        assert np.all(np.tril(Tl, -1) == 0.0)
        U = np.stack([refl[l * s + j][1] for j in range(s)], axis=1)
        P = np.eye(b)
        for j in range(s):
            tau, u = refl[l * s + j]
            P = P @ (np.eye(b) - tau * np.outer(u, u))
        np.testing.assert_allclose(np.eye(b) - U @ Tl @ U.T, P, atol=1e-13, rtol=0)
    # Q_kk^T A_kk = R_kk  with Q^T = I - U T^T U^T per block (R1)
    X = A.copy()
    for l in range(b // s):
        Tl = T[:, l * s:(l + 1) * s]
        U = np.stack([refl[l * s + j][1] for j in range(s)], axis=1)
        X = X - U @ (Tl.T @ (U.T @ X))
    np.testing.assert_allclose(X, np.triu(Af), atol=tol, rtol=0)


def test_geqrt_wrong_transpose_would_fail():
    """Guard on reading R1: the literal (I - V T V^T) A misses R for b >= 2."""
    b = 6
    A = rand(b, b, 7)
    Af, T = oracle.geqrt(A, b)
    U = np.tril(Af, -1) + np.eye(b)
    right = A - U @ (T.T @ (U.T @ A))
    wrong = A - U @ (T @ (U.T @ A))
    assert np.linalg.norm(right - np.triu(Af)) < 1e-13
    assert np.linalg.norm(wrong - np.triu(Af)) > 1e-3


def test_geqrt_identity():
    for b, s in ((4, 2), (8, 8)):
        Af, T = oracle.geqrt(np.eye(b), s)
        np.testing.assert_array_equal(Af, np.eye(b))
        np.testing.assert_array_equal(T, np.zeros((s, b)))


@pytest.mark.parametrize("b,s", [(1, 1), (3, 1), (4, 2), (4, 4), (8, 4), (16, 8)])
def test_tsqrt_equals_stacked_qr(b, s):
    """TSQRT == textbook Householder QR of the dense 2b x b stack [R; A]."""
    Rin = np.triu(rand(b, b, 200 + b))
    junk = np.tril(rand(b, b, 300 + b), -1)  # V_kk lives there: must not be read or written
    R0 = Rin + junk
    B = rand(b, b, 400 + b)
    Rf, Bf, T = oracle.tsqrt(R0, B, s)
    np.testing.assert_array_equal(np.tril(Rf, -1), junk)
    S = np.vstack([Rin, B])
    taus, vs = [], []
    for c in range(b):
        x = S[c + 1:, c].copy()
        beta, tau, v = dense_house(S[c, c], x)
        u = np.concatenate([np.zeros(c), [1.0], v])
        S = S - tau * np.outer(u, u @ S)
        S[c, c] = beta
        S[c + 1:, c] = 0
        taus.append(tau); vs.append(v)
    tol = 100 * b * EPS * max(1.0, np.linalg.norm(np.vstack([Rin, B])))
    np.testing.assert_allclose(np.triu(Rf), S[:b], atol=tol, rtol=0)
    for c in range(b):
        # the stacked reflector is zero on R's rows below c (upper-triangular R): only V_ik is stored
        np.testing.assert_allclose(vs[c][: b - c - 1], 0.0, atol=0)
        np.testing.assert_allclose(Bf[:, c], vs[c][b - c - 1:], atol=tol, rtol=0)
        l, j = divmod(c, s)
        assert abs(T[j, l * s + j] - taus[c]) <= tol
    # T_l identity on the 2b-dimensional stack, Y_l = [E_l; V_l]
    for l in range(b // s):
        Tl = T[:, l * s:(l + 1) * s]
        Y = np.zeros((2 * b, s))
        P = np.eye(2 * b)
        for j in range(s):
            c = l * s + j
            Y[c, j] = 1.0
            Y[b:, j] = Bf[:, c]
            P = P @ (np.eye(2 * b) - taus[c] * np.outer(Y[:, j], Y[:, j]))
        np.testing.assert_allclose(np.eye(2 * b) - Y @ Tl @ Y.T, P, atol=1e-13, rtol=0)


def test_tsqrt_zero_block():
    b, s = 8, 4
    R0 = np.triu(rand(b, b, 5))
    Rf, Bf, T = oracle.tsqrt(R0, np.zeros((b, b)), s)
    np.testing.assert_array_equal(Rf, R0)
    np.testing.assert_array_equal(Bf, 0.0)
    np.testing.assert_array_equal(T, 0.0)


def dense_q_from_geqrt(Af, T, s):
    b = Af.shape[0]
    Q = np.eye(b)
    for tau, u in reflectors_from_geqrt(Af, T, s):
        Q = Q @ (np.eye(b) - tau * np.outer(u, u))
    return Q


@pytest.mark.parametrize("b,s", [(4, 2), (8, 8), (16, 4), (12, 4)])
@pytest.mark.parametrize("trans", [1, 0])
def test_larfb_equals_dense_reflector_product(b, s, trans):
    A = rand(b, b, 11 + b)
    Af, T = oracle.geqrt(A, s)
    Q = dense_q_from_geqrt(Af, T, s)
    C = rand(b, b, 12 + b)
    got = oracle.larfb(Af, T, C, trans)
    want = (Q.T if trans else Q) @ C
    np.testing.assert_allclose(got, want, atol=100 * b * EPS * np.linalg.norm(C), rtol=0)


@pytest.mark.parametrize("b,s", [(4, 2), (8, 8), (16, 4), (12, 6)])
@pytest.mark.parametrize("trans", [1, 0])
def test_ssrfb_equals_dense_reflector_product(b, s, trans):
    R0 = np.triu(rand(b, b, 21 + b))
    Rf, V, T = oracle.tsqrt(R0, rand(b, b, 22 + b), s)
    Q = np.eye(2 * b)
    for c in range(b):
        l, j = divmod(c, s)
        y = np.zeros(2 * b); y[c] = 1.0; y[b:] = V[:, c]
        Q = Q @ (np.eye(2 * b) - T[j, l * s + j] * np.outer(y, y))
    C1, C2 = rand(b, b, 23 + b), rand(b, b, 24 + b)
    g1, g2 = oracle.ssrfb(V, T, C1, C2, trans)
    want = (Q.T if trans else Q) @ np.vstack([C1, C2])
    tol = 100 * b * EPS * np.linalg.norm(np.vstack([C1, C2]))
    np.testing.assert_allclose(np.vstack([g1, g2]), want, atol=tol, rtol=0)


def test_update_kernels_zero_factors_bitwise_identity():
    b, s = 8, 4
    C1, C2 = rand(b, b, 1), rand(b, b, 2)
    Z, ZT = np.zeros((b, b)), np.zeros((s, b))
    g1, g2 = oracle.ssrfb(Z, ZT, C1, C2)
    np.testing.assert_array_equal(g1, C1)
    np.testing.assert_array_equal(g2, C2)
    np.testing.assert_array_equal(oracle.larfb(Z, ZT, C1), C1)


def test_kernel_invalid_args():
    with pytest.raises(ValueError):
        oracle.geqrt(np.eye(4), 3)  # s does not divide b


# ----------------------------------------------------------------------------------------
# whole factorization
# ----------------------------------------------------------------------------------------

@pytest.mark.parametrize("m,n,b,s", [
    (1, 1, 1, 1), (2, 1, 1, 1), (3, 3, 1, 1), (4, 3, 2, 1), (4, 4, 2, 2), (6, 4, 2, 2),
    (9, 9, 3, 1), (9, 6, 3, 3), (7, 5, 3, 1), (12, 8, 4, 2), (12, 12, 4, 4), (5, 9, 2, 1),
    (8, 12, 4, 2), (11, 7, 4, 4),
])
def test_factorization_equals_brute_force(m, n, b, s):
    """Tiled R, V and tau equal the dense eager reflector QR of the same flat tree,
    with the same signs (SURVEY 8(c) 'Brute force')."""
    A = rand(m, n, 1000 + 31 * m + n + b)
    At, T = oracle.geqrf(A, b, s)
    M, Q, refl = brute_force_tiled_qr(A, b)
    tol = 1e-13 * max(1.0, np.linalg.norm(A))
    R = oracle.get_r(At, m, n, b)
    k = min(m, n)
    np.testing.assert_allclose(R, np.triu(M[:k, :n]), atol=tol, rtol=0)
    p, q = oracle.dims(m, n, b)
    for kind, kk, i, c, tau, v in refl:
        l, j = divmod(c, s)
        Tt = tslot(T, i, kk, p, s, b)
        assert abs(Tt[j, l * s + j] - tau) <= tol, (kind, kk, i, c)
        V = tile_of(At, i, kk, p, b)
        if kind == "G":
            np.testing.assert_allclose(V[c + 1:, c], v, atol=tol, rtol=0)
        else:
            np.testing.assert_allclose(V[:, c], v, atol=tol, rtol=0)
    # explicit Q from the brute force: A = Q R on the padded matrix
    P = np.zeros((p * b, q * b)); P[:m, :n] = A
    np.testing.assert_allclose(Q @ M, P, atol=tol, rtol=0)


def test_b1_worked_example():
    """[[3],[4]] with b=1: GEQRT gives tau=0, R=3; TSQRT gives beta=-5, tau=1.6 -> R=[-5]."""
    At, T = oracle.geqrf(np.array([[3.0], [4.0]]), 1, 1)
    assert oracle.get_r(At, 2, 1, 1)[0, 0] == -5.0
    assert T[0] == 0.0 and T[1] == 1.6 and At[1] == 0.5


def sign_normalise(R):
    d = np.sign(np.diag(R))
    d[d == 0] = 1
    return R * d[:, None]


@pytest.mark.parametrize("m,n,b,s", [(256, 256, 64, 16), (200, 150, 16, 8), (150, 200, 32, 8), (96, 96, 96, 32)])
def test_matches_lapack_up_to_signs(m, n, b, s):
    """LAPACK dgeqrf (numpy) R, sign-normalised, matches the oracle's R."""
    A = rand(m, n, 55 + m)
    At, T = oracle.geqrf(A, b, s)
    R = oracle.get_r(At, m, n, b)
    Rl = np.linalg.qr(A, mode="r")
    np.testing.assert_allclose(sign_normalise(R), sign_normalise(Rl), atol=1e-10 * np.linalg.norm(A), rtol=0)


@pytest.mark.parametrize("m,n,b,s,dist", [
    (256, 256, 64, 16, "uniform"),     # C1
    (67, 41, 16, 8, "uniform"),        # padding case SPEC.md:541
    (41, 67, 16, 16, "uniform"),       # m < n
    (512, 64, 32, 8, "normal"),        # tall-skinny, C4-shaped
])
def test_invariants_backward_error_orthogonality(m, n, b, s, dist):
    """R^T R = A^T A, column norms, ||A - QR|| / (||A|| n eps) < 10, ||I - Q^TQ|| / (n eps) < 10,
    Q^T A = R (BASELINE.json north_star)."""
    A = tqr_inputs.make(m, n, dist, 77 + m)
    At, T = oracle.geqrf(A, b, s)
    R = oracle.get_r(At, m, n, b)
    k = min(m, n)
    nA = np.linalg.norm(A)
    assert np.linalg.norm(R.T @ R - A.T @ A) / (nA ** 2 * max(m, n) * EPS) < 10
    np.testing.assert_allclose(np.linalg.norm(R, axis=0), np.linalg.norm(A, axis=0), rtol=1e-12)
    Q = oracle.orgqr(At, T, m, n, b, s, k=k)
    assert np.linalg.norm(A - Q @ R) / (nA * n * EPS) < 10
    assert np.linalg.norm(np.eye(k) - Q.T @ Q) / (n * EPS) < 10
    QtA = oracle.ormqr(At, T, m, n, b, s, A, trans=1)
    np.testing.assert_allclose(QtA[:k], R, atol=10 * n * EPS * nA, rtol=0)
    np.testing.assert_allclose(QtA[k:], 0.0, atol=10 * n * EPS * nA)
    # Q (Q^T B) = B round trip
    B = rand(m, 5, 3)
    np.testing.assert_allclose(oracle.ormqr(At, T, m, n, b, s, oracle.ormqr(At, T, m, n, b, s, B, 1), 0), B,
                               atol=10 * m * EPS * np.linalg.norm(B), rtol=0)


def test_identity_input():
    """Identity -> R = I, all T = 0."""
    for m, n, b, s in ((64, 64, 16, 8), (40, 24, 16, 4)):
        A = np.eye(m, n)
        At, T = oracle.geqrf(A, b, s)
        np.testing.assert_array_equal(oracle.get_r(At, m, n, b), np.eye(min(m, n), n))
        np.testing.assert_array_equal(T, 0.0)


@pytest.mark.parametrize("m,n,b", [(256, 256, 64), (96, 160, 32)])
def test_inner_blocking_independence(m, n, b):
    """R, V, taus do not depend on s in exact arithmetic; T_l are the diagonal blocks of T(s=b)."""
    A = rand(m, n, 9)
    At_b, T_b = oracle.geqrf(A, b, b)
    p, q = oracle.dims(m, n, b)
    for s in (b // 8, b // 4, b // 2):
        At_s, T_s = oracle.geqrf(A, b, s)
        np.testing.assert_allclose(At_s, At_b, atol=1e-12 * np.linalg.norm(A), rtol=0)
        for k in range(min(p, q)):
            for i in range(k, p):
                Tb, Ts = tslot(T_b, i, k, p, b, b), tslot(T_s, i, k, p, s, b)
                for l in range(b // s):
                    np.testing.assert_allclose(Ts[:, l * s:(l + 1) * s],
                                               Tb[l * s:(l + 1) * s, l * s:(l + 1) * s], atol=1e-12, rtol=0)


@pytest.mark.parametrize("nthreads", [2, 4, 7])
def test_threaded_dag_bitwise_equals_sequential(nthreads):
    """Any DAG-respecting order gives bitwise-identical results."""
    m, n, b, s = 320, 256, 32, 8
    A = rand(m, n, 4)
    At1, T1 = oracle.geqrf(A, b, s, nthreads=1)
    c1 = oracle.task_counts()
    Atn, Tn = oracle.geqrf(A, b, s, nthreads=nthreads)
    cn = oracle.task_counts()
    assert np.array_equal(At1, Atn) and np.array_equal(T1, Tn)
    assert c1 == cn
    p, q = oracle.dims(m, n, b)
    K = min(p, q)
    assert c1["G"] == K
    assert c1["L"] == sum(q - k - 1 for k in range(K))
    assert c1["T"] == sum(p - k - 1 for k in range(K))
    assert c1["S"] == sum((p - k - 1) * (q - k - 1) for k in range(K))


# ---- the oracle's DAG edges -------------------------
def _spec_edges(p, q):
    """SPEC.md:334-337 restated 0-based (k = 0 .. min(p,q)-1): predecessor -> successor."""
    E = set()
    for k in range(min(p, q)):
        G = ("G", k, k, k)
        if k > 0:
            E.add((("S", k - 1, k, k), G))
        for j in range(k + 1, q):
            E.add((G, ("L", k, k, j)))
            if k > 0:
                E.add((("S", k - 1, k, j), ("L", k, k, j)))
        for i in range(k + 1, p):
            E.add((G if i == k + 1 else ("T", k, i - 1, k), ("T", k, i, k)))
            if k > 0:
                E.add((("S", k - 1, i, k), ("T", k, i, k)))
            for j in range(k + 1, q):
                E.add((("T", k, i, k), ("S", k, i, j)))
                E.add((("L", k, k, j) if i == k + 1 else ("S", k, i - 1, j), ("S", k, i, j)))
                if k > 0:
                    E.add((("S", k - 1, i, j), ("S", k, i, j)))
    return E


def _sequential_tasks(p, q):
    """Algorithm 1's loop order."""
    out = []
    for k in range(min(p, q)):
        out.append(("G", k, k, k))
        out += [("L", k, k, j) for j in range(k + 1, q)]
        for i in range(k + 1, p):
            out.append(("T", k, i, k))
            out += [("S", k, i, j) for j in range(k + 1, q)]
    return out


def _access(t):
    """(reads, writes) of a task over data regions, from the kernels' definitions (SURVEY
    8(c) c-3..c-6): A(k,k) is split into its upper triangle 'R' (R_kk) and strict lower part
    'V' (V_kk) -- TSQRT touches only R_kk, LARFB reads only V_kk."""
    kind, k, i, j = t
    if kind == "G":
        r, w = set(), {("R", k, k), ("V", k, k), ("T", k, k)}
    elif kind == "L":
        r, w = {("V", k, k), ("T", k, k)}, {("A", k, j)}
    elif kind == "T":
        r, w = set(), {("R", k, k), ("A", i, k), ("T", i, k)}
    else:
        r, w = {("A", i, k), ("T", i, k)}, {("A", k, j), ("A", i, j)}

    def split(regs):  # a diagonal tile as a whole (update target) = its R and V parts
        out = set()
        for x in regs:
            out |= {("R", x[1], x[1]), ("V", x[1], x[1])} if x[0] == "A" and x[1] == x[2] else {x}
        return out
    return split(r), split(w)


def _verify_serialization(p, q, edges):
    """Every pair of tasks that conflict (one writes a region the other reads or writes) must
    be ordered by a DAG path in Algorithm 1's sequential order, and every edge must join two
    conflicting tasks in that order.  Returns a list of violations."""
    tasks = _sequential_tasks(p, q)
    pos = {t: n for n, t in enumerate(tasks)}
    succ = {t: set() for t in tasks}
    for a, b in edges:
        succ[a].add(b)
    reach = {}
    for t in reversed(tasks):   # reachability; a cycle shows up as an order violation below
        r = set()
        for u in succ[t]:
            r.add(u)
            r |= reach.get(u, set())
        reach[t] = r
    acc = {t: _access(t) for t in tasks}
    bad = []
    for a, b in edges:
        (ra, wa), (rb, wb) = acc[a], acc[b]
        if pos[a] >= pos[b] or not (wa & (rb | wb) or wb & ra):
            bad.append(("edge", a, b))
    for x in range(len(tasks)):
        a = tasks[x]
        ra, wa = acc[a]
        for y in range(x + 1, len(tasks)):
            b = tasks[y]
            rb, wb = acc[b]
            if (wa & (rb | wb) or wb & ra) and b not in reach[a]:
                bad.append(("unordered", a, b))
    return bad


@pytest.mark.parametrize("p,q", [(1, 1), (2, 2), (3, 3), (4, 2), (2, 4), (5, 3), (3, 6)])
def test_dag_edges_equal_spec_and_serialize(p, q):
    """The oracle's edge set equals SPEC.md:334-337 exactly, every edge is a read/write
    conflict of the kernels in Algorithm 1's order, and every conflicting pair is ordered."""
    got = oracle.dag_edges(p, q)
    assert len(got) == len(set(got))
    assert set(got) == _spec_edges(p, q)
    assert _verify_serialization(p, q, got) == []
    if p == q == 2:   # SPEC.md:341 worked example: G(2)'s sole predecessor is S(1,2,2)
        assert [a for a, b in got if b == ("G", 1, 1, 1)] == [("S", 0, 1, 1)]
    if p == q == 1:
        assert got == []


def test_dag_edge_drop_or_flip_is_detected():
    """Negative check of the pin: removing or reversing ANY single edge of the 3 x 3 DAG
    (Fig. 3's instance) leaves a conflicting pair unordered or breaks the order."""
    edges = oracle.dag_edges(3, 3)
    for e in range(len(edges)):
        dropped = edges[:e] + edges[e + 1:]
        assert _verify_serialization(3, 3, dropped), f"dropping {edges[e]} went unnoticed"
        a, b = edges[e]
        flipped = edges[:e] + [(b, a)] + edges[e + 1:]
        assert _verify_serialization(3, 3, flipped), f"flipping {edges[e]} went unnoticed"


def test_dag_node_counts_golden():
    cases = json.load(open(os.path.join(GOLDEN, "dag_counts.json")))["cases"]
    for c in cases:
        p, q = c["p"], c["q"]
        oracle.geqrf(rand(p * 2, q * 2, 1), 2, 1, nthreads=2)
        got = sum(oracle.task_counts().values())
        assert got == c["nodes"], c["cite"]


def test_pack_unpack_roundtrip():
    A = rand(37, 53, 8)
    At = oracle.pack(A, 16)
    p, q = oracle.dims(37, 53, 16)
    assert At.size == p * q * 256
    np.testing.assert_array_equal(oracle.unpack(At, 37, 53, 16), A)
    # tile (i,j) column-major at (i + j p) b^2
    t = tile_of(At, 1, 2, p, 16)
    np.testing.assert_array_equal(t[:5, :3], A[16:21, 32:35])
    np.testing.assert_array_equal(tile_of(At, 2, 3, p, 16)[5:, :], 0.0)  # zero padding


# ----------------------------------------------------------------------------------------
# flop models
# ----------------------------------------------------------------------------------------

def test_flop_model_golden():
    g = json.load(open(os.path.join(GOLDEN, "flop_model.json")))
    for c in g["kernel"]:
        assert oracle.kernel_flops(c["kind"], c["b"]) == pytest.approx(c["flops"], rel=1e-15), c["cite"]
    for c in g["standard"]:
        assert oracle.flops_standard(c["m"], c["n"]) == pytest.approx(c["flops"], rel=1e-15), c["cite"]
    for c in g["eq4"]:
        assert oracle.flops_eq4(c["p"], c["q"], c["b"]) == pytest.approx(c["flops"], rel=1e-14), c["cite"]
    r = g["eq4_ratio"]
    ratio = oracle.flops_eq4(r["p"], r["q"], r["b"]) / oracle.flops_standard(r["p"] * r["b"], r["q"] * r["b"])
    assert r["lo"] <= ratio <= r["hi"], r["cite"]


def test_flop_eq4_asymptote():
    """Eq. 4 tends to 5/2 n^2 (m - n/3), i.e. 25% over 2 n^2 (m - n/3)."""
    p = q = 400
    assert oracle.flops_eq4(p, q, 1) / oracle.flops_standard(p, q) == pytest.approx(1.25, abs=0.01)


def test_inputs_generator():
    """Generator sanity: exact U[-0.5,0.5), deterministic, column-major index stream."""
    A = tqr_inputs.uniform(64, 32, 5)
    assert A.flags.f_contiguous and A.min() >= -0.5 and A.max() < 0.5
    np.testing.assert_array_equal(A, tqr_inputs.uniform(64, 32, 5))
    B = tqr_inputs.uniform(64 * 32, 1, 5)
    np.testing.assert_array_equal(A.reshape(-1, order="F"), B[:, 0])
    N = tqr_inputs.normal(4000, 50, 6)
    assert abs(N.mean()) < 0.01 and abs(N.std() - 1) < 0.01
