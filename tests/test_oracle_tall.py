"""Pins for the oracle's non-square-tile mode (reading R30; PAPER.md:582-583,
"using 2b x b blocks would reduce the overhead at 12.5%").  The tile rows below the diagonal
are grouped in units of h (units start right below the diagonal tile; the last may be
shorter); TSQRT / SSRFB work on the (nt b) x b stack of a unit.

Each pin is independent of the oracle's own arithmetic: textbook Householder QR of the
dense stack, the dense block-reflector product, a brute-force eager dense-reflector QR of the
whole flat tree with units, the paper's 12.5% overhead figure, invariants, the DAG's
read/write serialization.
"""
import numpy as np
import pytest

import oracle
import tqr_inputs

EPS = np.finfo(np.float64).eps


def rand(m, n, seed):
    return tqr_inputs.uniform(m, n, seed)


def dense_house(alpha, x):
    sigma = float(np.dot(x, x))
    if sigma == 0.0:
        return alpha, 0.0, np.zeros_like(x)
    nu = np.sqrt(alpha * alpha + sigma)
    beta = -nu if alpha >= 0 else nu
    return beta, (beta - alpha) / beta, x / (alpha - beta)


def tile_of(At, i, j, p, b):
    off = (i + j * p) * b * b
    return At[off:off + b * b].reshape((b, b), order="F")


def tslot(T, i, k, p, s, b):
    off = (i + k * p) * s * b
    return T[off:off + s * b].reshape((s, b), order="F")


def units(k, p, h):
    """DESIGN.md R30: tile rows k+1 .. p-1 in consecutive groups of h."""
    out, i = [], k + 1
    while i < p:
        out.append(list(range(i, min(p, i + h))))
        i += h
    return out


@pytest.mark.parametrize("b,s,nt", [(3, 1, 2), (4, 2, 2), (4, 4, 3), (8, 4, 2), (6, 3, 2)])
def test_tsqrt_rows_equals_stacked_qr(b, s, nt):
    """TSQRT on a (nt b) x b lower block == textbook Householder QR of [R; B] (same signs)."""
    Rin = np.triu(rand(b, b, 50 + b))
    junk = np.tril(rand(b, b, 60 + b), -1)
    B = rand(nt * b, b, 70 + b + nt)
    Rf, Bf, T = oracle.tsqrt_rows(Rin + junk, B, s)
    np.testing.assert_array_equal(np.tril(Rf, -1), junk)  # V_kk: never read or written
    S = np.vstack([Rin, B])
    taus = []
    for c in range(b):
        beta, tau, v = dense_house(S[c, c], S[c + 1:, c].copy())
        u = np.concatenate([np.zeros(c), [1.0], v])
        S = S - tau * np.outer(u, u @ S)
        S[c, c] = beta
        S[c + 1:, c] = 0.0
        taus.append(tau)
        np.testing.assert_allclose(v[: b - c - 1], 0.0, atol=0)  # zero on R's rows below c
        np.testing.assert_allclose(Bf[:, c], v[b - c - 1:], atol=100 * b * EPS * 10, rtol=0)
    tol = 100 * b * EPS * max(1.0, np.linalg.norm(np.vstack([Rin, B])))
    np.testing.assert_allclose(np.triu(Rf), S[:b], atol=tol, rtol=0)
    for c in range(b):
        l, j = divmod(c, s)
        assert abs(T[j, l * s + j] - taus[c]) <= tol


@pytest.mark.parametrize("b,s,nt", [(4, 2, 2), (8, 8, 2), (6, 2, 3)])
@pytest.mark.parametrize("trans", [1, 0])
def test_ssrfb_rows_equals_dense_reflector_product(b, s, nt, trans):
    R0 = np.triu(rand(b, b, 80 + b))
    _, V, T = oracle.tsqrt_rows(R0, rand(nt * b, b, 81 + b), s)
    n = (1 + nt) * b
    Q = np.eye(n)
    for c in range(b):
        l, j = divmod(c, s)
        y = np.zeros(n); y[c] = 1.0; y[b:] = V[:, c]
        Q = Q @ (np.eye(n) - T[j, l * s + j] * np.outer(y, y))
    C1, C2 = rand(b, b, 82 + b), rand(nt * b, b, 83 + b)
    g1, g2 = oracle.ssrfb_rows(V, T, C1, C2, trans)
    want = (Q.T if trans else Q) @ np.vstack([C1, C2])
    tol = 100 * n * EPS * np.linalg.norm(np.vstack([C1, C2]))
    np.testing.assert_allclose(np.vstack([g1, g2]), want, atol=tol, rtol=0)


def brute_force_units(A, b, h):
    """Flat-tree tiled QR with units of h tile rows, written densely: every reflector an
    explicit m x m matrix applied eagerly in creation order.  GEQRT(k) column c: 1 at row
    kb+c, v below within tile row k; TSQRT(k, unit) column c: 1 at row kb+c, v on the unit's
    rows.  Returns (R_dense, Q, reflectors)."""
    A = np.array(A, dtype=np.float64)
    m, n = A.shape
    p, q = -(-m // b), -(-n // b)
    M = np.zeros((p * b, q * b)); M[:m, :n] = A
    Q = np.eye(p * b)
    refl = []
    for k in range(min(p, q)):
        for c in range(b):
            col = k * b + c
            rows = list(range(col, (k + 1) * b))
            beta, tau, v = dense_house(M[col, col], M[col + 1:(k + 1) * b, col].copy())
            u = np.zeros(p * b); u[rows] = np.concatenate([[1.0], v])
            H = np.eye(p * b) - tau * np.outer(u, u)
            M = H @ M; M[col, col] = beta; M[col + 1:(k + 1) * b, col] = 0.0
            Q = Q @ H
            refl.append(("G", k, k, c, tau, v))
        for un in units(k, p, h):
            r0, r1 = un[0] * b, (un[-1] + 1) * b
            for c in range(b):
                col = k * b + c
                beta, tau, v = dense_house(M[col, col], M[r0:r1, col].copy())
                u = np.zeros(p * b); u[col] = 1.0; u[r0:r1] = v
                H = np.eye(p * b) - tau * np.outer(u, u)
                M = H @ M; M[col, col] = beta; M[r0:r1, col] = 0.0
                Q = Q @ H
                refl.append(("T", k, un[0], c, tau, v))
    return M, Q, refl


@pytest.mark.parametrize("m,n,b,s,h", [(9, 6, 3, 1, 2), (12, 8, 2, 2, 2), (16, 8, 4, 2, 2), (14, 6, 2, 1, 3),
                                       (10, 10, 2, 2, 2), (13, 5, 4, 4, 2), (8, 12, 2, 1, 2), (20, 4, 2, 2, 4)])
def test_tall_units_equal_brute_force(m, n, b, s, h):
    """R (with its signs), V and tau equal the dense eager reflector QR with the same units."""
    A = rand(m, n, 500 + 7 * m + n + h)
    At, T = oracle.geqrf(A, b, s, h=h)
    M, Q, refl = brute_force_units(A, b, h)
    tol = 1e-13 * max(1.0, np.linalg.norm(A))
    R = oracle.get_r(At, m, n, b)
    np.testing.assert_allclose(R, np.triu(M[:min(m, n), :n]), atol=tol, rtol=0)
    p, q = -(-m // b), -(-n // b)
    for kind, k, i0, c, tau, v in refl:
        l, j = divmod(c, s)
        assert abs(tslot(T, i0, k, p, s, b)[j, l * s + j] - tau) <= tol
        if kind == "G":
            np.testing.assert_allclose(tile_of(At, k, k, p, b)[c + 1:, c], v, atol=tol, rtol=0)
        else:
            nt = len(v) // b
            got = np.concatenate([tile_of(At, i0 + t, k, p, b)[:, c] for t in range(nt)])
            np.testing.assert_allclose(got, v, atol=tol, rtol=0)
    P = np.zeros((p * b, q * b)); P[:m, :n] = A
    np.testing.assert_allclose(Q @ M, P, atol=tol, rtol=0)
    # the T slots of a unit's other tile rows stay zero
    for k in range(min(p, q)):
        for un in units(k, p, h):
            for i in un[1:]:
                assert np.all(tslot(T, i, k, p, s, b) == 0.0)


def test_units_change_r_but_not_the_factorization():
    """h = 2 gives a DIFFERENT R than h = 1 (signs / rounding: other reflectors) while both are
    QR factorizations of A: same |R| row norms up to sign, R^T R = A^T A."""
    m, n, b, s = 96, 48, 8, 4
    A = rand(m, n, 9)
    R1 = oracle.get_r(oracle.geqrf(A, b, s)[0], m, n, b)
    R2 = oracle.get_r(oracle.geqrf(A, b, s, h=2)[0], m, n, b)
    assert not np.allclose(R1, R2)
    D = np.sign(np.diag(R1)) * np.sign(np.diag(R2))
    np.testing.assert_allclose(D[:, None] * R1, R2, atol=1e-12 * np.linalg.norm(A), rtol=0)
    np.testing.assert_allclose(R2.T @ R2, A.T @ A, atol=50 * m * EPS * np.linalg.norm(A) ** 2, rtol=0)


@pytest.mark.parametrize("h", [2, 3])
def test_tall_threaded_equals_sequential_and_s_independence(h):
    m, n, b = 200, 120, 16
    A = rand(m, n, 33 + h)
    At1, T1 = oracle.geqrf(A, b, 4, h=h)
    At4, T4 = oracle.geqrf(A, b, 4, nthreads=5, h=h)
    assert np.array_equal(At1, At4) and np.array_equal(T1, T4)
    Atb, _ = oracle.geqrf(A, b, b, h=h)  # s = b (the paper's unblocked kernels)
    np.testing.assert_allclose(oracle.get_r(At1, m, n, b), oracle.get_r(Atb, m, n, b),
                               atol=1e-12 * np.linalg.norm(A), rtol=0)


@pytest.mark.parametrize("m,n,b,s,h", [(300, 200, 32, 8, 2), (517, 130, 64, 16, 2), (260, 260, 32, 32, 3)])
def test_tall_invariants_backward_error_orthogonality(m, n, b, s, h):
    A = rand(m, n, 44 + m)
    At, T = oracle.geqrf(A, b, s, nthreads=4, h=h)
    R = oracle.get_r(At, m, n, b)
    k = min(m, n)
    Q = oracle.orgqr(At, T, m, n, b, s, k=k, nthreads=4, h=h)
    nA = np.linalg.norm(A)
    assert np.linalg.norm(A - Q @ R) / (nA * n * EPS) < 10
    assert np.linalg.norm(np.eye(k) - Q.T @ Q) / (n * EPS) < 10
    QtA = oracle.ormqr(At, T, m, n, b, s, A, 1, nthreads=4, h=h)
    np.testing.assert_allclose(QtA[:k], R, atol=50 * n * EPS * nA, rtol=0)
    np.testing.assert_allclose(QtA[k:], 0.0, atol=50 * n * EPS * nA)


def test_paper_overhead_figure():
    """square tiles need 25% more flops than LAPACK (Eq. 4), 2b x b
    tiles 12.5% -- the s = b flop count of the unit algorithm tends to 1 + 1/(4h)."""
    std = lambda nn: 4.0 / 3.0 * nn ** 3
    r1 = oracle.flops_eq4_h(400, 400, 1, 1) / std(400)
    r2 = oracle.flops_eq4_h(400, 400, 1, 2) / std(400)
    assert abs(r1 - 1.25) < 0.005 and abs(r2 - 1.125) < 0.005
    assert oracle.flops_eq4_h(20, 20, 1, 1) == pytest.approx(13593.0 + 1.0 / 3.0, rel=1e-12)


def _seq_tasks(p, q, h):
    out = []
    for k in range(min(p, q)):
        out.append(("G", k, k, k))
        out += [("L", k, k, j) for j in range(k + 1, q)]
        for un in units(k, p, h):
            out.append(("T", k, un[0], k))
            out += [("S", k, un[0], j) for j in range(k + 1, q)]
    return out


def _access(t, p, h):
    kind, k, i0, j = t
    un = next((u for u in units(k, p, h) if u[0] == i0), [i0])

    def split(regs):
        out = set()
        for x in regs:
            out |= {("R", x[1], x[1]), ("V", x[1], x[1])} if x[0] == "A" and x[1] == x[2] else {x}
        return out
    if kind == "G":
        return set(), {("R", k, k), ("V", k, k), ("T", k, k)}
    if kind == "L":
        return {("V", k, k), ("T", k, k)}, split({("A", k, j)})
    if kind == "T":
        return set(), {("R", k, k), ("T", i0, k)} | {("A", i, k) for i in un}
    return {("A", i, k) for i in un} | {("T", i0, k)}, split({("A", k, j)} | {("A", i, j) for i in un})


@pytest.mark.parametrize("p,q,h", [(5, 3, 2), (6, 4, 2), (7, 7, 3), (9, 3, 2), (4, 6, 2)])
def test_tall_dag_serializes_every_conflict(p, q, h):
    """Every edge of the unit DAG joins two conflicting tasks in Algorithm 1's order, and every
    conflicting pair is ordered by a path (read/write sets from the kernels' definitions)."""
    edges = oracle.dag_edges(p, q, h)
    tasks = _seq_tasks(p, q, h)
    pos = {t: n for n, t in enumerate(tasks)}
    succ = {t: set() for t in tasks}
    for a, b_ in edges:
        succ[a].add(b_)
    reach = {}
    for t in reversed(tasks):
        r = set()
        for u in succ[t]:
            r |= {u} | reach.get(u, set())
        reach[t] = r
    acc = {t: _access(t, p, h) for t in tasks}
    for a, b_ in edges:
        (ra, wa), (rb, wb) = acc[a], acc[b_]
        assert pos[a] < pos[b_] and (wa & (rb | wb) or wb & ra), (a, b_)
    for x, a in enumerate(tasks):
        ra, wa = acc[a]
        for b_ in tasks[x + 1:]:
            rb, wb = acc[b_]
            if wa & (rb | wb) or wb & ra:
                assert b_ in reach[a], ("unordered", a, b_)
    assert oracle.dag_edges(p, q, 1) == oracle.dag_edges(p, q)
