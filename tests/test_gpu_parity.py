"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded
inputs.  Tolerances (BASELINE.json north_star): R elementwise within 1e-10 * ||A||_F of the
oracle's R; backward error and orthogonality of the GPU's own factors below 10 * n * eps.
"""
import numpy as np
import pytest

import oracle
import tqr_inputs
from gpu_util import run_factor

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


def _cases():
    # (m, n, b, s, dist): several tiles and a ragged tail for each built (b, s)
    return [
        (256, 256, 64, 16, "uniform"),   # C1
        (67, 41, 16, 8, "uniform"),      # padding case
        (41, 67, 16, 16, "uniform"),     # m < n, s == b
        (100, 90, 32, 8, "uniform"),
        (96, 96, 32, 32, "uniform"),     # s == b (the paper's unblocked kernels)
        (300, 200, 64, 64, "uniform"),
        (520, 300, 128, 32, "uniform"),
        (700, 600, 256, 32, "uniform"),  # C3 tiling, ragged
        (1280, 300, 256, 32, "normal"),  # C4-shaped tall-skinny
        (1100, 1030, 512, 64, "uniform"),  # C5 tiling (internal 16-column blocks + form_t), ragged
        # degenerate shapes: 1x1, one row, one column, one exact tile, a tile + 1-element tail
        (1, 1, 16, 8, "uniform"), (1, 50, 16, 8, "uniform"), (50, 1, 16, 8, "uniform"),
        (64, 64, 64, 16, "normal"), (65, 65, 64, 16, "uniform"), (257, 3, 256, 32, "normal"),
    ]


@pytest.mark.parametrize("m,n,b,s,dist", _cases())
def test_factor_parity(m, n, b, s, dist):
    A = tqr_inputs.make(m, n, dist, 4242 + m + n + b)
    g = run_factor(A, b, s)
    At_o, T_o = oracle.geqrf(A, b, s, nthreads=4)
    R_o = oracle.get_r(At_o, m, n, b)
    nA = np.linalg.norm(A)
    err = np.max(np.abs(np.triu(g["R"]) - np.triu(R_o)))
    assert err <= 1e-10 * nA, f"R mismatch {err:.3e} > {1e-10 * nA:.3e}"
    assert np.all(np.tril(g["R"], -1) == 0), "get_r writes exact zeros below the diagonal"
    # V and T (diagnostic, same tolerance scale)
    assert np.max(np.abs(g["At"] - At_o)) <= 1e-9 * max(1.0, nA)
    assert np.max(np.abs(g["T"] - T_o)) <= 1e-9 * max(1.0, nA)
    # backward error / orthogonality of the GPU factors, Q formed by the oracle's apply-Q
    k = min(m, n)
    Q = oracle.orgqr(g["At"], g["T"], m, n, b, s, k=k, nthreads=4)
    assert np.linalg.norm(A - Q @ g["R"]) / (nA * n * EPS) < 10
    assert np.linalg.norm(np.eye(k) - Q.T @ Q) / (n * EPS) < 10


def test_factor_deterministic():
    A = tqr_inputs.uniform(700, 600, 5)
    g1 = run_factor(A, 256, 32)
    g2 = run_factor(A, 256, 32)
    assert np.array_equal(g1["At"], g2["At"]) and np.array_equal(g1["T"], g2["T"])


@pytest.mark.parametrize("m,n,b,s", [(8192, 8192, 256, 32), (4096, 4096, 128, 32), (8192, 4096, 256, 32)])
def test_locality_schedule_bitwise_equal(m, n, b, s):
    """TQR_FLAG_LOCALITY changes only the dispatch order (R22): same bits as the
    default order, and the plan really runs a different order (on grids large enough that the
    ready queue outgrows the 148 CTAs; below that, every order is the ready order)."""
    A = tqr_inputs.uniform(m, n, 77 + m)
    g0 = run_factor(A, b, s)
    g1 = run_factor(A, b, s, locality=True)
    assert np.array_equal(g0["At"], g1["At"]) and np.array_equal(g0["T"], g1["T"])
    r0, r1 = g0["plan"].records(), g1["plan"].records()
    assert r0.shape == r1.shape and not np.array_equal(r0, r1)


@pytest.mark.parametrize("m,n,b,s,nrhs", [(256, 256, 64, 16, 100), (700, 600, 256, 32, 300), (67, 41, 16, 8, 20),
                                           (520, 300, 128, 32, 128), (1100, 700, 512, 64, 200)])
@pytest.mark.parametrize("trans", ["T", "N"])
def test_ormqr_parity(m, n, b, s, nrhs, trans):
    import torch
    from paper_0707_3548_b200 import Plan
    A = tqr_inputs.uniform(m, n, 17 + m)
    g = run_factor(A, b, s)
    plan = g["plan"]
    Bm = tqr_inputs.uniform(m, nrhs, 99)
    Bt = torch.from_numpy(oracle.pack(Bm, b)).cuda()
    plan.ormqr(trans, g["At_dev"], g["T_dev"], Bt, nrhs)
    plan.sync()
    got = oracle.unpack(Bt.cpu().numpy(), m, nrhs, b)
    want = oracle.ormqr(g["At"], g["T"], m, n, b, s, Bm, 1 if trans == "T" else 0, nthreads=4)
    # an orthogonal transformation of each column: the GPU and the oracle differ only in
    # rounding order, so every column agrees to a few ulps of its norm (10 m eps, relative)
    col_err = np.linalg.norm(got - want, axis=0) / np.linalg.norm(Bm, axis=0)
    assert np.max(col_err) <= 10 * m * EPS, np.max(col_err)


@pytest.mark.parametrize("m,n,b,s", [(256, 256, 64, 16), (700, 600, 256, 32), (520, 300, 128, 32),
                                     (1100, 700, 512, 64)])
def test_orgqr_and_backward_error_on_gpu(m, n, b, s):
    import torch
    A = tqr_inputs.uniform(m, n, 23 + m)
    g = run_factor(A, b, s)
    plan = g["plan"]
    k = n
    qb = -(-k // b)
    Qt = torch.empty(plan.p * qb * b * b, dtype=torch.float64, device="cuda")
    plan.orgqr(g["At_dev"], g["T_dev"], k, Qt)
    plan.sync()
    Q = oracle.unpack(Qt.cpu().numpy(), m, k, b)
    Q_o = oracle.orgqr(g["At"], g["T"], m, n, b, s, k=k, nthreads=4)
    assert np.max(np.abs(Q - Q_o)) <= 10 * m * EPS  # unit-norm columns: 10 m eps absolute
    nA = np.linalg.norm(A)
    assert np.linalg.norm(A - Q @ g["R"]) / (nA * n * EPS) < 10
    assert np.linalg.norm(np.eye(k) - Q.T @ Q) / (n * EPS) < 10


def test_identity_and_zero_columns():
    for m, n, b, s in ((128, 128, 32, 8), (256, 192, 64, 16)):
        g = run_factor(np.eye(m, n), b, s)
        np.testing.assert_array_equal(g["R"], np.eye(min(m, n), n))
        assert np.all(g["T"] == 0.0)
    A = tqr_inputs.uniform(200, 150, 3)
    A[:, 10:20] = 0.0   # rank-deficient: tau = 0 reflectors, not an error
    g = run_factor(A, 64, 16)
    At_o, T_o = oracle.geqrf(A, 64, 16)
    assert np.max(np.abs(g["R"] - oracle.get_r(At_o, 200, 150, 64))) <= 1e-10 * np.linalg.norm(A)


@pytest.mark.parametrize("m,n,b,s,reps", [(4096, 4096, 128, 32, 4), (8192, 1024, 256, 32, 4), (3000, 2100, 512, 64, 3),
                                          (1024, 1024, 64, 16, 6)])
def test_repeat_bitwise_stress(m, n, b, s, reps):
    """Races show up as run-to-run differences: the out-of-order executor must give bitwise
    identical R/V/T on every run (each tile's operation sequence is fixed by the DAG)."""
    A = tqr_inputs.uniform(m, n, 99 + m)
    g0 = run_factor(A, b, s)
    for _ in range(reps - 1):
        g = run_factor(A, b, s)
        assert np.array_equal(g["At"], g0["At"]) and np.array_equal(g["T"], g0["T"])


def test_misaligned_pointers_are_invalid_args():
    """include/tqr.h: data pointers must be 16-byte aligned; a misaligned one is reported as
    TQR_ERR_INVALID_ARG with its argument index (not a TMA fault), and the caller's current
    device is left as it was."""
    import torch
    from paper_0707_3548_b200 import Plan
    from paper_0707_3548_b200.tqr import TqrError
    plan = Plan(64, 64, 16, 8)
    At, T = plan.alloc()
    A = torch.zeros(64 * 64 + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(TqrError) as e:
        plan.pack(A[1:], At)              # 8-byte offset
    assert e.value.status == 1 and e.value.bad_arg == 2
    big = torch.zeros(At.numel() + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(TqrError) as e:
        plan.geqrf(big[1:], T)
    assert e.value.status == 1 and e.value.bad_arg == 2
    assert torch.cuda.current_device() == 0
    plan.pack(A[:-1], At)                 # aligned: fine
    plan.sync()


def test_layout_roundtrip_odd_leading_dimension():
    """pack/unpack/get_r with an odd leading dimension (unaligned column starts take the
    scalar path of the run kernels) and ragged tiles: bitwise round trip, exact R layout."""
    import torch
    from paper_0707_3548_b200 import Plan
    for m, n, b, s in ((67, 41, 16, 8), (301, 257, 64, 16), (999, 130, 128, 32), (513, 700, 256, 32)):
        A = tqr_inputs.uniform(m, n, 8 + m)
        Ac = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
        plan = Plan(m, n, b, s)
        At, T = plan.alloc()
        plan.pack(Ac, At)
        back = torch.full_like(Ac, 7.0)
        plan.unpack(At, back)
        R = torch.full((n, min(m, n)), 7.0, dtype=torch.float64, device="cuda")
        plan.get_r(At, R)
        plan.sync()
        assert torch.equal(back, Ac)
        assert np.array_equal(At.cpu().numpy(), oracle.pack(A, b))
        np.testing.assert_array_equal(R.cpu().numpy().T, np.triu(A[:min(m, n), :]))
