"""GPU parity of the non-square 2b x b tiles (TQR_FLAG_TALL_TILES; R30)
against the oracle's unit mode (oracle.geqrf(..., h=2)) on the same seeded inputs: R elementwise
within 1e-10 ||A||_F, V and T within 1e-9 ||A||_F; units of one and two tiles (ragged tails,
m < n), C4 in full; plus the backward error of the GPU factors through the oracle's apply-Q."""
import os

import numpy as np
import pytest

import oracle
import tqr_inputs

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps
THREADS = max(1, len(os.sched_getaffinity(0)))


def _factor_tall(A, b=256, s=32):
    import torch
    from paper_0707_3548_b200 import Plan
    m, n = A.shape
    plan = Plan(m, n, b, s, tall=True)
    assert plan.info()["h"] == 2
    Ac = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(A).T)).cuda()
    At, T = plan.alloc()
    plan.pack(Ac, At)
    plan.geqrf(At, T)
    R = torch.empty((n, min(m, n)), dtype=torch.float64, device="cuda")
    plan.get_r(At, R)
    plan.sync()
    return plan, At.cpu().numpy(), T.cpu().numpy(), R.cpu().numpy().T.copy()


@pytest.mark.parametrize("m,n,dist", [(1280, 300, "normal"), (2048, 512, "normal"), (3000, 700, "uniform"),
                                      (700, 600, "uniform"), (768, 768, "uniform"), (300, 700, "uniform"),
                                      (2560, 256, "normal"), (513, 257, "uniform")])
def test_tall_tiles_parity(m, n, dist):
    A = tqr_inputs.make(m, n, dist, 777 + m + n)
    _, At, T, R = _factor_tall(A)
    At_o, T_o = oracle.geqrf(A, 256, 32, nthreads=THREADS, h=2)
    R_o = oracle.get_r(At_o, m, n, 256)
    nA = np.linalg.norm(A)
    assert np.max(np.abs(R - R_o)) <= 1e-10 * nA
    assert np.max(np.abs(At - At_o)) <= 1e-9 * nA
    assert np.max(np.abs(T - T_o)) <= 1e-9 * nA
    k = min(m, n)
    Q = oracle.orgqr(At, T, m, n, 256, 32, k=k, nthreads=THREADS, h=2)
    assert np.linalg.norm(A - Q @ R) / (nA * n * EPS) < 10
    assert np.linalg.norm(np.eye(k) - Q.T @ Q) / (n * EPS) < 10


def test_tall_tiles_differ_from_square_and_repeat_bitwise():
    from gpu_util import run_factor
    A = tqr_inputs.normal(2048, 512, 5)
    _, At1, T1, R1 = _factor_tall(A)
    _, At2, T2, _ = _factor_tall(A)
    assert np.array_equal(At1, At2) and np.array_equal(T1, T2)  # out-of-order, bitwise reproducible
    g = run_factor(A, 256, 32)
    assert not np.allclose(g["R"], R1)  # another reflector sequence (R30): other signs / rounding
    D = np.sign(np.diag(g["R"])) * np.sign(np.diag(R1))
    np.testing.assert_allclose(D[:, None] * g["R"], R1, atol=1e-10 * np.linalg.norm(A), rtol=0)


def test_tall_tiles_c4_full_oracle_parity():
    cfg = tqr_inputs.CONFIGS["C4"]
    m, n = cfg["m"], cfg["n"]
    A = tqr_inputs.make(m, n, cfg["dist"], cfg["seed"])
    _, At, T, R = _factor_tall(A)
    At_o, T_o = oracle.geqrf(A, 256, 32, nthreads=THREADS, h=2)
    nA = np.linalg.norm(A)
    assert np.max(np.abs(R - oracle.get_r(At_o, m, n, 256))) <= 1e-10 * nA
    assert np.max(np.abs(At - At_o)) <= 1e-9 * nA
    assert np.max(np.abs(T - T_o)) <= 1e-9 * nA


def test_tall_tiles_unsupported_combinations():
    from paper_0707_3548_b200 import Plan
    from paper_0707_3548_b200.tqr import TqrError
    with pytest.raises(TqrError):
        Plan(512, 256, 128, 32, tall=True)
    plan = Plan(1024, 256, 256, 32, tall=True)
    At, T = plan.alloc()
    with pytest.raises(TqrError):
        plan.orgqr(At, T, 256, At)
