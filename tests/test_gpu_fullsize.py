"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(default Plan: persistent executor, one CTA per SM).

* C2 (4096^2, b=128), C3 (16384^2, b=256, the bench workload; ~80 s of oracle on 16 host
  threads) and C4 (131072 x 2048, b=256, N(0,1)): the full oracle on the same seeded input;
  R elementwise within 1e-10 * ||A||_F (BJ north_star), V and T elementwise, plus backward
  error / orthogonality of the GPU's own factors through the library's form-Q.
* C5 (65536^2, b=512): strip parity -- the oracle factors the first 2 tile columns (m x 2b);
  tiled QR on those columns performs exactly the operations the full factorization performs
  on them (their tasks never read later columns), so R[:2b, :2b] and the V tiles of those
  columns must match -- plus properties that hold at any size: column norms
  ||R[:, j]|| = ||A[:, j]||, an R^T R = A^T A sketch, and backward-error / orthogonality
  sketches through the library's apply-Q.  Reference matmuls in the checks are cuBLAS fp64 via torch (test
  infrastructure only).
"""
import os

import numpy as np
import pytest

import oracle
import tqr_inputs

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps
THREADS = max(1, len(os.sched_getaffinity(0)))


def _factor(cfg, A):
    import torch
    from paper_0707_3548_b200 import Plan
    m, n, b, s = cfg["m"], cfg["n"], cfg["b"], cfg["s"]
    plan = Plan(m, n, b, s)
    Ad = torch.from_numpy(A.T).cuda()  # column-major storage (A is Fortran-ordered)
    At, T = plan.alloc()
    plan.pack(Ad, At)
    plan.geqrf(At, T)
    R = torch.empty((n, min(m, n)), dtype=torch.float64, device="cuda")  # column-major R
    plan.get_r(At, R)
    plan.sync()
    return plan, Ad, At, T, R


def _colnorm_and_gram_sketch(Ad, R):
    """||R[:,j]|| == ||A[:,j]|| for every column; R^T(Rx) vs A^T(Ax) for 8 Gaussian x."""
    import torch
    nA = torch.linalg.norm(Ad).item()
    cn_A = torch.linalg.norm(Ad, dim=1)          # rows of the storage = matrix columns
    cn_R = torch.linalg.norm(R, dim=1)
    m = Ad.shape[1]
    assert torch.max(torch.abs(cn_A - cn_R)).item() <= 10 * m * EPS * torch.max(cn_A).item()
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(Ad.shape[0], 8, dtype=torch.float64, device="cuda", generator=g)
    A_ = Ad.t()                                  # m x n view
    R_ = R.t()                                   # k x n view
    lhs = R_.t() @ (R_ @ x)
    rhs = A_.t() @ (A_ @ x)
    rel = torch.linalg.norm(lhs - rhs).item() / (nA * nA * torch.linalg.norm(x).item())
    assert rel < 10 * max(Ad.shape) * EPS, rel
    return nA


def _strip_parity(cfg, A, At, R, c=2):
    """Oracle on the first c tile columns; compare R[:cb, :cb] and the strip's V tiles."""
    m, b, s = cfg["m"], cfg["b"], cfg["s"]
    w = c * b
    At_o, _ = oracle.geqrf(np.asfortranarray(A[:, :w]), b, s, nthreads=THREADS)
    R_o = oracle.get_r(At_o, m, w, b)
    R_g = R[:w, :w].cpu().numpy().T
    nA = np.linalg.norm(A[:, :w])
    assert np.max(np.abs(np.triu(R_g) - np.triu(R_o))) <= 1e-10 * np.linalg.norm(A)
    p = -(-m // b)
    strip_g = At[: p * w * b].cpu().numpy()       # tile columns 0..c-1 (contiguous slabs)
    assert np.max(np.abs(strip_g - At_o)) <= 1e-9 * max(1.0, nA)


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_full_oracle_parity(name):
    import torch
    cfg = tqr_inputs.CONFIGS[name]
    m, n, b, s = cfg["m"], cfg["n"], cfg["b"], cfg["s"]
    A = tqr_inputs.make(m, n, cfg["dist"], cfg["seed"])
    plan, Ad, At, T, R = _factor(cfg, A)
    At_o, T_o = oracle.geqrf(A, b, s, nthreads=THREADS)
    R_o = oracle.get_r(At_o, m, n, b)
    nA = np.linalg.norm(A)
    assert np.max(np.abs(R.cpu().numpy().T - R_o)) <= 1e-10 * nA
    del R_o
    assert np.max(np.abs(At.cpu().numpy() - At_o)) <= 1e-9 * nA
    del At_o
    assert np.max(np.abs(T.cpu().numpy() - T_o)) <= 1e-9 * nA
    del T_o
    _colnorm_and_gram_sketch(Ad, R)
    # backward error and orthogonality of the GPU factors, thin Q by the library's form-Q
    qb = -(-n // b)
    Qt = torch.empty(plan.p * qb * b * b, dtype=torch.float64, device="cuda")
    plan.orgqr(At, T, n, Qt)
    Qc = torch.empty((n, m), dtype=torch.float64, device="cuda")
    _unpack_into(plan, Qt, Qc, m, n, b)
    Q = Qc.t()
    Rm = R.t()
    be = torch.linalg.norm(Ad.t() - Q @ Rm).item() / (nA * n * EPS)
    orth = torch.linalg.norm(torch.eye(n, dtype=torch.float64, device="cuda") - Q.t() @ Q).item() / (n * EPS)
    assert be < 10 and orth < 10, (be, orth)


def _unpack_into(plan, Qt, Qc, m, k, b):
    """Tile-major m x k (p x ceil(k/b) tiles) -> column-major storage (k, m), on the GPU."""
    p, qb = plan.p, -(-k // b)
    tiles = Qt.view(qb, p, b, b)                     # [jt][i][c][r]
    full = tiles.permute(0, 2, 1, 3).reshape(qb * b, p * b)  # [col][row]
    Qc.copy_(full[:k, :m])


def test_c5_strip_parity_and_sketches():
    import torch
    cfg = tqr_inputs.CONFIGS["C5"]
    m, n, b = cfg["m"], cfg["n"], cfg["b"]
    A = tqr_inputs.make(m, n, cfg["dist"], cfg["seed"])
    plan, Ad, At, T, R = _factor(cfg, A)
    _strip_parity(cfg, A, At, R)
    del A
    nA = _colnorm_and_gram_sketch(Ad, R)
    # backward-error sketch ||A X - Q (R X)||, orthogonality sketch ||Q^T Q x - x||, X: m x 8
    g = torch.Generator(device="cuda").manual_seed(11)
    X = torch.randn(n, 8, dtype=torch.float64, device="cuda", generator=g)
    RX = R.t() @ X                                   # n x 8 (k = n)
    Bt = torch.zeros(plan.p * b * b, dtype=torch.float64, device="cuda")
    Bv = Bt.view(plan.p, b, b)                       # [i][c][r]: one tile column of width b
    Bv[:, :8, :] = RX.t().reshape(8, plan.p, b).permute(1, 0, 2)
    plan.ormqr("N", At, T, Bt, 8)
    plan.sync()
    QRX = Bv[:, :8, :].permute(1, 0, 2).reshape(8, m).t()
    AX = Ad.t() @ X
    be = torch.linalg.norm(AX - QRX).item() / (nA * torch.linalg.norm(X).item() * n * EPS)
    plan.ormqr("T", At, T, Bt, 8)
    plan.sync()
    back = Bv[:, :8, :].permute(1, 0, 2).reshape(8, m).t()
    orth = torch.linalg.norm(back - RX).item() / (torch.linalg.norm(RX).item() * n * EPS)
    assert be < 10 and orth < 10, (be, orth)
