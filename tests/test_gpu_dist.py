"""GPU tests of the multi-GPU path on one B200 (include/tqr.h, multi-GPU section).

The 1D block-cyclic protocol (per-rank ticket streams, panel tasks storing packed V/T into
every rank's workspace and releasing every rank's panel counter) runs as ONE cooperative
launch over all ranks' data (TQR_FLAG_EMULATE_RANKS; the B200 profiling recipe forbids
separate waiting launches per rank on one GPU).  Invariant: R, V and T are
bitwise identical to the single-GPU factorization, and within 1e-10*||A||_F of the oracle.
The real-rank storage layout (own tile columns only) is checked through pack/unpack/get_r.
"""
import numpy as np
import pytest

import oracle
import tqr_inputs
from gpu_util import run_factor

pytestmark = pytest.mark.gpu


def _factor_emulated(A, b, s, G):
    import torch
    from paper_0707_3548_b200 import Plan
    m, n = A.shape
    plan = Plan(m, n, b, s, nranks=G, rank=0, emulate=True)
    Ac = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(A).T)).cuda()
    At, T = plan.alloc()
    plan.pack(Ac, At)
    plan.geqrf(At, T)
    R = torch.empty((n, min(m, n)), dtype=torch.float64, device="cuda")
    plan.get_r(At, R)
    plan.sync()
    return At.cpu().numpy(), T.cpu().numpy(), R.cpu().numpy().T.copy()


@pytest.mark.parametrize("m,n,b,s,G", [(256, 256, 64, 16, 2), (256, 256, 64, 16, 3), (700, 600, 256, 32, 2),
                                       (700, 600, 256, 32, 4), (1280, 300, 256, 32, 2), (520, 300, 128, 32, 8),
                                       (67, 41, 16, 8, 3), (2048, 2048, 128, 32, 8), (1100, 1030, 512, 64, 2)])
def test_emulated_ranks_bitwise_equal_single_gpu(m, n, b, s, G):
    A = tqr_inputs.uniform(m, n, 31 + m + G)
    g1 = run_factor(A, b, s)
    At, T, R = _factor_emulated(A, b, s, G)
    assert np.array_equal(At, g1["At"]), "V/R differ from the single-GPU factorization"
    assert np.array_equal(T, g1["T"]), "T differs from the single-GPU factorization"
    assert np.array_equal(R, g1["R"])
    if m * n <= 700 * 600:
        At_o, _ = oracle.geqrf(A, b, s, nthreads=4)
        R_o = oracle.get_r(At_o, m, n, b)
        assert np.max(np.abs(R - R_o)) <= 1e-10 * np.linalg.norm(A)


def test_emulated_ranks_repeat_and_trace():
    """Counter generations: repeated calls on one plan stay correct (no counter reset)."""
    import torch
    from paper_0707_3548_b200 import Plan
    A = tqr_inputs.uniform(512, 512, 77)
    g1 = run_factor(A, 128, 32)
    plan = Plan(512, 512, 128, 32, nranks=4, rank=0, emulate=True, trace=True)
    Ac = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(A).T)).cuda()
    At, T = plan.alloc()
    for _ in range(3):
        plan.pack(Ac, At)
        plan.geqrf(At, T)
    plan.sync()
    assert np.array_equal(At.cpu().numpy(), g1["At"])
    rec = plan.trace()
    # one trace record per executed task of the last call, over all four ranks' streams
    assert len(rec) == sum(len(plan.records(li)) for li in range(4))
    assert set(np.unique(rec[:, 0])) == {0, 1, 2, 3}
    assert np.all(rec[:, 7] >= rec[:, 6])  # end >= start


@pytest.mark.parametrize("G", [2, 3])
def test_real_rank_layout_pack_unpack_get_r(G):
    """Real multi-rank plans store only their own tile columns (storage column jl <-> global
    column rank + jl*G): pack -> unpack round trip per rank and get_r of the owned columns."""
    import torch
    from paper_0707_3548_b200 import Plan
    from paper_0707_3548_b200.dist import owned_columns
    m, n, b, s = 300, 700, 64, 16
    A = tqr_inputs.uniform(m, n, 5)
    Ac = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(A).T)).cuda()
    q = -(-n // b)
    back = torch.zeros_like(Ac)
    for r in range(G):
        plan = Plan(m, n, b, s, nranks=G, rank=r)
        At, T = plan.alloc()
        cols = owned_columns(q, G, r)
        assert At.numel() == plan.p * len(cols) * b * b
        plan.pack(Ac, At)
        plan.unpack(At, back)
        plan.sync()
        tiles = At.cpu().numpy().reshape(len(cols), plan.p, b, b)  # [jl][i][c][r]
        for jl, j in enumerate(cols):
            for i in range(plan.p):
                blk = A[i * b:(i + 1) * b, j * b:(j + 1) * b]
                got = tiles[jl, i].T[:blk.shape[0], :blk.shape[1]]
                assert np.array_equal(got, blk)
        R = torch.full((n, min(m, n)), 7.0, dtype=torch.float64, device="cuda")
        plan.get_r(At, R)
        plan.sync()
        Rn = R.cpu().numpy().T
        for j in range(n):
            if (j // b) % G == r:
                np.testing.assert_array_equal(Rn[:, j], np.where(np.arange(min(m, n)) <= j, A[:min(m, n), j], 0.0))
            else:
                assert np.all(Rn[:, j] == 7.0)
        with pytest.raises(Exception):
            plan.geqrf(At, T)  # not connected to its peers
        plan.close()
    assert np.array_equal(back.cpu().numpy(), Ac.cpu().numpy())


def _ipc_rank(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_0707_3548_b200 import Plan
    from paper_0707_3548_b200 import dist as tdist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        plan = Plan(1024, 1024, 128, 32, nranks=world, rank=rank)
        tdist.connect(plan)               # CUDA IPC blobs over torch.distributed
        plan.comm_ping(7000)              # peer stores into every rank's ping slots
        dist.barrier()
        out.put((rank, plan.comm_flags()))
        dist.barrier()
        plan.close()
    finally:
        dist.destroy_process_group()


def test_real_ranks_ipc_connect_and_peer_stores():
    """The real multi-GPU connection path, two processes on ONE GPU (no kernel waits on
    another rank, as the profiling recipe requires): export/exchange/open the CUDA IPC
    handles of each rank's symmetric buffer and store through the peer mappings at system
    scope; every rank must see every rank's store in its own ping slots."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_rank, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    assert res[0] == [7000, 7001] and res[1] == [7000, 7001], res


@pytest.mark.parametrize("m,n,b,s,G,nrhs", [(700, 600, 256, 32, 2, 300), (520, 300, 128, 32, 3, 260),
                                            (1100, 1030, 512, 64, 2, 200), (2048, 2048, 128, 32, 4, 500),
                                            (67, 41, 16, 8, 3, 20)])
def test_emulated_ranks_ormqr_orgqr_bitwise_equal_single_gpu(m, n, b, s, G, nrhs):
    """Multi-rank apply-Q / form-Q (include/tqr.h): B's tile columns block-cyclic over the
    ranks, every rank's workspace filled with every rank's reflector panels, each rank
    applying Q to its own columns -- bitwise equal to the single-GPU apply (same per-tile
    operation sequence) and within the oracle's tolerance."""
    import torch
    from paper_0707_3548_b200 import Plan
    A = tqr_inputs.uniform(m, n, 41 + m + G)
    g1 = run_factor(A, b, s)
    p1 = g1["plan"]
    pe = Plan(m, n, b, s, nranks=G, rank=0, emulate=True)
    At = torch.from_numpy(g1["At"]).cuda()
    T = torch.from_numpy(g1["T"]).cuda()
    Bm = tqr_inputs.uniform(m, nrhs, 7 + G)
    for trans in ("T", "N"):
        B1 = torch.from_numpy(oracle.pack(Bm, b)).cuda()
        Be = B1.clone()
        p1.ormqr(trans, g1["At_dev"], g1["T_dev"], B1, nrhs)
        pe.ormqr(trans, At, T, Be, nrhs)
        torch.cuda.synchronize()
        assert torch.equal(B1, Be), f"apply-Q ({trans}) differs from the single-GPU result"
        want = oracle.ormqr(g1["At"], g1["T"], m, n, b, s, Bm, 1 if trans == "T" else 0, nthreads=4)
        got = oracle.unpack(Be.cpu().numpy(), m, nrhs, b)
        col_err = np.linalg.norm(got - want, axis=0) / np.linalg.norm(Bm, axis=0)
        assert np.max(col_err) <= 10 * m * np.finfo(np.float64).eps
    k = min(m, n)
    qb = -(-k // b)
    Q1 = torch.empty(p1.p * qb * b * b, dtype=torch.float64, device="cuda")
    Qe = torch.full_like(Q1, 3.0)
    p1.orgqr(g1["At_dev"], g1["T_dev"], k, Q1)
    pe.orgqr(At, T, k, Qe)
    torch.cuda.synchronize()
    assert torch.equal(Q1, Qe), "form-Q differs from the single-GPU result"
    pe.close()
