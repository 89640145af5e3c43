"""Parity on the task granularities that carry the headline flops (R23).

At C3 / C5 the factorization runs update tasks of np = 2 / 4 register passes that publish one
counter per pass (ocnt = np), switches to 1-pass tasks for the lookahead column and for the
tail steps, and prefetches the next pass of a task while the current one computes.  Shapes
of at most 6 x 5 tiles never leave the tail rule, so these mid-size shapes are chosen to
reach the multi-pass tasks: (4096^2, b=256) runs np = 2 in steps 0-3, (6144^2, b=512, s=64)
np = 4 in steps 0-2, and the emulated 4-rank job at 4096^2 the same np = 2 tasks on four
ranks' task streams.  Each test first asserts -- from the records the plan actually executes
(tqr_plan_records) -- that multi-pass tasks, multi-counter publications and the switch to
1-pass tasks are present, then compares R, V and T with the oracle on the same seeded input.
"""
import os

import numpy as np
import pytest

import oracle
import tqr_inputs

pytestmark = pytest.mark.gpu
THREADS = max(1, len(os.sched_getaffinity(0)))
K_L, K_S = 2, 3


def _plan_records(plan, G):
    return np.concatenate([plan.records(li) for li in range(G if G > 1 else 1)])


@pytest.mark.parametrize("m,n,b,s,G,npmax", [(4096, 4096, 256, 32, 1, 2), (6144, 6144, 512, 64, 1, 4),
                                             (4096, 4096, 256, 32, 4, 2)])
def test_multipass_tasks_parity(m, n, b, s, G, npmax):
    import torch
    from paper_0707_3548_b200 import Plan
    A = tqr_inputs.uniform(m, n, 60606 + m + G)
    plan = Plan(m, n, b, s, nranks=G, rank=0, emulate=G > 1)
    rec = _plan_records(plan, G)
    upd = rec[np.isin(rec[:, 0], (K_L, K_S))]
    npass, ocnt = upd[:, 15] & 0xFF, (upd[:, 15] >> 8) & 0xFF
    assert npass.max() == npmax and np.array_equal(npass, ocnt), "multi-pass tasks publish one counter per pass"
    multi_steps = set(upd[npass > 1, 1].tolist())
    assert 0 in multi_steps, "step 0 runs multi-pass update tasks"
    tail_steps = {k for k in set(upd[:, 1].tolist()) if np.all(npass[upd[:, 1] == k] == 1)}
    assert tail_steps and min(tail_steps) > max(multi_steps), "granularity switches to 1-pass tasks in the tail"
    # the lookahead column k+1 runs 1-pass tasks inside the multi-pass steps
    la = upd[(upd[:, 1] == 0) & (upd[:, 3] == 1)]
    assert len(la) and np.all(la[:, 15] & 0xFF == 1)

    Ac = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    At, T = plan.alloc()
    plan.pack(Ac, At)
    plan.geqrf(At, T)
    R = torch.empty((n, min(m, n)), dtype=torch.float64, device="cuda")
    plan.get_r(At, R)
    plan.sync()
    At_o, T_o = oracle.geqrf(A, b, s, nthreads=THREADS)
    R_o = oracle.get_r(At_o, m, n, b)
    nA = np.linalg.norm(A)
    err_r = np.max(np.abs(R.cpu().numpy().T - R_o))
    assert err_r <= 1e-10 * nA, (err_r, 1e-10 * nA)
    assert np.max(np.abs(At.cpu().numpy() - At_o)) <= 1e-9 * nA
    assert np.max(np.abs(T.cpu().numpy() - T_o)) <= 1e-9 * nA
