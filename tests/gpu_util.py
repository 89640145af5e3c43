"""Helpers for the GPU parity tests: run the CUDA path through the C-ABI binding."""
import numpy as np


def run_factor(A, b, s, trace=False, return_plan=False, locality=False):
    """A: numpy (m, n) float64 (any order).  Returns dict with numpy At, T, R and the plan."""
    import torch
    from paper_0707_3548_b200 import Plan
    m, n = A.shape
    plan = Plan(m, n, b, s, trace=trace, locality=locality)
    Ac = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(A).T)).cuda()  # column-major storage
    At, T = plan.alloc()
    plan.pack(Ac, At)
    plan.geqrf(At, T)
    R = torch.empty((n, min(m, n)), dtype=torch.float64, device="cuda")  # column-major min(m,n) x n
    plan.get_r(At, R)
    plan.sync()
    out = dict(At=At.cpu().numpy(), T=T.cpu().numpy(), R=R.cpu().numpy().T.copy(), plan=plan, At_dev=At, T_dev=T)
    return out


def tiles_to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()
