"""Per-kind task statistics of one traced tlu_getrf (development aid): SM-time shares,
median durations, busy fraction, utilisation by decile."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import tqr_inputs
from paper_0707_3548_b200 import tlu

NAMES = {0: "GETRF", 1: "TSTRF", 2: "GESSM", 3: "SSSSM"}
for arg in sys.argv[1:]:
    n, b, s = (int(x) for x in arg.split(","))
    plan = tlu.LUPlan(n, n, b, s, trace=True)
    A = torch.from_numpy(np.ascontiguousarray(tqr_inputs.make(n, n, "uniform", 9).T)).cuda()
    At, W, piv = plan.alloc()
    for _ in range(2):
        plan.pack(A, At)
        plan.getrf(At, W, piv)
        plan.sync()
    tr = plan.trace()
    t0 = tr[:, 5].min()
    start, end = tr[:, 6] - t0, tr[:, 7] - t0
    dur = (end - start) / 1e3
    span = (end.max()) / 1e6
    nsm = len(np.unique(tr[:, 4]))
    tot = dur.sum() / 1e3
    print(f"n={n} b={b} s={s}: makespan {span:.2f} ms, {len(tr)} tasks on {nsm} SMs, busy {tot / (span * nsm):.3f}")
    for k in range(4):
        sel = tr[:, 0] == k
        if sel.any():
            print(f"  {NAMES[k]}: n={sel.sum():6d} median {np.median(dur[sel]):8.1f} us  total {dur[sel].sum() / 1e3:9.1f} SM-ms ({100 * dur[sel].sum() / 1e3 / tot:.1f}%)")
    wait = (tr[:, 6] - tr[:, 5]) / 1e3
    print(f"  dependency wait: mean {wait.mean():.1f} us, total {wait.sum() / 1e3:.1f} SM-ms")
    edges = np.linspace(0, end.max(), 11)
    util = []
    for a, b_ in zip(edges[:-1], edges[1:]):
        ov = np.clip(np.minimum(end, b_) - np.maximum(start, a), 0, None).sum()
        util.append(ov / ((b_ - a) * nsm))
    print("  utilisation by decile: " + " ".join(f"{u:.2f}" for u in util))
    kk = tr[:, 1]
    gs = [start[(tr[:, 0] == 0) & (kk == k)].min() / 1e6 for k in range(0, n // b, max(1, n // b // 8))]
    print("  GETRF(k) start ms every few k: " + " ".join(f"{x:.1f}" for x in gs))
