"""Quick timing of tlu_getrf (development aid; bench.py --method lu is the measured path)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import tqr_inputs
from paper_0707_3548_b200 import tlu

for arg in sys.argv[1:]:
    n, b, s = (int(x) for x in arg.split(","))
    plan = tlu.LUPlan(n, n, b, s, trace=False)
    A = torch.from_numpy(np.ascontiguousarray(tqr_inputs.make(n, n, "uniform", 9).T)).cuda()
    At, W, piv = plan.alloc()
    plan.pack(A, At)
    At0 = At.clone()
    ts = []
    for r in range(4):
        At.copy_(At0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(plan.stream)
        plan.getrf(At, W, piv)
        e1.record(plan.stream)
        plan.sync()
        ts.append(e0.elapsed_time(e1))
    t = min(ts[1:])
    f = tlu.flops_standard(n, n)
    print(f"LU n={n} b={b} s={s}: {t:.2f} ms  {f / t / 1e9:.1f} TFLOP/s std  ({tlu.flops_tiled(n, n, b, s) / t / 1e9:.1f} executed)  runs {['%.2f' % x for x in ts]}", flush=True)
