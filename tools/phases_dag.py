"""Phase breakdown (thread-0 clock64 totals per CTA) of ONE real DAG factorization, with the
profiling build (TQR_PHASES=1 python paper_0707_3548_b200/build.py).  Development aid.
  TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_phases.so python tools/phases_dag.py --config C3
"""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0707_3548_b200 as tqr  # noqa: E402
import tqr_inputs  # noqa: E402

NAMES = ["prologue", "ticket+record", "end barrier", "release", "update blocks", "store", "dep wait",
         "panel-update", "stage", "factor", "V/R out", "gram+Yp", "build_t", "T out", "upd setup",
         "C1 wait"]
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
a = ap.parse_args()
cfg = tqr_inputs.CONFIGS[a.config]
m, n, b, s = cfg["m"], cfg["n"], cfg["b"], cfg["s"]
plan = tqr.Plan(m, n, b, s)
At, T = plan.alloc()
At.uniform_(-0.5, 0.5)
A0 = At.clone()
PH = torch.zeros(16, dtype=torch.int64, device="cuda")
plan.geqrf(At, T)
plan.sync()
At.copy_(A0)
plan.phase_counters(PH)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(plan.stream)
plan.geqrf(At, T)
e1.record(plan.stream)
plan.sync()
ms = e0.elapsed_time(e1)
v = PH.cpu().numpy().astype(np.float64)
tot = v.sum()
print(f"{a.config}: {ms:.1f} ms; thread-0 cycles per CTA {tot / 148 / 1.965e6:.1f} ms-equivalent")
for name, x in zip(NAMES, v):
    if x:
        print(f"  {name:14s} {100 * x / tot:5.1f}%")
