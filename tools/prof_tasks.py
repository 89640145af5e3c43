"""Time (and, under ncu, profile) independent batches of one task kind through the executor.

  python tools/prof_tasks.py [--b 256 --s 32] [--kinds 0,1,2,3] [--count N] [--reps R]
Prints per-task time and achieved GFLOP/s per SM for each kind (flop model of DESIGN.md R15).
"""
import argparse
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_0707_3548_b200 as tqr  # noqa: E402

PHASE_NAMES = ["prologue", "ticket+record", "end barrier", "release", "update blocks", "store", "dep wait",
               "panel-update", "stage", "factor", "V/R out", "gram+Yp", "build_t", "T out", "upd setup",
         "C1 wait"]
ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=256)
ap.add_argument("--s", type=int, default=32)
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--m", type=int, default=0, help="rows (default n; m >= 4n gives the tall-skinny plan)")
ap.add_argument("--kinds", default="0,1,2,3")
ap.add_argument("--count", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
b, s = a.b, a.s
plan = tqr.Plan(a.m or a.n, a.n, b, s)
info = plan.info()
import os  # noqa: E402
PH = None
if os.environ.get("TQR_LIB", "").endswith("libtqr_phases.so") or os.environ.get("TQR_PH") == "1":
    PH = torch.zeros(16, dtype=torch.int64, device="cuda")
    plan.phase_counters(PH)
At, T = plan.alloc()
At.uniform_(-0.5, 0.5)
T.uniform_(-0.1, 0.1)
W = plan.work()
W.view(torch.float64).uniform_(-0.1, 0.1) if W.numel() % 8 == 0 else None
B, S = float(b), float(s)
w = info["slice"] * info["passes"]  # columns per update task
fl = {0: 4 / 3 * B ** 3 + 2 / 3 * S * B * B, 1: 2 * B ** 3 + 4 / 3 * S * B * B, 2: 2 * B * B * w + S * B * w,
      3: 4 * B * B * w + S * B * w}
fl.update({4: fl[2], 5: fl[3], 6: fl[2], 7: fl[3]})
# factor parts alone (one inner block): rank-1 panel updates + Gram, per block
fl.update({8: (2 * B * S * S + B * S * S) / 2, 9: 2 * B * S * S + B * S * S})
for kind in [int(x) for x in a.kinds.split(",")]:
    count = a.count or (148 if kind in (0, 1, 8, 9) else 148 * 8)
    for r in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(plan.stream)
        plan.profile_tasks(kind, count, At, T)
        e1.record(plan.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    waves = -(-count // 148)
    if PH is not None:
        v = PH.cpu().tolist()
        PH.zero_()
        tot = sum(v)
        names = PHASE_NAMES
        print("   phases (% of warp-0 cycles, all reps): " + ", ".join(f"{n} {100*x/tot:.1f}" for n, x in zip(names, v) if x))
        per = count * a.reps
        print("   phases (cycles per task, thread 0): " + ", ".join(f"{n} {x / per:.0f}" for n, x in zip(names, v) if x)
              + f"  | total {tot / per:.0f}")
    per_task_us = ms * 1e3 / waves
    print(f"kind {['G','T','L','S','LQT','SQT','LQ','SQ','G-factor-part','T-factor-part'][kind]} b={b} s={s}: {count} tasks in {ms:.3f} ms -> {per_task_us:.1f} us/task/SM, "
          f"{fl[kind] / (per_task_us * 1e3):.1f} GFLOP/s per SM ({100 * fl[kind] / (per_task_us * 1e3) / 251:.1f}% of 251)",
          flush=True)
