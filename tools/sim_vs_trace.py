"""Compare the list schedule's model (TQR_DEV_SIMDUMP file) with a measured trace (bench.py
--trace JSON): makespan, utilisation by decile, per-kind median durations, the T-chain
progress of a few steps.  Development aid.
  python tools/sim_vs_trace.py SIMDUMP TRACE.json[.gz]"""
import gzip
import json
import sys

import numpy as np


def util(kind, k, st, en, nsm):
    T = en.max()
    bins = np.linspace(0, T, 11)
    return T, [np.clip(np.minimum(en, b) - np.maximum(st, a), 0, None).sum() / (nsm * (b - a))
               for a, b in zip(bins[:-1], bins[1:])]


sim = np.loadtxt(sys.argv[1], dtype=np.float64)
op = gzip.open if sys.argv[2].endswith(".gz") else open
tr = np.array(json.load(op(sys.argv[2]))["records"], dtype=np.int64)
nsm = len(set(tr[:, 5].tolist()))
sk, skk, si = sim[:, 0].astype(int), sim[:, 1].astype(int), sim[:, 2].astype(int)
ss, se = sim[:, 5] / 1e3, sim[:, 6] / 1e3
tk, tkk, ti = tr[:, 0], tr[:, 1], tr[:, 2]
t0 = tr[:, 6].min()
ts, te = (tr[:, 6] - t0) / 1e3, (tr[:, 7] - t0) / 1e3
for name, (kd, kk, st, en) in (("model", (sk, skk, ss, se)), ("trace", (tk, tkk, ts, te))):
    T, u = util(kd, kk, st, en, nsm)
    print(f"{name}: makespan {T / 1e3:.2f} ms; utilisation by decile " + " ".join(f"{x:.2f}" for x in u))
    print("   median us " + " ".join(f"{n}:{np.median((en - st)[kd == c]):.1f}" for c, n in enumerate("GTLS") if (kd == c).any()))
    for step in (0, 1, 2, 8):
        m = (kd == 1) & (kk == step)
        if m.any():
            print(f"   step {step}: T chain {st[m].min() / 1e3:.2f} -> {en[m].max() / 1e3:.2f} ms")
