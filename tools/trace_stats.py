"""Summarise a bench.py --trace JSON: per-kind durations, SM utilisation over time, panel
critical-path timing.  Development aid."""
import json
import sys

import numpy as np

d = json.load(open(sys.argv[1]))
r = np.array(d["records"], dtype=np.int64)
kind, k, i, j, slf, sm, st, en = r.T
sl = slf & 0xFF  # slice (low byte; tall apply sub-tasks carry lp + 1 in bits 8..15) | task flags << 16
t0 = st.min()
st = (st - t0) / 1e3
en = (en - t0) / 1e3
dur = en - st
T = en.max()
nsm = len(set(sm.tolist()))
print(f"makespan {T / 1e3:.1f} ms, tasks {len(r)}, SMs {nsm}")
for kd, name in enumerate("GTLS"):
    m = kind == kd
    if m.any():
        print(f"  {name}: n={m.sum():6d} median {np.median(dur[m]):8.1f} us  total {dur[m].sum() / 1e3:9.1f} SM-ms "
              f"({100 * dur[m].sum() / (nsm * T):.1f}% of SM-time)")
print(f"  busy fraction {dur.sum() / (nsm * T):.3f}")
g = np.where(kind == 0)[0]
gs = st[g][np.argsort(k[g])]
print("  G(k) start (ms) every 8th:", np.round(gs[::8] / 1e3, 1))
# panel chain: T tasks of step k: time from first to last
for kk in [0, 1, 8, 32, 48, 60]:
    m = (kind == 1) & (k == kk)
    if m.any():
        print(f"  step {kk}: T chain {st[m].min() / 1e3:.1f} -> {en[m].max() / 1e3:.1f} ms ({m.sum()} TSQRTs, "
              f"median {np.median(dur[m]):.0f} us)")
bins = np.linspace(0, T, 11)
u = []
for a, b in zip(bins[:-1], bins[1:]):
    u.append(np.clip(np.minimum(en, b) - np.maximum(st, a), 0, None).sum() / (nsm * (b - a)))
print("  utilisation by decile:", " ".join(f"{x:.2f}" for x in u))

# panel sub-tasks by inner block l (slice field)
for kd, name in ((0, "G"), (1, "T")):
    m = kind == kd
    if m.any() and sl[m].max() > 0:
        print(f"  {name} sub-task median by block l:", " ".join(f"{np.median(dur[m & (sl == l)]):.0f}"
                                                            for l in range(sl[m].max() + 1)))

# per-SM gaps (dispatch + dependency wait) attributed to the task that follows the gap
order = np.lexsort((st, sm))
gap = np.zeros(len(r))
same = sm[order][1:] == sm[order][:-1]
g = (st[order][1:] - en[order][:-1])
gap[order[1:][same]] = g[same]
for kd, name in enumerate("GTLS"):
    m = kind == kd
    if m.any():
        print(f"  gap before {name}: mean {gap[m].mean():7.1f} us, p90 {np.percentile(gap[m], 90):7.1f} us, "
              f"total {gap[m].sum() / 1e3:8.1f} SM-ms")
# panel parts per inner block (R21): apply (flags 2) / factor (flags 4) / fused
fl = (slf >> 16) & 0xFF
blk = sl
pm = (kind <= 1)
if pm.any():
    print("  panel parts per block l (median us): l: apply / factor / fused")
    for l in sorted(set(blk[pm].tolist())):
        mA = pm & (blk == l) & ((fl & 2) != 0)
        mF = pm & (blk == l) & ((fl & 4) != 0)
        mU = pm & (blk == l) & ((fl & 6) == 0)
        f = lambda m: f"{np.median(dur[m]):6.1f}" if m.any() else "    - "
        print(f"    l={l}: {f(mA)} / {f(mF)} / {f(mU)}")
