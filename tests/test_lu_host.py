"""CPU-side checks of the tiled-LU entry points (include/tlu.h): exports, flop counts (an
implementation independent of the oracle's, checked against it), argument validation, and a
replay of the dispatch order (tlu_schedule_records) against the data dependences of the
oracle's sequential order (oracle_lu.c's driver, LU7)."""
import os
import random
import re
import subprocess

import pytest

import oracle
from conftest import ROOT


@pytest.fixture(scope="module")
def L():
    from paper_0707_3548_b200.build import build
    build()
    from paper_0707_3548_b200 import tlu
    return tlu


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "tlu.h")).read()
    declared = sorted(set(re.findall(r"\b(tlu_[a-z_]+)\s*\(", hdr)))
    from paper_0707_3548_b200.tqr import LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (tlu_[a-z_]+)", out))
    assert not [s for s in declared if s not in exported]
    assert len(declared) >= 15


def test_flop_counts_match_oracle(L):
    for m, n in [(3000, 3000), (4096, 1024), (100, 300), (1, 1)]:
        assert L.flops_standard(m, n) == pytest.approx(oracle.lu_flops_standard(m, n), rel=1e-15)
    for m, n, b, s in [(16384, 16384, 256, 32), (4096, 4096, 128, 32), (1000, 700, 64, 16), (64, 64, 64, 64)]:
        assert L.flops_tiled(m, n, b, s) == pytest.approx(oracle.lu_flops_tiled(m, n, b, s), rel=1e-13)


def test_invalid_args_and_support(L):
    import ctypes
    lib = L.lib()
    h = ctypes.c_void_p()
    for bad, idx in [(dict(m=0), 1), (dict(n=0), 2), (dict(b=0), 3), (dict(s=3), 4), (dict(s=0), 4)]:
        prm = dict(m=100, n=100, b=64, s=16)
        prm.update(bad)
        P = L._Params(prm["m"], prm["n"], prm["b"], prm["s"], 0, None, 0)
        assert lib.tlu_plan_create(ctypes.byref(h), ctypes.byref(P)) == 1 and lib.tqr_last_bad_arg() == idx, bad
    assert L.supported(256, 32) and L.supported(128, 32) and L.supported(64, 16) and not L.supported(32, 8)
    P = L._Params(100, 100, 32, 8, 0, None, 0)
    assert lib.tlu_plan_create(ctypes.byref(h), ctypes.byref(P)) == 5   # valid, not built


def _footprint(rec):
    """(reads, writes) of one task as region keys; tile (k,k) is split into its U part (upper
    incl. diagonal: GETRF, TSTRF) and its L part (strict lower: GETRF writes, GESSM reads),
    update tasks touch one 64-column slice of their tiles (LU7)."""
    kind, k, i, j, sl = (int(x) for x in rec[:5])
    if kind == 0:
        return set(), {("U", k, k), ("L", k, k), ("T", k, k, "all")}
    if kind == 1:
        return {("U", k, k)}, {("U", k, k), ("T", i, k, "all")}
    if kind == 2:
        return {("L", k, k), ("T", k, k, "all")}, {("T", k, j, sl)}
    return {("T", i, k, "all")}, {("T", k, j, sl), ("T", i, j, sl)}


def _sequential_order(p, q, nsl):
    """oracle_lu.c's order: step k: GETRF, TSTRF(k, i) for all i, then per column j: GESSM, SSSSM chain"""
    K = min(p, q)
    seq = []
    for k in range(K):
        seq.append((0, k, k, k, -1))
        seq += [(1, k, i, k, -1) for i in range(k + 1, p)]
        for j in range(k + 1, q):
            for sl in range(nsl):
                seq.append((2, k, k, j, sl))
                seq += [(3, k, i, j, sl) for i in range(k + 1, p)]
    return seq


def _conflicts(a, b):
    ra, wa = _footprint(a)
    rb, wb = _footprint(b)
    def hit(x, y):  # "all" slices of a tile overlap every slice of it
        for u in x:
            for v in y:
                if u[:3] == v[:3] and (u[0] != "T" or u[3] == "all" or v[3] == "all" or u[3] == v[3]):
                    return True
        return False
    return hit(wa, rb | wb) or hit(wb, ra)


@pytest.mark.parametrize("m,n,b,s,workers", [(256, 256, 64, 16, 3), (320, 192, 64, 16, 5), (192, 320, 64, 16, 4),
                                              (1024, 1024, 256, 32, 7), (640, 384, 128, 32, 6),
                                              (2048, 512, 256, 32, 9)])
def test_dispatch_order_respects_every_data_dependence(L, m, n, b, s, workers):
    """Replay the tickets on `workers` simulated CTAs that finish in random order; a task starts
    only when its counter dependencies hold.  Every pair of tasks that conflict on a region must
    run in the oracle's sequential order (the earlier one finished before the later starts), and
    every ticket must eventually run (no deadlock)."""
    rec, nctr = L.schedule_records(m, n, b, s, workers)
    p, q = -(-m // b), -(-n // b)
    nsl = b // min(64, b)
    seq = _sequential_order(p, q, nsl)
    pos = {t: x for x, t in enumerate(seq)}
    assert len(rec) == len(seq) and sorted(tuple(int(v) for v in r[:5]) for r in rec) == sorted(seq)
    by_region = {}
    for t in seq:
        r_, w_ = _footprint(t)
        for reg in r_ | w_:
            by_region.setdefault(reg[:3], []).append(t)
    for seed in range(3):
        rng = random.Random(seed)
        ctr = [0] * nctr
        done, running, nxt = set(), [], 0
        while nxt < len(rec) or running:
            while nxt < len(rec) and len(running) < workers:
                running.append(nxt)
                nxt += 1
            ready = []
            for t in running:
                r = rec[t]
                ok = all(ctr[(r[8 + 2 * d] & 0xFFFFFF) + x] >= r[9 + 2 * d]
                         for d in range(3) for x in range(int(r[8 + 2 * d]) >> 24))
                if ok:
                    ready.append(t)
            assert ready, "deadlock"
            t = rng.choice(ready)
            key = tuple(int(v) for v in rec[t][:5])
            for reg in (lambda rw: rw[0] | rw[1])(_footprint(key)):
                for other in by_region[reg[:3]]:
                    if pos[other] < pos[key] and _conflicts(other, key):
                        assert other in done, (key, other)
            running.remove(t)
            done.add(key)
            ctr[rec[t][5]] = max(ctr[rec[t][5]], int(rec[t][6]))
