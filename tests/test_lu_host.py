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


def _footprint(rec, nb):
    """(reads, writes) of one task as region keys (LU7, LU11): ("A", i, j, slice) a
    64-column slice of tile (i, j) ("all" = the whole tile); ("U", k, l) U_kk's rows of inner block
    l; ("L", k) A_kk's strict lower part with GETRF's W / interchange slots.  GETRF block l writes
    the rows of blocks >= l; TSTRF block l touches U_kk's block-l rows only."""
    kind, k, i, j, sl = (int(x) for x in rec[:5])
    if kind == 0:
        ls = range(nb) if sl < 0 else range(sl, nb)
        return set(), {("A", k, k, "all"), ("L", k)} | {("U", k, l) for l in ls}
    if kind == 1:
        ls = range(nb) if sl < 0 else [sl]
        rw = {("A", i, k, "all")} | {("U", k, l) for l in ls}
        return set(rw), set(rw)
    if kind == 2:
        return {("L", k)}, {("A", k, j, sl)}
    return {("A", i, k, "all")}, {("A", k, j, sl), ("A", i, j, sl)}


def _sequential_order(p, q, nsl, nb):
    """oracle_lu.c's order, panels by inner block: step k: GETRF(k) blocks, TSTRF(k, i) blocks
    for all i, then per column j: GESSM, SSSSM chain"""
    K = min(p, q)
    seq = []
    for k in range(K):
        seq += [(0, k, k, k, l) for l in range(nb)]
        seq += [(1, k, i, k, l) for i in range(k + 1, p) for l in range(nb)]
        for j in range(k + 1, q):
            for sl in range(nsl):
                seq.append((2, k, k, j, sl))
                seq += [(3, k, i, j, sl) for i in range(k + 1, p)]
    return seq


def _key(reg):
    return reg[:3] if reg[0] == "A" else reg


def _conflicts(a, b, nb):
    ra, wa = _footprint(a, nb)
    rb, wb = _footprint(b, nb)
    def hit(x, y):  # "all" slices of a tile overlap every slice of it
        for u in x:
            for v in y:
                if _key(u) == _key(v) and (u[0] != "A" or u[3] == "all" or v[3] == "all" or u[3] == v[3]):
                    return True
        return False
    return hit(wa, rb | wb) or hit(wb, ra)


def _replay(rec, nctr, p, q, nsl, nb, workers, seed, hold=False):
    """Replay the tickets on `workers` simulated CTAs that finish in random order; a task starts
    only when its counter dependencies hold.  Returns the first (task, earlier conflicting task
    not yet done) violation, or None; raises on deadlock.  hold: a CTA running an update task may
    take its next ticket early (the executor's dispatch pipelining, LU_NEXT); that ticket is
    then out of the pool but starts only after the CTA's current task."""
    seq = _sequential_order(p, q, nsl, nb)
    pos = {t: x for x, t in enumerate(seq)}
    by_region = {}
    for t in seq:
        r_, w_ = _footprint(t, nb)
        for reg in r_ | w_:
            by_region.setdefault(_key(reg), []).append(t)
    rng = random.Random(seed)
    ctr = [0] * nctr
    done, running, nxt = set(), [], 0
    held = {}  # running ticket -> the ticket its CTA holds ahead
    while nxt < len(rec) or running:
        while nxt < len(rec) and len(running) < workers:
            running.append(nxt)
            nxt += 1
        if hold:
            for t in running:
                if t not in held and nxt < len(rec) and rec[t][0] >= 2 and rng.random() < 0.7:
                    held[t] = nxt
                    nxt += 1
        ready = [t for t in running
                 if all(ctr[(rec[t][8 + 2 * d] & 0xFFFFFF) + x] >= rec[t][9 + 2 * d]
                        for d in range(3) for x in range(int(rec[t][8 + 2 * d]) >> 24))]
        if not ready:
            raise RuntimeError("deadlock")
        t = rng.choice(ready)
        key = tuple(int(v) for v in rec[t][:5])
        for reg in (lambda rw: rw[0] | rw[1])(_footprint(key, nb)):
            for other in by_region[_key(reg)]:
                if pos[other] < pos[key] and _conflicts(other, key, nb) and other not in done:
                    return key, other
        running.remove(t)
        if t in held:
            running.append(held.pop(t))  # the same CTA goes on with the ticket it holds
        done.add(key)
        ctr[rec[t][5]] = max(ctr[rec[t][5]], int(rec[t][6]))
    return None


@pytest.mark.parametrize("m,n,b,s,workers", [(256, 256, 64, 16, 3), (320, 192, 64, 16, 5), (192, 320, 64, 16, 4),
                                              (1024, 1024, 256, 32, 7), (640, 384, 128, 32, 6),
                                              (2048, 512, 256, 32, 9)])
def test_dispatch_order_respects_every_data_dependence(L, m, n, b, s, workers):
    """Every pair of tasks that conflict on a region runs in the oracle's sequential order (the
    earlier one finished before the later starts), and every ticket eventually runs."""
    rec, nctr = L.schedule_records(m, n, b, s, workers)
    p, q = -(-m // b), -(-n // b)
    nsl, nb = b // min(64, b), b // s
    seq = _sequential_order(p, q, nsl, nb)
    assert len(rec) == len(seq) and sorted(tuple(int(v) for v in r[:5]) for r in rec) == sorted(seq)
    for seed in range(3):
        assert _replay(rec, nctr, p, q, nsl, nb, workers, seed) is None


@pytest.mark.parametrize("m,n,b,s,workers", [(320, 192, 64, 16, 2), (1024, 1024, 256, 32, 7), (2048, 512, 256, 32, 3)])
def test_holding_one_ticket_ahead_neither_deadlocks_nor_races(L, m, n, b, s, workers):
    """The executor's dispatch pipelining (LU_NEXT): a CTA takes its next ticket half-way through
    an update task.  Every wait is on a smaller ticket and the smallest unfinished ticket is some
    CTA's current task, so the replay never stalls and the data dependences still hold."""
    rec, nctr = L.schedule_records(m, n, b, s, workers)
    p, q = -(-m // b), -(-n // b)
    nsl, nb = b // min(64, b), b // s
    for seed in range(4):
        assert _replay(rec, nctr, p, q, nsl, nb, workers, seed, hold=True) is None


def test_replay_detects_a_dropped_dependency(L):
    """Negative control: drop TSTRF(k,i,l)'s dependency on its tile's previous block (or a
    chain dependency of an SSSSM) and the replay finds the race."""
    m = n = 512
    b, s, workers = 128, 32, 6
    rec, nctr = L.schedule_records(m, n, b, s, workers)
    p = q = m // b
    nsl, nb = 2, 4
    for kind, slot in [(1, 1), (3, 1)]:
        bad = rec.copy()
        hits = [t for t in range(len(bad)) if bad[t][0] == kind and (kind != 1 or bad[t][4] > 0)
                and (bad[t][8 + 2 * slot] >> 24) > 0]
        for t in hits:
            bad[t][8 + 2 * slot] = 0
        found = any(_replay(bad, nctr, p, q, nsl, nb, workers, seed) is not None for seed in range(6))
        assert found, kind
