"""Race check of the executor's task footprints (no GPU needed).

The dispatch records (include/tqr.h; tqr_internal.h record layout) are replayed with the
adversarial event order of test_dist_protocol.PhasedSim while a happens-before relation is
built from the executor's counter semantics: a task that starts on `ctr >= v` acquires the
release of the task that published v (a counter advances by one, and each publisher of v has
acquired the publisher of v - 1 -- asserted), an early-releasing factor part (R24)
releases R_kk's rows mid-task, and a pipelined update task (R31) acquires block l's panel
counter before it reads block l.  Every task's footprint -- the rows x columns of each tile
and the packed-panel blocks it reads and writes, taken from tqr_exec.cu (panel_block,
update_phase, the split apply sub-tasks of the tall executor) -- is then checked: two
accesses to overlapping elements, at least one a write, must be ordered by happens-before.

This is the check that the per-block split of the tall executor's apply parts (R30)
first failed on the GPU: a GEQRT apply sub-task storing ALL rows of its block columns raced
with the TSQRT sub-applies of the first unit; `test_detects_full_row_geqrt_store` keeps that
variant as a negative case.
"""
from collections import defaultdict

import numpy as np
import pytest

from test_dist_protocol import K_G, K_L, K_S, K_T, NPT, PhasedSim, _deps, _global_j, _out_count


@pytest.fixture(scope="module")
def L():
    from paper_0707_3548_b200.build import build
    build()
    from paper_0707_3548_b200 import tqr
    return tqr


def inspected_geom(nsl, h):
    """Geometry of the inspected schedules (tqr_schedule_records_h): b = 64 nsl, s = 32 nsl,
    register passes of 64 columns."""
    return dict(b=64 * nsl, s=32 * nsl, sw=64, npt=NPT, h=h)


def footprint(rec, r, G, p, geom, full_row_geqrt_store=False):
    """(phase, key, write, r0, r1, c0, c1) of one record on rank r: element rows [r0, r1) x
    columns [c0, c1) of tile key ('A', i, j) (global tile coordinates), or the whole packed
    panel block key ('Y', rank copy, k, tile row, l).  Phase 0: from the start; phase 1: after
    the early release (factor parts: the packed Y_l / T_l stores) or, for a pipelined update
    task, after acquiring the panel counter of block l >= 1 (its reads of Y_l).
    geom: tile size b, panel block s, register-pass columns sw, blocks per tile npt, unit rows h."""
    b, s, sw, npt, h = geom["b"], geom["s"], geom["sw"], geom["npt"], geom["h"]
    kind, k, i = int(rec[0]), int(rec[1]), int(rec[2])
    fl, early = int(rec[14]) & 0xFF, (int(rec[14]) >> 8) > 0
    out = []
    if kind in (K_G, K_T):
        l, lp = int(rec[4]) & 0xFF, ((int(rec[4]) >> 8) & 0xFF) - 1
        cl = (l * s, (l + 1) * s)
        is_a, is_f = bool(fl & 2), bool(fl & 4)
        fused = not (is_a or is_f)
        ph_y = 1 if early else 0
        ys = [lp] if lp >= 0 else list(range(l))  # packed blocks an apply part reads
        if kind == K_G:
            if is_a:  # apply (sub-)part: U_lp is zero above row lp*s; stores only the rows it changes
                lo = 0 if (lp < 0 or full_row_geqrt_store) else lp * s
                out.append((0, ("A", k, k), True, lo, b, *cl))
            else:     # factor part: rows from the block's diagonal (fused: all rows, the apply too)
                out.append((0, ("A", k, k), True, l * s if is_f else 0, b, *cl))
                for g in range(G):
                    out.append((ph_y, ("Y", g, k, k, l), True, 0, 1, 0, 1))
        else:
            units = range(i, min(p, i + h))
            if is_a:  # R_kk rows of the applied blocks (TSQRT touches only R_kk's upper part)
                rows = (lp * s, (lp + 1) * s) if lp >= 0 else (0, l * s)
            else:
                rows = (l * s, (l + 1) * s) if is_f else (0, (l + 1) * s)
            out.append((0, ("A", k, k), True, *rows, *cl))
            for t in units:
                out.append((0, ("A", t, k), True, 0, b, *cl))
            if not is_a:
                for g in range(G):
                    out.append((ph_y, ("Y", g, k, i, l), True, 0, 1, 0, 1))
        if is_a or fused:
            for y in ys:
                out.append((0, ("Y", r, k, i, y), False, 0, 1, 0, 1))
    else:
        j = int(_global_j(rec, G, r))
        npass = max(1, int(rec[15]) & 0xFF)
        c = (int(rec[4]) * sw, (int(rec[4]) + npass) * sw)
        out.append((0, ("A", k, j), True, 0, b, *c))
        if kind == K_S:
            for t in range(i, min(p, i + h)):
                out.append((0, ("A", t, j), True, 0, b, *c))
        pipelined = bool(int(rec[14]) & 64)
        for y in range(npt):
            out.append((1 if (pipelined and y > 0) else 0, ("Y", r, k, k if kind == K_L else i, y), False, 0, 1, 0, 1))
    return out


class RaceSim(PhasedSim):
    """PhasedSim with happens-before sets (Python ints as bitsets over (task, phase) nodes)."""

    def __init__(self, per_rank, G, workers, seed=0, npt=NPT):
        super().__init__(per_rank, G, workers, ordered=True, seed=seed)
        self.npt = npt
        self.off = np.cumsum([0] + [len(r) for r, _ in per_rank])
        self.hb = {}                       # node -> bitset of nodes that happen before it
        self.pub = [dict() for _ in range(G)]  # (idx, val) -> (release set, publisher task)

    def _ready(self, r, rec, start=True):
        for d, (idx, cnt, val) in enumerate(_deps(rec)):
            if d == 0 and start and int(rec[14]) & 64:
                idx -= self.npt - 1
            if not np.all(self.ctr[r][idx:idx + cnt] >= val):
                return False
        return True

    def node(self, r, t, ph):
        return 2 * (int(self.off[r]) + t) + ph

    def _acq(self, r, idx, cnt, val):
        m = 0
        for x in range(cnt):
            if val >= 1:
                m |= self.pub[r][(idx + x, val)][0]
        return m

    def _release(self, r, idx, val, rel, task):
        if val > 1:  # the release chain: the publisher of val acquired the publisher of val - 1
            prev_set, prev_task = self.pub[r][(idx, val - 1)]
            assert prev_task == task or (rel >> self.node(*prev_task, 0)) & 1, \
                f"rank {r} counter {idx}: value {val} does not happen after value {val - 1}"
        self._publish(r, idx, val)
        self.pub[r][(idx, val)] = (rel, task)

    def run(self):
        G = self.G
        for _ in range(10 ** 7):
            for r in range(G):
                while len(self.held[r]) + len(self.running[r]) < self.workers and self.next[r] < len(self.recs[r]):
                    self.held[r].append(self.next[r])
                    self.next[r] += 1
            if all(self.done[r] == len(self.recs[r]) for r in range(G)):
                return
            ev = self._events()
            assert ev, "deadlock: no event can fire"
            best = min(e[0] for e in ev)
            cand = [e for e in ev if e[0] == best]
            _, r, what, t = cand[int(self.rng.integers(len(cand)))]
            rec = self.recs[r][t]
            n0, n1 = self.node(r, t, 0), self.node(r, t, 1)
            pipelined = bool(int(rec[14]) & 64)
            if what == "start":
                m = 0
                for d, (idx, cnt, val) in enumerate(_deps(rec)):
                    if d == 0 and pipelined:
                        idx -= self.npt - 1  # starts on block 0's panel counter
                    m |= self._acq(r, idx, cnt, val)
                self.hb[n0] = m
                self.held[r].remove(t)
                self.running[r].append([t, 0])
            elif what == "mid":
                pr = (int(rec[14]) >> 8) - 1
                self._release(r, pr, int(rec[6]), self.hb[n0] | (1 << n0), (r, t))
                next(x for x in self.running[r] if x[0] == t)[1] = 1
            else:
                m = self.hb[n0] | (1 << n0)
                if pipelined:  # block l's counter acquired before block l is read
                    idx, cnt, val = _deps(rec)[0]
                    for l_ in range(1, self.npt):
                        m |= self._acq(r, idx - (self.npt - 1) + l_, cnt, val)
                self.hb[n1] = m
                rel = m | (1 << n1)
                idx, val = int(rec[5]), int(rec[6])
                pr = (int(rec[14]) >> 8) - 1
                if pr >= 0 and val > 1:  # ordered publication: waits for PF >= v - 1 first
                    rel |= self._acq(r, idx, 1, val - 1)
                self.running[r] = [x for x in self.running[r] if x[0] != t]
                if rec[14] & 1:
                    for g in range(G):
                        self._release(g, idx, val, rel, (r, t))
                else:
                    for x in range(_out_count(rec)):
                        self._release(r, idx + x, val, rel, (r, t))
                self.done[r] += 1
        raise AssertionError("replay did not finish")


def races(per_rank, G, p, geom, workers, seed, **fpkw):
    sim = RaceSim(per_rank, G, workers, seed=seed, npt=geom["npt"])
    sim.run()
    acc = defaultdict(list)
    for r, (recs, _) in enumerate(per_rank):
        for t, rec in enumerate(recs):
            for ph, key, w, r0, r1, c0, c1 in footprint(rec, r, G, p, geom, **fpkw):
                acc[key].append((sim.node(r, t, ph), (r, t), w, r0, r1, c0, c1))
    bad = []
    for key, lst in acc.items():
        for a in range(len(lst)):
            na, ta, wa, ar0, ar1, ac0, ac1 = lst[a]
            for bidx in range(a + 1, len(lst)):
                nb, tb, wb, br0, br1, bc0, bc1 = lst[bidx]
                if ta == tb or not (wa or wb):
                    continue
                if ar0 >= br1 or br0 >= ar1 or ac0 >= bc1 or bc0 >= ac1:
                    continue
                if (sim.hb[nb] >> na) & 1 or (sim.hb[na] >> nb) & 1:
                    continue
                bad.append((key, ta, tb))
    return bad, sim


_CASES = [(6, 4, 1, 1, 3, 1), (8, 5, 2, 1, 5, 1), (9, 4, 2, 1, 4, 1), (7, 7, 2, 1, 6, 1), (10, 3, 1, 1, 3, 1),
          (8, 6, 2, 2, 3, 1), (9, 6, 1, 3, 2, 1),
          (9, 5, 2, 1, 5, 2), (10, 4, 2, 1, 6, 2), (12, 4, 1, 1, 4, 2), (11, 5, 2, 2, 4, 2), (10, 3, 1, 1, 3, 3)]


@pytest.mark.parametrize("p,q,nsl,G,workers,h", _CASES)
def test_no_unordered_conflicting_accesses(L, p, q, nsl, G, workers, h):
    per_rank = [L.schedule_records(p, q, nsl, workers, G, r, h=h) for r in range(G)]
    for seed in range(2):
        bad, sim = races(per_rank, G, p, inspected_geom(nsl, h), workers, seed)
        assert not bad, bad[:5]
        assert all(sim.done[r] == len(per_rank[r][0]) for r in range(G))


# Production schedules (the plan policy of tqr_plan_create): C2's b = 128 (fused panels,
# pipelined updates), b = 256 square (RW = 256, 128-column tasks) and tall-skinny (A/F split,
# RW = 128), b = 512 (SI = 16 < s), the tall-unit executor, multi-rank block-cyclic columns.
_PROD = [(1024, 1024, 128, 32, 1, 12, False), (1152, 896, 128, 32, 1, 9, False), (1536, 1536, 256, 32, 1, 16, False),
         (4096, 768, 256, 32, 1, 10, False), (2048, 1536, 512, 64, 1, 12, False), (3072, 768, 256, 32, 1, 10, True),
         (2560, 512, 256, 32, 1, 7, True), (1024, 1024, 128, 32, 2, 6, False), (1536, 1280, 256, 32, 3, 5, False),
         (4096, 512, 256, 32, 2, 6, False), (2048, 2048, 128, 32, 1, 40, False), (8192, 1024, 256, 32, 1, 30, True),
         (2048, 2048, 256, 32, 4, 8, False)]


@pytest.mark.parametrize("m,n,b,s,G,workers,tall,loc", [c + (False,) for c in _PROD] +
                         [(2048, 2048, 256, 32, 1, 16, False, True), (2048, 2048, 128, 32, 2, 12, False, True)])
def test_production_schedules_race_free(L, m, n, b, s, G, workers, tall, loc):
    per_rank, info = [], None
    for r in range(G):
        recs, nctr, info = L.schedule_records_policy(m, n, b, s, G, r, workers, tall=tall, locality=loc)
        per_rank.append((recs, nctr))
    npt, sw, nsl, h = info
    assert npt == b // s and sw * nsl >= b
    geom = dict(b=b, s=s, sw=sw, npt=npt, h=h)
    p = -(-m // b)
    for seed in range(2):
        bad, sim = races(per_rank, G, p, geom, workers, seed)
        assert not bad, bad[:5]
        assert all(sim.done[r] == len(per_rank[r][0]) for r in range(G))


def test_schedules_cover_every_task_form(L):
    """The cases above exercise split and fused panels, early release, pipelined updates,
    multi-pass update tasks, tall units and the split apply sub-tasks."""
    seen = set()
    for p, q, nsl, G, workers, h in _CASES:
        for r in range(G):
            recs, _ = L.schedule_records(p, q, nsl, workers, G, r, h=h)
            for rec in recs:
                f = int(rec[14])
                if rec[0] in (K_G, K_T):
                    seen.add("split" if f & 6 else "fused")
                    if f >> 8:
                        seen.add("early")
                    if (int(rec[4]) >> 8) & 0xFF:
                        seen.add("apply-sub")
                    if f & 128:
                        seen.add("unit2")
                else:
                    if f & 64:
                        seen.add("pipelined")
                    if (int(rec[15]) & 0xFF) > 1:
                        seen.add("multipass")
                    if f & 8:
                        seen.add("remote")
    assert seen >= {"split", "fused", "early", "apply-sub", "unit2", "pipelined", "multipass", "remote"}, seen


def test_detects_full_row_geqrt_store(L):
    """Negative check: the first split-apply kernel stored all rows of a GEQRT apply
    sub-task's block columns -- a write that races with the first unit's TSQRT sub-applies."""
    m, n, workers = 2560, 512, 7
    recs, nctr, (npt, sw, nsl, h) = L.schedule_records_policy(m, n, 256, 32, 1, 0, workers, tall=True)
    assert any((int(rec[4]) >> 8) & 0xFF for rec in recs)
    geom = dict(b=256, s=32, sw=sw, npt=npt, h=h)
    bad, _ = races([(recs, nctr)], 1, m // 256, geom, workers, 0)
    assert not bad
    bad, _ = races([(recs, nctr)], 1, m // 256, geom, workers, 0, full_row_geqrt_store=True)
    assert bad and all(key[0] == "A" and key[1] == key[2] for key, _, _ in bad)


def test_detects_a_dropped_dependency(L):
    """Negative check: removing the previous-unit dependency of one TSQRT apply sub-task
    (R_kk's rows of block lp: A(k,u-1,l,lp) before A(k,u,l,lp)) is reported as a race."""
    p, q, nsl, G, workers, h = 10, 4, 2, 1, 6, 2
    recs, nctr = L.schedule_records(p, q, nsl, workers, G, 0, h=h)
    recs = recs.copy()
    hit = False
    for rec in recs:
        if rec[0] == K_T and (int(rec[4]) >> 8) & 0xFF and int(rec[6]) > 2 and not hit:
            for d in range(3):
                code, val = int(rec[8 + 2 * d]), int(rec[9 + 2 * d])
                if (code >> 24) and val == int(rec[6]) - 1 and (code & 0xFFFFFF) == int(rec[5]):
                    rec[8 + 2 * d] = 0
                    rec[9 + 2 * d] = 0
                    hit = True
    assert hit
    found = False
    for seed in range(4):
        try:
            bad, _ = races([(recs, nctr)], G, p, inspected_geom(nsl, h), workers, seed)
        except AssertionError as e:  # the release chain of that counter breaks as well
            found = "does not happen after" in str(e) or "jumps" in str(e)
            break
        if bad:
            found = True
            break
    assert found
