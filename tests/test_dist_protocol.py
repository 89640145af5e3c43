"""Multi-GPU protocol on the CPU (no GPU needed): the per-rank dispatch records the library
builds for the 1D block-cyclic factorization (include/tqr.h, multi-GPU section)
are replayed with the executor's counter semantics -- ticket order per rank, waits on
`ctr[idx + x] >= val`, panel progress published to every rank -- once in-process and once
across two gloo processes (world_size 2) that exchange panel publications like peers over
NVLink.  Checks: ownership (columns j == r mod G), the union of all ranks' tasks is exactly
the single-GPU DAG, no deadlock with few workers, every published counter advances by one,
and each panel's V/T progress reaches every rank exactly once per value.
"""
import os
import socket

import numpy as np
import pytest

K_G, K_T, K_L, K_S = 0, 1, 2, 3
NPT = 2  # panel sub-tasks per tile in the inspected schedules (b / s = 64n / 32n; R21)


@pytest.fixture(scope="module")
def L():
    from paper_0707_3548_b200.build import build
    build()
    from paper_0707_3548_b200 import tqr
    return tqr


def _global_j(rec, G, r):
    """storage column -> global tile column (real multi-rank layout: jl -> r + jl*G)."""
    return rec[3] * G + r if G > 1 else rec[3]


def _task_keys(rec, G, r):
    """The DAG nodes a record covers: update tasks at register-pass granularity (a task covers
    passes [rec[4], rec[4] + np), np = rec[15] & 0xFF; the per-step task granularity is a
    scheduling policy that may differ between a 1-rank and a G-rank job)."""
    kind = int(rec[0])
    if kind in (K_L, K_S):
        j, npass = _global_j(rec, G, r), max(1, int(rec[15]) & 0xFF)
        return [(kind, int(rec[1]), int(rec[2]), int(j), int(rec[4]) + x) for x in range(npass)]
    return [(kind, int(rec[1]), int(rec[2]), int(rec[1]), int(rec[4]))]


def _out_count(rec):
    return max(1, (int(rec[15]) >> 8) & 0xFF)


def _deps(rec):
    out = []
    for d in range(3):
        code, val = int(rec[8 + 2 * d]), int(rec[9 + 2 * d])
        cnt, idx = (code >> 24) & 0xFF, code & 0xFFFFFF
        if cnt:
            out.append((idx, cnt, val))
    return out


class RankSim:
    """One rank's executor: `workers` CTAs taking tickets in order, a task runs when all its
    counter dependencies hold (it then completes at once and publishes)."""

    def __init__(self, recs, nctr, workers):
        self.recs, self.ctr, self.workers = recs, np.zeros(nctr, dtype=np.int64), workers
        self.next, self.held, self.done = 0, [], 0
        self.published = []  # (idx, val) of panel progress made by this rank (flags bit 0)

    def ready(self, rec):
        return all(np.all(self.ctr[idx:idx + cnt] >= val) for idx, cnt, val in _deps(rec))

    def publish(self, idx, val):
        assert val == self.ctr[idx] + 1, f"counter {idx} jumps {self.ctr[idx]} -> {val}"
        self.ctr[idx] = val

    def step(self):
        """Take tickets into free workers, run every held task that is ready.  Returns #run."""
        while len(self.held) < self.workers and self.next < len(self.recs):
            self.held.append(self.next)
            self.next += 1
        ran = 0
        for t in list(self.held):
            rec = self.recs[t]
            if self.ready(rec):
                self.held.remove(t)
                for x in range(_out_count(rec)):  # update tasks: one counter per register pass
                    self.publish(int(rec[5]) + x, int(rec[6]))
                pr = (int(rec[14]) >> 8) - 1  # panel factor parts: early-release counter (local)
                if pr >= 0:
                    self.publish(pr, int(rec[6]))
                if rec[14] & 1:
                    self.published.append((int(rec[5]), int(rec[6])))
                self.done += 1
                ran += 1
        return ran

    def finished(self):
        return self.done == len(self.recs)


@pytest.mark.parametrize("p,q,nsl,G,workers", [(6, 6, 1, 2, 1), (12, 9, 2, 3, 2), (9, 12, 2, 4, 3), (16, 5, 1, 8, 1),
                                               (20, 20, 2, 2, 4), (3, 2, 1, 8, 1), (30, 4, 2, 4, 2)])
def test_partition_and_replay(L, p, q, nsl, G, workers):
    single, _ = L.schedule_records(p, q, nsl, workers, 1, 0)
    ref = sorted(key for rec in single for key in _task_keys(rec, 1, 0))
    sims, keys = [], []
    for r in range(G):
        recs, nctr = L.schedule_records(p, q, nsl, workers, G, r)
        for rec in recs:
            kind = int(rec[0])
            k = int(rec[1])
            if kind in (K_G, K_T):
                assert k % G == r and rec[7] == k // G  # panel parts on owner(k)
                # factor parts (bit 2) and fused blocks publish their progress to every rank,
                # apply parts (bit 1) stay local
                assert rec[14] & 0xFF in (1, 2, 1 | 4)
            else:
                assert _global_j(rec, G, r) % G == r and not rec[14] & 1  # update on owner(j), local
                # dep 0 (the panel counter PF(k, last)) is acquired at system scope exactly when
                # a peer GPU publishes it; every other dependency is rank-local (gpu scope)
                assert bool(rec[14] & 8) == (k % G != r) and not rec[14] & 0x30 and not rec[14] & 0x80
                assert _deps(rec)[0][0] == k * 3 * NPT + NPT - 1
            keys.extend(_task_keys(rec, G, r))
        sims.append(RankSim(recs, nctr, workers))
    assert sorted(keys) == ref, "the ranks' tasks are not exactly the single-GPU DAG"
    # in-process replay; panel publications reach the other ranks' counter copies at once
    seen = [dict() for _ in range(G)]
    for _ in range(100000):
        progress = 0
        for r, sim in enumerate(sims):
            before = len(sim.published)
            progress += sim.step()
            for idx, val in sim.published[before:]:
                for g, other in enumerate(sims):
                    if g != r:
                        other.publish(idx, val)
                        seen[g][(idx, val)] = seen[g].get((idx, val), 0) + 1
        if all(s.finished() for s in sims):
            break
        assert progress, "deadlock: no rank can make progress"
    assert all(s.finished() for s in sims)
    K = min(p, q)
    for g, sim in enumerate(sims):
        # every rank ends with the complete panel progress of every step, received exactly once
        for k in range(K):
            for l in range(NPT):  # PF(k, l) at k*3*NPT + l
                assert sim.ctr[k * 3 * NPT + l] == max(1, p - k)
        assert all(v == 1 for v in seen[g].values())


class PhasedSim:
    """All ranks of a job in one process, with the executor's TWO publication events per
    early-releasing panel factor part (R24): the early release PR(k,l) mid-task and
    the end-of-task PF(k,l) (+ the publication to every rank).  Events are taken in an
    adversarial order: an early-released factor part finishes as LATE as possible (after
    every other runnable event), so the next tile's factor part of the same block, which
    starts on the early release, may reach its end first.  `ordered` models the executor's
    end-of-task rule (tqr_exec.cu: wait for PF >= v - 1 before releasing PF = v); without it
    PF(k,l) would jump.  Every publication asserts that the counter advances by exactly one,
    and every consumer that starts on PF >= v must find the task that published v finished."""

    def __init__(self, per_rank, G, workers, ordered=True, seed=0):
        self.G, self.workers, self.ordered = G, workers, ordered
        self.recs = [r for r, _ in per_rank]
        self.ctr = [np.zeros(n, dtype=np.int64) for _, n in per_rank]
        self.next = [0] * G
        self.held = [[] for _ in range(G)]      # tickets taken, not started
        self.running = [[] for _ in range(G)]   # [ticket, phase] (0: before PR, 1: after)
        self.done = [0] * G
        self.rng = np.random.default_rng(seed)

    def _publish(self, r, idx, val):
        assert val == self.ctr[r][idx] + 1, f"rank {r} counter {idx} jumps {self.ctr[r][idx]} -> {val}"
        self.ctr[r][idx] = val

    def _ready(self, r, rec, start=True):
        """start: a pipelined update task (record [14] bit 6, R31) starts on block 0's
        panel counter PF(k, 0) and can only FINISH once the last block's, PF(k, NPT-1), holds."""
        for d, (idx, cnt, val) in enumerate(_deps(rec)):
            if d == 0 and start and int(rec[14]) & 64:
                idx -= NPT - 1
            if not np.all(self.ctr[r][idx:idx + cnt] >= val):
                return False
        return True

    def _events(self):
        ev = []
        for r in range(self.G):
            for t in self.held[r]:
                if self._ready(r, self.recs[r][t]):
                    ev.append((1, r, "start", t))
            for t, ph in self.running[r]:
                rec = self.recs[r][t]
                pr = (int(rec[14]) >> 8) - 1
                if pr >= 0 and ph == 0:
                    ev.append((1, r, "mid", t))
                else:
                    can_end = self._ready(r, rec, start=False)  # pipelined: every panel block in
                    if self.ordered and pr >= 0 and int(rec[6]) > 1:
                        can_end = can_end and self.ctr[r][int(rec[5])] >= int(rec[6]) - 1
                    if can_end:   # early-released factor parts end last (adversarial)
                        ev.append((2 if pr >= 0 else 1, r, "end", t))
        return ev

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
            if what == "start":
                self.held[r].remove(t)
                self.running[r].append([t, 0])
            elif what == "mid":
                pr = (int(rec[14]) >> 8) - 1
                self._publish(r, pr, int(rec[6]))
                next(x for x in self.running[r] if x[0] == t)[1] = 1
            else:
                self.running[r] = [x for x in self.running[r] if x[0] != t]
                idx, val = int(rec[5]), int(rec[6])
                if rec[14] & 1:   # panel progress: every rank's copy
                    for g in range(G):
                        self._publish(g, idx, val)
                else:
                    for x in range(_out_count(rec)):
                        self._publish(r, idx + x, val)
                self.done[r] += 1
        raise AssertionError("replay did not finish")


_PHASED = [(8, 7, 1, 1, 4), (12, 7, 2, 1, 8), (30, 4, 2, 1, 16), (14, 6, 2, 1, 6), (10, 9, 2, 3, 3), (24, 4, 1, 4, 6),
           (10, 8, 2, 3, 3), (20, 7, 1, 2, 5)]


@pytest.mark.parametrize("p,q,nsl,G,workers", _PHASED)
def test_phased_adversarial_replay(L, p, q, nsl, G, workers):
    """The early release (PR mid-task) lets F(k,i+1,l) overtake F(k,i,l); with the executor's
    ordered end-of-task publication every PF(k,l) still advances by one on every rank, and
    the replay finishes (no deadlock from the extra wait)."""
    per_rank = [L.schedule_records(p, q, nsl, workers, G, r) for r in range(G)]
    if not any((int(rec[14]) >> 8) for recs, _ in per_rank for rec in recs):
        pytest.skip("schedule without early release")
    pipelined = sum(1 for recs, _ in per_rank for rec in recs if int(rec[14]) & 64)
    for seed in range(3):
        sim = PhasedSim(per_rank, G, workers, ordered=True, seed=seed)
        sim.run()
        for r in range(G):
            assert sim.done[r] == len(per_rank[r][0])
            for k in range(min(p, q)):
                for l_ in range(NPT):
                    assert sim.ctr[r][k * 3 * NPT + l_] == max(1, p - k)


@pytest.mark.parametrize("p,q,nsl,G,workers,h", [(9, 4, 2, 1, 5, 2), (12, 5, 1, 1, 7, 2), (11, 6, 2, 2, 4, 2),
                                                 (10, 3, 1, 1, 3, 3), (10, 4, 2, 1, 6, 2), (12, 6, 2, 2, 4, 2),
                                                 (13, 5, 1, 1, 3, 2)])
def test_phased_replay_tall_units(L, p, q, nsl, G, workers, h):
    """Units of h tile rows (TQR_FLAG_TALL_TILES, R30): the same adversarial replay;
    every step's panel chain ends at 1 + (number of units), and the ranks' tasks are exactly
    the single-rank unit DAG."""
    per_rank = [L.schedule_records(p, q, nsl, workers, G, r, h=h) for r in range(G)]
    single, _ = L.schedule_records(p, q, nsl, workers, 1, 0, h=h)
    ref = sorted(key for rec in single for key in _task_keys(rec, 1, 0))
    keys = sorted(key for r, (recs, _) in enumerate(per_rank) for rec in recs for key in _task_keys(rec, G, r))
    assert keys == ref
    assert any(int(rec[14]) & 128 for rec in single)  # two-tile units present
    for seed in range(2):
        sim = PhasedSim(per_rank, G, workers, ordered=True, seed=seed)
        sim.run()
        for r in range(G):
            for k in range(min(p, q)):
                for l_ in range(NPT):
                    assert sim.ctr[r][k * 3 * NPT + l_] == 1 + -(-(p - k - 1) // h)


def test_phased_replay_detects_unordered_publication(L):
    """Negative check: without the ordered publication, the adversarial order makes PF(k,l)
    jump (a consumer of PF >= v would read tile i's Y_l / T_l before they are stored)."""
    per_rank = [L.schedule_records(30, 4, 2, 16, 1, 0)]
    assert any((int(rec[14]) >> 8) for rec in per_rank[0][0])
    with pytest.raises(AssertionError, match="jumps"):
        for seed in range(5):
            PhasedSim(per_rank, 1, 16, ordered=False, seed=seed).run()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_rank(rank, world, port, p, q, nsl, workers, out):
    import torch.distributed as dist
    from paper_0707_3548_b200 import tqr
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        recs, nctr = tqr.schedule_records(p, q, nsl, workers, world, rank)
        sim = RankSim(recs, nctr, workers)
        rounds = 0
        while True:
            before = len(sim.published)
            ran = 0
            while True:
                x = sim.step()
                if not x:
                    break
                ran += x
            mine = sim.published[before:]
            allp = [None] * world
            dist.all_gather_object(allp, (mine, sim.finished(), ran))
            for g, (pubs, _, _) in enumerate(allp):
                if g != rank:
                    for idx, val in pubs:
                        sim.publish(idx, val)
            if all(f for _, f, _ in allp):
                break
            rounds += 1
            # nobody ran a task this round and some rank is unfinished: cross-rank deadlock
            assert rounds < 100000 and any(r for _, _, r in allp), "deadlock across ranks"
        out.put((rank, sim.done, len(recs), [int(sim.ctr[k * 3 * NPT + l]) for k in range(min(p, q))
                                             for l in range(NPT)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p,q,nsl,workers", [(10, 7, 2, 2), (24, 4, 1, 1)])
def test_gloo_two_ranks_replay(L, p, q, nsl, workers):
    """world_size 2 over gloo: each process replays its own rank's stream and receives the
    peer's panel publications through torch.distributed, as it would over NVLink."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_rank, args=(r, 2, port, p, q, nsl, workers, q_out)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q_out.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    K = min(p, q)
    for rank, done, n, ctr in res:
        assert done == n
        assert ctr == [max(1, p - k) for k in range(K) for _ in range(NPT)]


def test_exchange_blobs_gloo():
    """The one-time IPC blob all-gather of dist.connect, over gloo with 2 processes."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_blob_rank, args=(r, 2, port, q_out)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q_out.get(timeout=240) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    want = bytes([0]) * 256 + bytes([1]) * 256
    assert res[0] == want and res[1] == want


def _blob_rank(rank, world, port, out):
    import torch.distributed as dist
    from paper_0707_3548_b200 import dist as tdist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        out.put((rank, tdist.exchange_blobs(bytes([rank]) * 256)))
    finally:
        dist.destroy_process_group()


def test_owned_columns():
    from paper_0707_3548_b200 import dist as tdist
    cols = [tdist.owned_columns(10, 3, r) for r in range(3)]
    assert cols == [[0, 3, 6, 9], [1, 4, 7], [2, 5, 8]]
    assert sorted(sum(cols, [])) == list(range(10))
