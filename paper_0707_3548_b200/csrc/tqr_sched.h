// tqr_sched.h -- the host-side DAG list scheduler shared by the tiled-QR (tqr_host.cpp) and
// tiled-LU (tlu_host.cpp) runtimes: tasks with "progress counter >= value" dependencies, turned
// into a topological dispatch (ticket) order by a list schedule on the executor's CTAs.
// Internal (not part of the public ABI); included by exactly those two translation units.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <queue>
#include <unordered_map>
#include <vector>

#include "tqr_internal.h"

namespace tqr {
namespace sched {

struct Sched {
  std::vector<std::vector<int>> rec;  // per rank: TASK_INTS per task, dispatch order
  std::vector<int> nctr;              // per rank: counters used
  int ntasks = 0;
  int64_t nedges = 0;
  int64_t counts[4] = {0, 0, 0, 0};
  bool topo_ok = true;
  double makespan = 0.0;  // modelled (list-schedule simulation), ns
  double busy = 0.0;      // modelled worker utilisation (sum of durations / (makespan x workers))
};

// ---- generic task list with counter deps -> list-schedule order --------------------------
struct TaskGen {
  struct T {
    int kind, k, i, j, sl;
    int rank, kc, flags;  // executing rank, storage column of tile column k, TASK flags
    int out_idx, out_val;
    int dep_idx[TASK_NDEP], dep_cnt[TASK_NDEP], dep_val[TASK_NDEP];
    int ndep;
    double dur;
    int cls;
    int key[4];  // priority keys after cls (smaller first); default (k, i, j, sl)
    int64_t group;  // PRIO_BLEVEL: tasks of one group share the group's highest bottom level (-1: none)
    int np, ocnt;   // update tasks: register passes; consecutive out counters published (>= 1)
    int out2_idx;   // panel factor parts: early-release counter (set to out_val mid-task), or -1
  };
  std::vector<T> t;
  int add(int kind, int k, int i, int j, int sl, int out_idx, int out_val, double dur, int cls) {
    T x{};
    x.kind = kind; x.k = k; x.i = i; x.j = j; x.sl = sl;
    x.rank = 0; x.kc = k; x.flags = 0;
    x.out_idx = out_idx; x.out_val = out_val; x.ndep = 0; x.dur = dur; x.cls = cls;
    x.key[0] = k; x.key[1] = i; x.key[2] = j; x.key[3] = sl;
    x.group = -1;
    x.np = 1; x.ocnt = 1; x.out2_idx = -1;
    t.push_back(x);
    return (int)t.size() - 1;
  }
  bool overflow = false;  // a task with more than TASK_NDEP dependencies (schedule bug)
  void dep(int id, int idx, int cnt, int val) {
    T& x = t[id];
    if (x.ndep >= TASK_NDEP) { overflow = true; return; }
    x.dep_idx[x.ndep] = idx; x.dep_cnt[x.ndep] = cnt; x.dep_val[x.ndep] = val; x.ndep++;
  }
};

static inline uint64_t ckey(int idx, int val) { return ((uint64_t)(uint32_t)idx << 32) | (uint32_t)val; }

// Builds successor lists from counter deps (each (rank, counter, value) has exactly one
// producer; panel counters published to every rank resolve to their producer on any rank),
// then list-schedules the whole job on `workers[r]` identical workers per rank.  Each rank's
// dispatch order is the restriction of ONE global topological order, so per-rank ticket
// streams cannot deadlock across ranks.  Returns false if the dependency
// structure is inconsistent (missing producer or cycle).
// Priority of the list schedule (never affects results, only the ticket order):
//  * PRIO_CLASS: the paper's classes G > T > L > S with the lookahead of
//    DESIGN.md R10, ties by (k, i, j, slice);
//  * PRIO_BLEVEL: critical-path priority -- the task's bottom level (its duration plus the
//    longest duration-weighted path to the end of the DAG, `lat` ns per edge for the counter
//    handoff), ties as above.  The paper motivates its classes by the critical path
//    ("nodes that have the higher number of outgoing edges"); the bottom
//    level is that criterion computed exactly on the task graph.  It matters when many panel
//    chains are in flight at once (tall-skinny grids, R22): the updates of column
//    j at step k < j - 1 feed panel j's chain and outrank later-column work of earlier steps.
enum Prio { PRIO_CLASS = 0, PRIO_BLEVEL = 1 };

// lat_remote (ns): extra modelled delay of an edge whose producer runs on another rank (the
// NVLink peer store + system-scope release / acquire); used by the scaling model.
static inline bool list_schedule(TaskGen& G, const std::vector<int>& workers, Sched& out, int prio = PRIO_CLASS,
                          double lat = 0.0, double blq = 0.0, double lat_remote = 0.0, int gmode = 1) {
  const int n = (int)G.t.size();
  const int nr = (int)workers.size();
  if (G.overflow) return false;
  std::unordered_map<uint64_t, int> producer;
  producer.reserve(n * 2);
  auto pkey = [](int rank, int idx, int val) { return ((uint64_t)(uint32_t)rank << 56) ^ ckey(idx, val); };
  for (int id = 0; id < n; ++id) {
    const auto& x = G.t[id];
    if (x.flags & 1)
      for (int r = 0; r < nr; ++r) producer[pkey(r, x.out_idx, x.out_val)] = id;
    else
      for (int c = 0; c < x.ocnt; ++c) producer[pkey(x.rank, x.out_idx + c, x.out_val)] = id;
    if (x.out2_idx >= 0) producer[pkey(x.rank, x.out2_idx, x.out_val)] = id;
  }
  std::vector<int> indeg(n, 0);
  std::vector<std::vector<int>> succ(n);
  int64_t nedges = 0;
  for (int id = 0; id < n; ++id) {
    const auto& x = G.t[id];
    for (int d = 0; d < x.ndep; ++d)
      for (int c = 0; c < x.dep_cnt[d]; ++c) {
        auto it = producer.find(pkey(x.rank, x.dep_idx[d] + c, x.dep_val[d]));
        if (it == producer.end()) return false;
        succ[it->second].push_back(id);
        indeg[id]++;
        nedges++;
      }
  }
  std::vector<double> blevel;
  if (prio == PRIO_BLEVEL) {  // reverse topological DP (Kahn order)
    std::vector<int> topo, deg(indeg);
    topo.reserve(n);
    for (int id = 0; id < n; ++id)
      if (deg[id] == 0) topo.push_back(id);
    for (size_t h = 0; h < topo.size(); ++h)
      for (int sidx : succ[topo[h]])
        if (--deg[sidx] == 0) topo.push_back(sidx);
    if ((int)topo.size() != n) return false;  // cycle
    blevel.assign(n, 0.0);
    for (int h = n - 1; h >= 0; --h) {
      const int id = topo[h];
      double m = 0.0;
      for (int sidx : succ[id]) m = std::max(m, blevel[sidx] + lat);
      blevel[id] = G.t[id].dur + m;
    }
    // grouped tasks (the updates that read one reflector panel, R22) take one common
    // bottom level -- the group's highest (gmode 1, 3) or its median (gmode 2) -- so they are
    // dispatched together and share the panel in L2
    std::unordered_map<int64_t, std::vector<double>> gval;
    for (int id = 0; id < n; ++id)
      if (G.t[id].group >= 0) gval[G.t[id].group].push_back(blevel[id]);
    std::unordered_map<int64_t, double> gsel;
    for (auto& kv : gval) {
      auto& v = kv.second;
      if (gmode == 2) {
        std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
        gsel[kv.first] = v[v.size() / 2];
      } else {
        gsel[kv.first] = *std::max_element(v.begin(), v.end());
      }
    }
    for (int id = 0; id < n; ++id)
      if (G.t[id].group >= 0) blevel[id] = gsel[G.t[id].group];
    // quantised (blq > 0): tasks within one quantum keep the (k, i, j, slice) order, so the
    // updates sharing one reflector panel (k, i) run together and reuse it from L2
    if (blq > 0.0)
      for (double& x : blevel) x = std::floor(x / blq);
  }
  auto prio_less = [&](int a, int b) {  // true if a has LOWER priority than b (for max-heap)
    const auto &x = G.t[a], &y = G.t[b];
    if (prio == PRIO_BLEVEL) {
      if (blevel[a] != blevel[b]) return blevel[a] < blevel[b];
    } else if (x.cls != y.cls) {
      return x.cls > y.cls;
    }
    for (int c = 0; c < 4; ++c)
      if (x.key[c] != y.key[c]) return x.key[c] > y.key[c];
    return a > b;
  };
  using PQ = std::priority_queue<int, std::vector<int>, decltype(prio_less)>;
  std::vector<PQ> ready;
  for (int r = 0; r < nr; ++r) ready.emplace_back(prio_less);
  using Ev = std::pair<double, int>;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> events;
  for (int id = 0; id < n; ++id)
    if (indeg[id] == 0) ready[G.t[id].rank].push(id);
  std::vector<int> order;
  order.reserve(n);
  std::vector<double> sim_start(n, 0.0);  // development aid: TQR_DEV_SIMDUMP=<file>
  std::vector<int> free_w(nr);
  for (int r = 0; r < nr; ++r) free_w[r] = std::max(1, workers[r]);
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> arrivals;  // remote edges in flight
  double now = 0.0, work = 0.0;
  int done = 0;
  while (done < n) {
    for (int r = 0; r < nr; ++r)
      while (free_w[r] > 0 && !ready[r].empty()) {
        int id = ready[r].top();
        ready[r].pop();
        order.push_back(id);
        sim_start[id] = now;
        events.push({now + G.t[id].dur + lat, id});
        work += G.t[id].dur;
        free_w[r]--;
      }
    if (events.empty() && arrivals.empty()) return false;  // cycle
    if (!arrivals.empty() && (events.empty() || arrivals.top().first <= events.top().first)) {
      const Ev a = arrivals.top();
      arrivals.pop();
      now = a.first;
      if (--indeg[a.second] == 0) ready[G.t[a.second].rank].push(a.second);
      continue;
    }
    Ev e = events.top();
    events.pop();
    now = e.first;
    done++;
    free_w[G.t[e.second].rank]++;
    for (int sidx : succ[e.second]) {
      if (lat_remote > 0.0 && G.t[sidx].rank != G.t[e.second].rank)
        arrivals.push({now + lat_remote, sidx});
      else if (--indeg[sidx] == 0)
        ready[G.t[sidx].rank].push(sidx);
    }
  }
  {
    int64_t wt = 0;
    for (int x : workers) wt += std::max(1, x);
    out.makespan = now;
    out.busy = now > 0.0 ? work / (now * (double)wt) : 0.0;
  }
  if (const char* f = getenv("TQR_DEV_SIMDUMP")) {  // modelled start/end per task (ns), dispatch order
    if (FILE* fp = fopen(f, "w")) {
      for (int id : order) {
        const auto& x = G.t[id];
        fprintf(fp, "%d %d %d %d %d %.0f %.0f\n", x.kind, x.k, x.i, x.j, x.sl, sim_start[id], sim_start[id] + x.dur);
      }
      fclose(fp);
    }
  }
  // emit per-rank records; verify the global order is topological
  std::vector<int> pos(n);
  for (int r = 0; r < n; ++r) pos[order[r]] = r;
  out.rec.assign(nr, {});
  out.topo_ok = true;
  for (int r = 0; r < n; ++r) {
    const auto& x = G.t[order[r]];
    auto& v = out.rec[x.rank];
    const size_t o = v.size();
    v.resize(o + TASK_INTS, 0);
    int* q = &v[o];
    q[0] = x.kind; q[1] = x.k; q[2] = x.i; q[3] = x.j; q[4] = x.sl; q[5] = x.out_idx; q[6] = x.out_val;
    q[7] = x.kc;
    for (int d = 0; d < x.ndep; ++d) {
      q[8 + 2 * d] = x.dep_idx[d] | (x.dep_cnt[d] << 24);
      q[9 + 2 * d] = x.dep_val[d];
    }
    q[14] = x.flags;
    q[15] = x.np | (x.ocnt << 8);
  }
  for (int id = 0; id < n; ++id)
    for (int sidx : succ[id])
      if (pos[id] >= pos[sidx]) out.topo_ok = false;
  out.ntasks = n;
  out.nedges = nedges;
  return true;
}

}  // namespace sched
}  // namespace tqr
