// tqr_host.cpp -- host runtime of the tiled QR library: plan, DAG task tables, list-schedule
// dispatch order, and the C ABI declared in include/tqr.h.
//
// DAG (edges derived from each kernel's read/write sets, SPEC dag module):
//   G(k)        <- S(k-1,k,k,*)
//   L(k,j,sl)   <- G(k), S(k-1,k,j,sl)
//   T(k,i)      <- G(k) | T(k,i-1), S(k-1,i,k,*)
//   S(k,i,j,sl) <- T(k,i), L(k,j,sl) | S(k,i-1,j,sl), S(k-1,i,j,sl)
// Every dependency is a chain, so it is expressed on the device as "progress counter >=
// value": panel[k] counts G(k), T(k,k+1), ... ; col[k][j][sl] counts L(k,j,sl), S(k,k+1,j,sl), ...
// The dispatch (ticket) order is a list schedule of the DAG on `workers` CTAs with the
// paper's priorities G > T > L > S, ties by (k, i, j, slice); it is
// topological by construction, so with all CTAs co-resident no ticket can wait forever.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tqr.h"
#include "tqr_internal.h"

using namespace tqr;

namespace {

thread_local std::string g_err;
thread_local int32_t g_badarg = 0;

tqr_status bad_arg(int idx, const char* what) {
  g_badarg = idx;
  g_err = what;
  return TQR_ERR_INVALID_ARG;
}
tqr_status cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return TQR_ERR_CUDA;
}
#define CU(call)                                            \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);     \
  } while (0)

struct Sched {
  std::vector<int> rec;  // TASK_INTS per task, dispatch order
  int ntasks = 0;
  int nctr = 0;
  int64_t nedges = 0;
  int64_t counts[4] = {0, 0, 0, 0};
  bool topo_ok = true;
};

// ---- generic task list with counter deps -> list-schedule order --------------------------
struct TaskGen {
  struct T {
    int kind, k, i, j, sl;
    int out_idx, out_val;
    int dep_idx[TASK_NDEP], dep_cnt[TASK_NDEP], dep_val[TASK_NDEP];
    int ndep;
    double dur;
    int cls;
    int key[4];  // priority keys after cls (smaller first); default (k, i, j, sl)
  };
  std::vector<T> t;
  int add(int kind, int k, int i, int j, int sl, int out_idx, int out_val, double dur, int cls) {
    T x{};
    x.kind = kind; x.k = k; x.i = i; x.j = j; x.sl = sl;
    x.out_idx = out_idx; x.out_val = out_val; x.ndep = 0; x.dur = dur; x.cls = cls;
    x.key[0] = k; x.key[1] = i; x.key[2] = j; x.key[3] = sl;
    t.push_back(x);
    return (int)t.size() - 1;
  }
  void dep(int id, int idx, int cnt, int val) {
    T& x = t[id];
    x.dep_idx[x.ndep] = idx; x.dep_cnt[x.ndep] = cnt; x.dep_val[x.ndep] = val; x.ndep++;
  }
};

static inline uint64_t ckey(int idx, int val) { return ((uint64_t)(uint32_t)idx << 32) | (uint32_t)val; }

// Builds successor lists from counter deps (each (counter, value) has exactly one producer),
// then list-schedules on `workers` identical workers.  Returns false if the dependency
// structure is inconsistent (missing producer or cycle).
static bool list_schedule(TaskGen& G, int workers, int nctr, Sched& out) {
  const int n = (int)G.t.size();
  std::unordered_map<uint64_t, int> producer;
  producer.reserve(n * 2);
  for (int id = 0; id < n; ++id) producer[ckey(G.t[id].out_idx, G.t[id].out_val)] = id;
  std::vector<int> indeg(n, 0);
  std::vector<std::vector<int>> succ(n);
  int64_t nedges = 0;
  for (int id = 0; id < n; ++id) {
    const auto& x = G.t[id];
    for (int d = 0; d < x.ndep; ++d)
      for (int c = 0; c < x.dep_cnt[d]; ++c) {
        auto it = producer.find(ckey(x.dep_idx[d] + c, x.dep_val[d]));
        if (it == producer.end()) return false;
        succ[it->second].push_back(id);
        indeg[id]++;
        nedges++;
      }
  }
  auto prio_less = [&](int a, int b) {  // true if a has LOWER priority than b (for max-heap)
    const auto &x = G.t[a], &y = G.t[b];
    if (x.cls != y.cls) return x.cls > y.cls;
    for (int c = 0; c < 4; ++c)
      if (x.key[c] != y.key[c]) return x.key[c] > y.key[c];
    return a > b;
  };
  std::priority_queue<int, std::vector<int>, decltype(prio_less)> ready(prio_less);
  using Ev = std::pair<double, int>;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> events;
  for (int id = 0; id < n; ++id)
    if (indeg[id] == 0) ready.push(id);
  std::vector<int> order;
  order.reserve(n);
  int free_w = std::max(1, workers);
  double now = 0.0;
  int done = 0;
  while (done < n) {
    while (free_w > 0 && !ready.empty()) {
      int id = ready.top();
      ready.pop();
      order.push_back(id);
      events.push({now + G.t[id].dur, id});
      free_w--;
    }
    if (events.empty()) return false;  // cycle
    Ev e = events.top();
    events.pop();
    now = e.first;
    done++;
    free_w++;
    for (int s : succ[e.second])
      if (--indeg[s] == 0) ready.push(s);
  }
  // emit records; verify topological order against the counter semantics
  std::vector<int> pos(n);
  for (int r = 0; r < n; ++r) pos[order[r]] = r;
  out.rec.assign((size_t)n * TASK_INTS, 0);
  out.topo_ok = true;
  for (int r = 0; r < n; ++r) {
    const auto& x = G.t[order[r]];
    int* q = &out.rec[(size_t)r * TASK_INTS];
    q[0] = x.kind; q[1] = x.k; q[2] = x.i; q[3] = x.j; q[4] = x.sl; q[5] = x.out_idx; q[6] = x.out_val;
    for (int d = 0; d < x.ndep; ++d) {
      q[8 + 2 * d] = x.dep_idx[d] | (x.dep_cnt[d] << 24);
      q[9 + 2 * d] = x.dep_val[d];
    }
  }
  for (int id = 0; id < n; ++id)
    for (int s : succ[id])
      if (pos[id] >= pos[s]) out.topo_ok = false;
  out.ntasks = n;
  out.nctr = nctr;
  out.nedges = nedges;
  return true;
}

// Rough per-task durations (ns) for the list schedule only (never affect results):
// fp64 DMMA peak per SM ~251 GFLOP/s (M0 probe), efficiencies per kind as measured by
// tools/prof_tasks.py (r01: GEQRT ~9%, TSQRT ~14%, LARFB ~34%, SSRFB ~60% of the SM peak).
struct DurModel {
  double g, t, l, s;
  DurModel(int b, int s_, int w) {
    const double B = b, Sv = s_, W = w, sm = 251.0;  // GFLOP/s per SM == flop/ns
    g = 3000 + (4.0 / 3 * B * B * B + 2.0 / 3 * Sv * B * B) / (0.09 * sm);
    t = 3000 + (2.0 * B * B * B + 4.0 / 3 * Sv * B * B) / (0.14 * sm);
    l = 1500 + (2.0 * B * B * W + Sv * B * W) / (0.34 * sm);
    s = 1500 + (4.0 * B * B * W + Sv * B * W) / (0.6 * sm);
  }
};

static void build_factor_sched(int64_t p, int64_t q, int b, int s, int nsl, int workers, Sched& out) {
  const int K = (int)std::min(p, q);
  const int w = (b + nsl - 1) / nsl;
  DurModel dm(b, s, w);
  TaskGen G;
  auto PANEL = [&](int k) { return k; };
  auto COL = [&](int k, int j, int sl) { return K + (int)(((int64_t)k * q + j) * nsl + sl); };
  const int nctr = K + (int)((int64_t)K * q * nsl);
  for (int k = 0; k < K; ++k) {
    int id = G.add(K_G, k, k, k, 0, PANEL(k), 1, dm.g, 0);
    if (k > 0) G.dep(id, COL(k - 1, k, 0), nsl, 2);
    out.counts[0]++;
    for (int j = k + 1; j < q; ++j)
      for (int sl = 0; sl < nsl; ++sl) {
        // lookahead (R10): updates of column k+1 feed panel k+1 -> critical path
        id = G.add(K_L, k, k, j, sl, COL(k, j, sl), 1, dm.l, j == k + 1 ? 1 : 2);
        G.dep(id, PANEL(k), 1, 1);
        if (k > 0) G.dep(id, COL(k - 1, j, sl), 1, 2);
        out.counts[2]++;
      }
    for (int i = k + 1; i < p; ++i) {
      id = G.add(K_T, k, i, k, 0, PANEL(k), i - k + 1, dm.t, 1);
      G.dep(id, PANEL(k), 1, i - k);
      if (k > 0) G.dep(id, COL(k - 1, k, 0), nsl, i - k + 2);
      out.counts[1]++;
      for (int j = k + 1; j < q; ++j)
        for (int sl = 0; sl < nsl; ++sl) {
          id = G.add(K_S, k, i, j, sl, COL(k, j, sl), i - k + 1, dm.s, j == k + 1 ? 1 : 3);
          G.dep(id, PANEL(k), 1, i - k + 1);
          G.dep(id, COL(k, j, sl), 1, i - k);
          if (k > 0) G.dep(id, COL(k - 1, j, sl), 1, i - k + 2);
          out.counts[3]++;
        }
    }
  }
  if (!list_schedule(G, workers, nctr, out)) out.topo_ok = false;
}

// apply-Q^T (trans) or apply-Q to a tile-major B with qb tile columns.
//   Q^T: step k ascending: L(k,jb,sl), then S(k,i,jb,sl) for i ascending (chain on B(k,jb)).
//        cnt[k][jb][sl]: L -> 1, S(k,i) -> i-k+1.
//   Q  : step k descending: S(k,i,jb,sl) for i descending, then L(k,jb,sl).
//        cnt[k][jb][sl]: S(k,i) -> p-i, L -> p-k.
static void build_orm_sched(int64_t p, int64_t q, int64_t qb, int b, int s, int nsl, bool trans, int workers,
                            Sched& out) {
  const int K = (int)std::min(p, q);
  const int w = (b + nsl - 1) / nsl;
  DurModel dm(b, s, w);
  TaskGen G;
  auto CNT = [&](int k, int jb, int sl) { return (int)(((int64_t)k * qb + jb) * nsl + sl); };
  const int nctr = (int)((int64_t)K * qb * nsl);
  for (int jb = 0; jb < qb; ++jb)
    for (int sl = 0; sl < nsl; ++sl) {
      if (trans) {
        for (int k = 0; k < K; ++k) {
          int id = G.add(K_LQT, k, k, jb, sl, CNT(k, jb, sl), 1, dm.l, 0);
          if (k > 0) G.dep(id, CNT(k - 1, jb, sl), 1, 2);
          for (int i = k + 1; i < p; ++i) {
            id = G.add(K_SQT, k, i, jb, sl, CNT(k, jb, sl), i - k + 1, dm.s, 1);
            G.dep(id, CNT(k, jb, sl), 1, i - k);
            if (k > 0) G.dep(id, CNT(k - 1, jb, sl), 1, i - k + 2);
          }
        }
      } else {
        for (int k = K - 1; k >= 0; --k) {
          for (int i = (int)p - 1; i > k; --i) {
            int id = G.add(K_SQ, k, i, jb, sl, CNT(k, jb, sl), (int)p - i, dm.s, 1);
            G.t[id].key[0] = K - 1 - k;  // reverse order: later steps first
            G.t[id].key[1] = (int)p - 1 - i;
            if (i < p - 1) G.dep(id, CNT(k, jb, sl), 1, (int)p - i - 1);
            if (k + 1 < K) G.dep(id, CNT(k + 1, jb, sl), 1, (int)p - i);
          }
          int id = G.add(K_LQ, k, k, jb, sl, CNT(k, jb, sl), (int)p - k, dm.l, 0);
          G.t[id].key[0] = K - 1 - k;
          if (k + 1 < p) G.dep(id, CNT(k, jb, sl), 1, (int)p - k - 1);
        }
      }
    }
  if (!list_schedule(G, workers, nctr, out)) out.topo_ok = false;
}

struct DevSched {
  int* d_tasks = nullptr;
  int ntasks = 0;
  int nctr = 0;
  int mode = 0;  // executor instance: 0 factorization, 1 apply Q^T, 2 apply Q
};

}  // namespace

struct tqr_plan {
  tqr_params prm;
  int64_t p, q, K;
  int nsl, workers;
  cudaStream_t st;
  DevSched fact;
  std::map<std::pair<int, int64_t>, DevSched> orm;
  int* d_ctr = nullptr;   // sized for the largest schedule so far
  int nctr_cap = 0;
  int* d_ticket = nullptr;
  unsigned long long* d_trace = nullptr;
  long long* d_phases = nullptr;  // set by tqr_phase_counters (profiling builds)
  int trace_cap = 0;
  int trace_n = 0;
};

static tqr_status upload(tqr_plan* P, const Sched& s, DevSched& d) {
  CU(cudaMalloc(&d.d_tasks, s.rec.size() * sizeof(int) + 16));
  CU(cudaMemcpy(d.d_tasks, s.rec.data(), s.rec.size() * sizeof(int), cudaMemcpyHostToDevice));
  d.ntasks = s.ntasks;
  d.nctr = s.nctr;  // (mode is set by the caller)
  if (s.nctr > P->nctr_cap) {
    if (P->d_ctr) cudaFree(P->d_ctr);
    CU(cudaMalloc(&P->d_ctr, sizeof(int) * (size_t)std::max(1, s.nctr)));
    P->nctr_cap = s.nctr;
  }
  return TQR_OK;
}

static tqr_status run(tqr_plan* P, const DevSched& d, double* A, double* T, double* Bt, void* work, bool trace) {
  if (d.ntasks == 0) return TQR_OK;
  CU(cudaMemsetAsync(P->d_ctr, 0, sizeof(int) * (size_t)std::max(1, d.nctr), P->st));
  CU(cudaMemsetAsync(P->d_ticket, 0, sizeof(int), P->st));
  ExecArgs a;
  a.A = A; a.T = T; a.Bt = Bt;
  a.Yp = reinterpret_cast<double*>(work);
  a.Tp = a.Yp + (size_t)P->p * P->q * P->prm.b * P->prm.b;
  a.tasks = d.d_tasks;
  a.ntasks = d.ntasks;
  a.p = (int)P->p;
  a.ticket = P->d_ticket;
  a.ctr = P->d_ctr;
  a.trace = nullptr;
  a.phases = P->d_phases;
  if (trace) {
    if (P->trace_cap < d.ntasks) {
      if (P->d_trace) cudaFree(P->d_trace);
      CU(cudaMalloc(&P->d_trace, sizeof(unsigned long long) * 4 * (size_t)d.ntasks));
      P->trace_cap = d.ntasks;
    }
    a.trace = P->d_trace;
    P->trace_n = d.ntasks;
  }
  const int grid = std::min(P->workers, std::max(1, d.ntasks));
  CU(launch_exec(P->prm.b, P->prm.s, d.mode, a, grid, P->st));
  return TQR_OK;
}

extern "C" {

const char* tqr_status_string(tqr_status st) {
  switch (st) {
    case TQR_OK: return "TQR_OK";
    case TQR_ERR_INVALID_ARG: return "TQR_ERR_INVALID_ARG";
    case TQR_ERR_CUDA: return "TQR_ERR_CUDA";
    case TQR_ERR_NCCL: return "TQR_ERR_NCCL";
    case TQR_ERR_OOM: return "TQR_ERR_OOM";
    case TQR_ERR_UNSUPPORTED: return "TQR_ERR_UNSUPPORTED";
  }
  return "TQR_ERR_UNKNOWN";
}
const char* tqr_last_error(void) { return g_err.c_str(); }
int32_t tqr_last_bad_arg(void) { return g_badarg; }
int32_t tqr_supported(int32_t b, int32_t s) { return exec_supported(b, s) ? 1 : 0; }

double tqr_flops_standard(int64_t m, int64_t n) {
  const double M = (double)m, N = (double)n;
  return m >= n ? 2.0 * N * N * (M - N / 3.0) : 2.0 * M * M * (N - M / 3.0);
}

double tqr_flops_tiled(int64_t m, int64_t n, int32_t b, int32_t s) {
  const int64_t p = (m + b - 1) / b, q = (n + b - 1) / b, K = std::min(p, q);
  const double B = b, S = s, B3 = B * B * B, B2 = B * B;
  const double fg = 4.0 / 3 * B3 + 2.0 / 3 * S * B2, fl = 2.0 * B3 + S * B2;
  const double ft = 2.0 * B3 + 4.0 / 3 * S * B2, fs = 4.0 * B3 + S * B2;
  double tot = 0.0;
  for (int64_t k = 0; k < K; ++k)
    tot += fg + (double)(q - k - 1) * fl + (double)(p - k - 1) * ft + (double)(p - k - 1) * (double)(q - k - 1) * fs;
  return tot;
}

tqr_status tqr_plan_create(tqr_plan** out, const tqr_params* p) {
  g_badarg = 0;
  if (!out) return bad_arg(1, "out is NULL");
  *out = nullptr;
  if (!p) return bad_arg(2, "params is NULL");
  if (p->m < 1) return bad_arg(1, "m < 1");
  if (p->n < 1) return bad_arg(2, "n < 1");
  if (p->b < 1) return bad_arg(3, "b < 1");
  if (p->s < 1 || p->s > p->b || p->b % p->s != 0) return bad_arg(4, "s must satisfy 1 <= s <= b and s | b");
  if (p->nranks < 1) return bad_arg(7, "nranks < 1");
  if (p->rank < 0 || p->rank >= p->nranks) return bad_arg(8, "rank outside [0, nranks)");
  if (p->nranks != 1) {
    g_err = "multi-GPU plans are not built in this version";
    return TQR_ERR_UNSUPPORTED;
  }
  if (!exec_supported(p->b, p->s)) {
    g_err = "no kernel instance for this (b, s)";
    return TQR_ERR_UNSUPPORTED;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || p->device < 0 || p->device >= ndev)
    return bad_arg(5, "device ordinal not available");
  CU(cudaSetDevice(p->device));
  tqr_plan* P = new tqr_plan();
  P->prm = *p;
  P->p = (p->m + p->b - 1) / p->b;
  P->q = (p->n + p->b - 1) / p->b;
  P->K = std::min(P->p, P->q);
  P->nsl = (p->b + exec_slice(p->b, p->s) - 1) / exec_slice(p->b, p->s);
  P->st = (cudaStream_t)p->stream;
  P->workers = exec_max_ctas(p->b, p->s, p->device);
  if (P->workers < 1) {
    delete P;
    g_err = "executor does not fit on this device";
    return TQR_ERR_UNSUPPORTED;
  }
  if ((int64_t)P->K * P->q * P->nsl + P->K >= (1 << 24)) {
    delete P;
    g_err = "problem too large for 24-bit counter indices";
    return TQR_ERR_UNSUPPORTED;
  }
  Sched s;
  build_factor_sched(P->p, P->q, p->b, p->s, P->nsl, P->workers, s);
  if (!s.topo_ok) {
    delete P;
    g_err = "internal: schedule is not topological";
    return TQR_ERR_UNSUPPORTED;
  }
  tqr_status st = upload(P, s, P->fact);
  if (st != TQR_OK) { delete P; return st; }
  if (cudaMalloc(&P->d_ticket, sizeof(int)) != cudaSuccess) { delete P; return TQR_ERR_OOM; }
  *out = P;
  return TQR_OK;
}

tqr_status tqr_plan_destroy(tqr_plan* P) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (P->fact.d_tasks) cudaFree(P->fact.d_tasks);
  for (auto& kv : P->orm) cudaFree(kv.second.d_tasks);
  if (P->d_ctr) cudaFree(P->d_ctr);
  if (P->d_ticket) cudaFree(P->d_ticket);
  if (P->d_trace) cudaFree(P->d_trace);
  delete P;
  return TQR_OK;
}

tqr_status tqr_tiles_size(const tqr_plan* P, size_t* a, size_t* t) {
  if (!P) return bad_arg(1, "plan is NULL");
  const size_t b = (size_t)P->prm.b, s = (size_t)P->prm.s;
  if (a) *a = (size_t)P->p * P->q * b * b;
  if (t) *t = (size_t)P->p * P->q * s * b;
  return TQR_OK;
}
static size_t work_bytes(const tqr_plan* P) {
  const size_t b = (size_t)P->prm.b, s = (size_t)P->prm.s;
  return ((size_t)P->p * P->q * b * b + (size_t)P->p * P->q * s * b) * sizeof(double);
}
tqr_status tqr_workspace_size(const tqr_plan* P, size_t* bytes) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (bytes) *bytes = work_bytes(P);
  return TQR_OK;
}

tqr_status tqr_pack(tqr_plan* P, const double* A, int64_t lda, double* At) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!A) return bad_arg(2, "A is NULL");
  if (lda < P->prm.m) return bad_arg(3, "lda < m");
  if (!At) return bad_arg(4, "At is NULL");
  CU(launch_pack(A, lda, At, P->prm.m, P->prm.n, P->prm.b, P->p, P->q, P->st));
  return TQR_OK;
}
tqr_status tqr_unpack(tqr_plan* P, const double* At, double* A, int64_t lda) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!At) return bad_arg(2, "At is NULL");
  if (!A) return bad_arg(3, "A is NULL");
  if (lda < P->prm.m) return bad_arg(4, "lda < m");
  CU(launch_unpack(At, A, lda, P->prm.m, P->prm.n, P->prm.b, P->p, P->st));
  return TQR_OK;
}
tqr_status tqr_get_r(tqr_plan* P, const double* At, double* R, int64_t ldr) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!At) return bad_arg(2, "At is NULL");
  if (!R) return bad_arg(3, "R is NULL");
  if (ldr < std::min(P->prm.m, P->prm.n)) return bad_arg(4, "ldr < min(m, n)");
  CU(launch_get_r(At, R, ldr, P->prm.m, P->prm.n, P->prm.b, P->p, P->st));
  return TQR_OK;
}

tqr_status tqr_geqrf(tqr_plan* P, double* At, double* T, void* work) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!At) return bad_arg(2, "At is NULL");
  if (!T) return bad_arg(3, "T is NULL");
  if (!work) return bad_arg(4, "work is NULL (tqr_workspace_size bytes required)");
  const size_t tsz = (size_t)P->p * P->q * P->prm.s * P->prm.b;
  CU(cudaMemsetAsync(T, 0, tsz * sizeof(double), P->st));
  return run(P, P->fact, At, T, nullptr, work, (P->prm.flags & TQR_FLAG_TRACE) != 0);
}

static tqr_status orm_sched(tqr_plan* P, bool trans, int64_t nrhs, DevSched** out) {
  auto key = std::make_pair(trans ? 1 : 0, nrhs);
  auto it = P->orm.find(key);
  if (it == P->orm.end()) {
    const int64_t qb = (nrhs + P->prm.b - 1) / P->prm.b;
    if ((int64_t)P->K * qb * P->nsl >= (1 << 24)) {
      g_err = "nrhs too large for 24-bit counter indices";
      return TQR_ERR_UNSUPPORTED;
    }
    Sched s;
    build_orm_sched(P->p, P->q, qb, P->prm.b, P->prm.s, P->nsl, trans, P->workers, s);
    if (!s.topo_ok) {
      g_err = "internal: apply-Q schedule is not topological";
      return TQR_ERR_UNSUPPORTED;
    }
    DevSched d;
    d.mode = trans ? 1 : 2;
    tqr_status st = upload(P, s, d);
    if (st != TQR_OK) return st;
    it = P->orm.emplace(key, d).first;
  }
  *out = &it->second;
  return TQR_OK;
}

tqr_status tqr_ormqr(tqr_plan* P, char trans, const double* At, const double* T, double* Bt, int64_t nrhs,
                     void* work) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (trans != 'T' && trans != 'N' && trans != 't' && trans != 'n') return bad_arg(2, "trans must be 'T' or 'N'");
  if (!At) return bad_arg(3, "At is NULL");
  if (!T) return bad_arg(4, "T is NULL");
  if (!Bt) return bad_arg(5, "Bt is NULL");
  if (nrhs < 1) return bad_arg(6, "nrhs < 1");
  if (!work) return bad_arg(7, "work is NULL (tqr_workspace_size bytes required)");
  DevSched* d = nullptr;
  tqr_status st = orm_sched(P, trans == 'T' || trans == 't', nrhs, &d);
  if (st != TQR_OK) return st;
  double* Yp = reinterpret_cast<double*>(work);
  double* Tp = Yp + (size_t)P->p * P->q * P->prm.b * P->prm.b;
  CU(launch_pack_factors(At, T, Yp, Tp, P->prm.b, P->prm.s, P->p, P->K, P->st));
  return run(P, *d, const_cast<double*>(At), const_cast<double*>(T), Bt, work, false);
}

tqr_status tqr_orgqr(tqr_plan* P, const double* At, const double* T, int64_t k, double* Qt, void* work) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!At) return bad_arg(2, "At is NULL");
  if (!T) return bad_arg(3, "T is NULL");
  if (k < 1 || k > P->prm.m) return bad_arg(4, "k outside [1, m]");
  if (!Qt) return bad_arg(5, "Qt is NULL");
  if (!work) return bad_arg(6, "work is NULL (tqr_workspace_size bytes required)");
  const int64_t qb = (k + P->prm.b - 1) / P->prm.b;
  CU(launch_eye_tiles(Qt, P->prm.m, k, P->prm.b, P->p, qb, P->st));
  return tqr_ormqr(P, 'N', At, T, Qt, k, work);
}

tqr_status tqr_sync(tqr_plan* P) {
  if (!P) return bad_arg(1, "plan is NULL");
  CU(cudaStreamSynchronize(P->st));
  CU(cudaGetLastError());
  return TQR_OK;
}

tqr_status tqr_schedule_inspect(int64_t p, int64_t q, int32_t nslice, int32_t workers, int64_t counts[4],
                                int64_t* n_edges) {
  g_badarg = 0;
  if (p < 1) return bad_arg(1, "p < 1");
  if (q < 1) return bad_arg(2, "q < 1");
  if (nslice < 1) return bad_arg(3, "nslice < 1");
  if (workers < 1) return bad_arg(4, "workers < 1");
  Sched s;
  build_factor_sched(p, q, 64 * nslice, 8, nslice, workers, s);
  if (counts)
    for (int c = 0; c < 4; ++c) counts[c] = s.counts[c];
  if (n_edges) *n_edges = s.nedges;
  if (!s.topo_ok) {
    g_err = "schedule is not a topological order";
    return TQR_ERR_UNSUPPORTED;
  }
  return TQR_OK;
}

tqr_status tqr_trace_fetch(tqr_plan* P, int64_t* rec, int64_t cap, int64_t* n) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!rec && cap > 0) return bad_arg(2, "rec is NULL");
  if (!n) return bad_arg(4, "n is NULL");
  *n = 0;
  if (!P->d_trace || P->trace_n == 0) return TQR_OK;
  const int64_t cnt = std::min<int64_t>(cap, P->trace_n);
  std::vector<unsigned long long> raw((size_t)cnt * 4);
  std::vector<int> tasks((size_t)cnt * TASK_INTS);
  CU(cudaStreamSynchronize(P->st));
  CU(cudaMemcpy(raw.data(), P->d_trace, raw.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(tasks.data(), P->fact.d_tasks, tasks.size() * sizeof(int), cudaMemcpyDeviceToHost));
  for (int64_t r = 0; r < cnt; ++r) {
    const int* t = &tasks[(size_t)r * TASK_INTS];
    int64_t* o = rec + r * 8;
    o[0] = t[0]; o[1] = t[1]; o[2] = t[2]; o[3] = t[3]; o[4] = t[4];
    o[5] = (int64_t)(raw[r * 4] >> 32);
    o[6] = (int64_t)raw[r * 4 + 2];
    o[7] = (int64_t)raw[r * 4 + 3];
  }
  *n = cnt;
  return TQR_OK;
}

tqr_status tqr_profile_tasks(tqr_plan* P, int32_t kind, int64_t count, double* At, double* T, void* work) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (kind < 0 || kind > 7) return bad_arg(2, "kind outside [0, 7]");
  if (count < 1 || count > (1 << 24)) return bad_arg(3, "count outside [1, 2^24]");
  if (!At) return bad_arg(4, "At is NULL");
  if (!T) return bad_arg(5, "T is NULL");
  if (P->p < 2 || P->q < 2) {
    g_err = "profiling needs p >= 2 and q >= 2";
    return TQR_ERR_UNSUPPORTED;
  }
  Sched s;
  s.rec.assign((size_t)count * TASK_INTS, 0);
  for (int64_t t = 0; t < count; ++t) {
    int* q = &s.rec[(size_t)t * TASK_INTS];
    const int i = 1 + (int)(t % (P->p - 1));
    const int j = 1 + (int)((t / (P->p - 1)) % (P->q - 1));
    q[0] = kind;
    q[1] = kind == 0 ? (int)(t % P->K) : 0;
    const bool lkind = kind == 2 || kind == 4 || kind == 6;
    q[2] = (kind == 0 || lkind) ? q[1] : i;
    q[3] = (kind == 0 || kind == 1) ? q[1] : j;
    q[4] = (int)(t % P->nsl);
    q[5] = 0;
    q[6] = 1;
  }
  s.ntasks = (int)count;
  s.nctr = 1;
  DevSched d;
  d.mode = kind >= 6 ? 2 : (kind >= 4 ? 1 : 0);
  tqr_status st = upload(P, s, d);
  if (st != TQR_OK) return st;
  if (!work) return bad_arg(6, "work is NULL");
  st = run(P, d, At, T, At, work, false);
  cudaStreamSynchronize(P->st);
  cudaFree(d.d_tasks);
  return st;
}

// Profiling builds (-DTQR_PROFILE_PHASES): attach a device array of 8 int64 phase-cycle
// totals (NULL detaches).  Not declared in tqr.h: development aid only.
tqr_status tqr_phase_counters(tqr_plan* P, long long* d_counters) {
  if (!P) return bad_arg(1, "plan is NULL");
  P->d_phases = d_counters;
  return TQR_OK;
}

}  // extern "C"
