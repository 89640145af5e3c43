// tlu_host.cpp -- host runtime of the tiled LU (include/tlu.h): plan, DAG task table in
// list-schedule order, and the C ABI.  The DAG is the tiled QR's with the
// kernels renamed (LU7); every dependency is a chain, expressed on the device as
// "progress counter >= value":
//   PF[k][l]      counts GETRF(k) block l (1), TSTRF(k,i) block l (i - k + 1) -- block lane l of
//                 the chain on U_kk (panel tasks per inner block, LU11)
//   col[k][j][sl] counts GESSM(k,j,sl) (1), SSSSM(k,i,j,sl) (i - k + 1)  -- the chain on A_kj
//   G(k,l)       <- PF[k][l-1] >= 1 (l > 0) | col[k-1][k][*] >= 2 (l = 0; A_kk after step k-1)
//   L(k,j,sl)    <- PF[k][last] >= 1;  col[k-1][j][sl] >= 2
//   T(k,i,l)     <- PF[k][l] >= i - k;  PF[k][l-1] >= i - k + 1 (l > 0) | col[k-1][k][*] >= i - k + 2
//   S(k,i,j,sl)  <- PF[k][last] >= i - k + 1;  col[k][j][sl] >= i - k;  col[k-1][j][sl] >= i - k + 2
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tlu.h"
#include "tlu_internal.h"
#include "tqr_internal.h"
#include "tqr_sched.h"

using namespace tqr;
using namespace tqr::lu;
using namespace tqr::sched;

struct tlu_plan {
  tlu_params prm{};
  int64_t p = 0, q = 0, K = 0;
  int nsl = 1, w = 0, grid = 0;
  cudaStream_t st = nullptr;
  int* d_tasks = nullptr;
  int ntasks = 0;
  int* d_ctr = nullptr;  // nctr counters + the ticket
  int nctr = 0;
  std::vector<int> rec;
  unsigned long long* d_trace = nullptr;
  double makespan = 0.0, busy = 0.0;
};

namespace {

tqr_status bad(int idx, const char* what) {
  set_last_error(what, idx);
  return TQR_ERR_INVALID_ARG;
}
tqr_status cuda_err(cudaError_t e, const char* where) {
  set_last_error((std::string(where) + ": " + cudaGetErrorString(e)).c_str(), 0);
  return TQR_ERR_CUDA;
}
struct DevGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
    else prev = -1;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
#define LU_CU(call)                                          \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return cuda_err(e_, #call);       \
  } while (0)
inline bool misaligned(const void* ptr) { return ((uintptr_t)ptr & 15u) != 0; }

// Modelled task durations (ns; the list schedule's priorities only, never results): update
// tasks at ~60% of the 251 GFLOP/s per-SM fp64 DMMA peak plus ~3 us of interchange / solve
// work per block; panels latency-bound at ~(1 + b/128) us per column.
struct LuDur {
  double g, t, l, s;
  LuDur(int b, int s_, int w) {
    const double sm = 251.0 * 0.6;
    const double nb = (double)b / s_;
    const double upd = nb * (2.0 * b * s_ * w / sm + 3000.0 * w / 64.0);
    l = 0.5 * upd;
    s = upd;
    const double col = 1000.0 + 8.0 * b;
    g = b * col + 0.5 * nb * upd;
    t = b * col + nb * upd;
  }
};

void build_lu_sched(int64_t p, int64_t q, int b, int s, int nsl, int w, int workers, Sched& out, int& nctr,
                    bool split = true) {
  // split (LU11): GETRF / TSTRF tasks per inner block l -- the flat TSTRF chain on
  // U_kk becomes a wavefront over (i, l), as for the QR panels (R21).  Block l of a tile touches
  // U_kk's rows of block l only (its column loop and the trailing update of those rows), so
  // block lane l is a chain G(k,l) -> T(k,k+1,l) -> T(k,k+2,l) -> ..., and inside a tile
  // T(k,i,l-1) -> T(k,i,l) (the trailing update of block l-1 feeds block l's columns).
  const int K = (int)std::min(p, q);
  const int NB = split ? b / s : 1;
  auto PF = [&](int k, int l) { return k * NB + l; };
  auto col = [&](int k, int j, int sl) { return K * NB + ((k * (int)q) + j) * nsl + sl; };
  nctr = K * NB + K * (int)q * nsl;
  const LuDur D(b, s, w);
  TaskGen T;
  for (int k = 0; k < K; ++k) {
    for (int l = 0; l < NB; ++l) {
      int id = T.add(LK_G, k, k, k, split ? l : -1, PF(k, l), 1, D.g / NB, 0);
      if (l > 0) T.dep(id, PF(k, l - 1), 1, 1);
      else if (k > 0) T.dep(id, col(k - 1, k, 0), nsl, 2);
    }
    for (int j = k + 1; j < q; ++j)
      for (int sl = 0; sl < nsl; ++sl) {
        int id = T.add(LK_L, k, k, j, sl, col(k, j, sl), 1, D.l, 2);
        T.dep(id, PF(k, NB - 1), 1, 1);
        if (k > 0) T.dep(id, col(k - 1, j, sl), 1, 2);
      }
    for (int i = k + 1; i < p; ++i) {
      for (int l = 0; l < NB; ++l) {
        int id = T.add(LK_T, k, i, k, split ? l : -1, PF(k, l), i - k + 1, D.t / NB, 1);
        T.dep(id, PF(k, l), 1, i - k);
        if (l > 0) T.dep(id, PF(k, l - 1), 1, i - k + 1);
        else if (k > 0) T.dep(id, col(k - 1, k, 0), nsl, i - k + 2);
      }
      for (int j = k + 1; j < q; ++j)
        for (int sl = 0; sl < nsl; ++sl) {
          int id = T.add(LK_S, k, i, j, sl, col(k, j, sl), i - k + 1, D.s, 3);
          T.dep(id, PF(k, NB - 1), 1, i - k + 1);
          T.dep(id, col(k, j, sl), 1, i - k);
          if (k > 0) T.dep(id, col(k - 1, j, sl), 1, i - k + 2);
        }
    }
  }
  for (auto& x : T.t) {
    if (x.kind == LK_G) out.counts[0]++;
    else if (x.kind == LK_T) out.counts[1]++;
    else if (x.kind == LK_L) out.counts[2]++;
    else out.counts[3]++;
  }
  // per-edge handoff term of the bottom-level priority (as the QR policy: the panel-chain-bound
  // b <= 128 grids favour chain hops -- LU C2 9.21 -> 8.97 ms; C3 insensitive)
  double lat = b <= 128 ? 200000.0 : 4000.0;
  if (const char* e = getenv("TLU_DEV_LAT")) lat = atof(e);
  if (!list_schedule(T, std::vector<int>{workers}, out, PRIO_BLEVEL, lat)) out.topo_ok = false;
}

}  // namespace

extern "C" {

int32_t tlu_supported(int32_t b, int32_t s) { return lu_supported(b, s) ? 1 : 0; }

double tlu_flops_standard(int64_t m, int64_t n) {
  const double M = (double)m, N = (double)n;
  return m >= n ? M * N * N - N * N * N / 3.0 : N * M * M - M * M * M / 3.0;
}

// executed count (LU9): per kernel, multiply-adds x 2 plus the divisions
double tlu_flops_tiled(int64_t m, int64_t n, int32_t b, int32_t s) {
  if (b < 1 || s < 1 || b % s) return 0.0;
  const double B = b, Sv = s;
  double g = 0, l = 0, t = 0, ss = 0;
  for (int c0 = 0; c0 < b; c0 += s) {
    const double tc = B - c0 - Sv;
    for (int c = c0; c < c0 + s; ++c) {
      g += (B - c - 1) + 2.0 * (B - c - 1) * (c0 + Sv - c - 1);
      t += B + 2.0 * B * (c0 + Sv - c - 1);
    }
    g += Sv * (Sv - 1) * tc + 2.0 * tc * Sv * tc;
    t += Sv * (Sv - 1) * tc + 2.0 * B * Sv * tc;
    l += Sv * (Sv - 1) * B + 2.0 * tc * Sv * B;
    ss += Sv * (Sv - 1) * B + 2.0 * B * Sv * B;
  }
  const int64_t p = (m + b - 1) / b, q = (n + b - 1) / b, K = std::min(p, q);
  double f = 0.0;
  for (int64_t k = 0; k < K; ++k) {
    const double nr = (double)(p - k - 1), nc = (double)(q - k - 1);
    f += g + nc * l + nr * t + nr * nc * ss;
  }
  return f;
}

tqr_status tlu_plan_create(tlu_plan** out, const tlu_params* prm) {
  if (!out) return bad(1, "out is NULL");
  if (!prm) return bad(2, "params is NULL");
  if (prm->m < 1) return bad(1, "m < 1");
  if (prm->n < 1) return bad(2, "n < 1");
  if (prm->b < 1) return bad(3, "b < 1");
  if (prm->s < 1 || prm->s > prm->b || prm->b % prm->s != 0) return bad(4, "s must satisfy 1 <= s <= b and s | b");
  if (!lu_supported(prm->b, prm->s)) {
    set_last_error("tlu: no kernel instance for this (b, s)", 0);
    return TQR_ERR_UNSUPPORTED;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || prm->device < 0 || prm->device >= ndev)
    return bad(5, "device ordinal not available");
  DevGuard dg(prm->device);
  if (dg.err != cudaSuccess) return cuda_err(dg.err, "cudaSetDevice");
  tlu_plan* P = new tlu_plan();
  P->prm = *prm;
  P->st = (cudaStream_t)prm->stream;
  P->p = (prm->m + prm->b - 1) / prm->b;
  P->q = (prm->n + prm->b - 1) / prm->b;
  P->K = std::min(P->p, P->q);
  P->w = lu_slice(prm->b, prm->s);
  P->nsl = prm->b / P->w;
  P->grid = lu_max_ctas(prm->b, prm->s, prm->device);
  if (P->grid < 1) {
    delete P;
    set_last_error("tlu: the executor does not fit on this device", 0);
    return TQR_ERR_UNSUPPORTED;
  }
  Sched sc;
  build_lu_sched(P->p, P->q, prm->b, prm->s, P->nsl, P->w, P->grid, sc, P->nctr);
  if (!sc.topo_ok) {
    delete P;
    set_last_error("tlu: inconsistent task graph (internal error)", 0);
    return TQR_ERR_UNSUPPORTED;
  }
  P->rec = sc.rec[0];
  P->ntasks = (int)(P->rec.size() / TASK_INTS);
  P->makespan = sc.makespan;
  P->busy = sc.busy;
  cudaError_t e = cudaMalloc(&P->d_tasks, sizeof(int) * std::max<size_t>(1, P->rec.size()));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_ctr, sizeof(int) * (P->nctr + 1));
  if (e == cudaSuccess && (prm->flags & TQR_FLAG_TRACE))
    e = cudaMalloc(&P->d_trace, sizeof(unsigned long long) * 4 * std::max(1, P->ntasks));
  if (e == cudaSuccess && !P->rec.empty())
    e = cudaMemcpy(P->d_tasks, P->rec.data(), sizeof(int) * P->rec.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(P->d_tasks);
    cudaFree(P->d_ctr);
    cudaFree(P->d_trace);
    delete P;
    cudaGetLastError();
    set_last_error("tlu_plan_create: device allocation failed", 0);
    return TQR_ERR_OOM;
  }
  *out = P;
  return TQR_OK;
}

tqr_status tlu_plan_destroy(tlu_plan* P) {
  if (!P) return TQR_OK;
  DevGuard dg(P->prm.device);
  cudaFree(P->d_tasks);
  cudaFree(P->d_ctr);
  cudaFree(P->d_trace);
  delete P;
  return TQR_OK;
}

tqr_status tlu_sizes(const tlu_plan* P, size_t* a_doubles, size_t* w_doubles, size_t* piv_ints) {
  if (!P) return bad(1, "plan is NULL");
  const size_t b = (size_t)P->prm.b, s = (size_t)P->prm.s;
  if (a_doubles) *a_doubles = (size_t)P->p * (size_t)P->q * b * b;
  if (w_doubles) *w_doubles = (size_t)P->p * (size_t)P->K * s * b;
  if (piv_ints) *piv_ints = (size_t)P->p * (size_t)P->K * b;
  return TQR_OK;
}

// workspace = the blocks' interchange lists, then (16-byte aligned) the Ltilde tiles (LU12)
static size_t perm_bytes(const tlu_plan* P) {
  const size_t n = sizeof(int) * (size_t)P->p * (size_t)P->K * (size_t)lu_perm_ints(P->prm.b, P->prm.s);
  return (n + 15) & ~(size_t)15;
}

tqr_status tlu_workspace_size(const tlu_plan* P, size_t* bytes) {
  if (!P) return bad(1, "plan is NULL");
  if (!bytes) return bad(2, "bytes is NULL");
  *bytes = perm_bytes(P);
  if (lu_uses_ltilde(P->prm.b, P->prm.s))
    *bytes += sizeof(double) * (size_t)P->p * (size_t)P->K * (size_t)lu_ltilde_doubles(P->prm.b, P->prm.s);
  return TQR_OK;
}

tqr_status tlu_pack(tlu_plan* P, const double* A, int64_t lda, double* At) {
  if (!P) return bad(1, "plan is NULL");
  if (!A || misaligned(A)) return bad(2, "A is NULL or not 16-byte aligned");
  if (lda < P->prm.m) return bad(3, "lda < m");
  if (!At || misaligned(At)) return bad(4, "At is NULL or not 16-byte aligned");
  DevGuard dg(P->prm.device);
  LU_CU(launch_pack(A, lda, At, P->prm.m, P->prm.n, P->prm.b, P->p, P->q, 1, 0, P->st));
  return TQR_OK;
}

tqr_status tlu_unpack(tlu_plan* P, const double* At, double* A, int64_t lda) {
  if (!P) return bad(1, "plan is NULL");
  if (!At || misaligned(At)) return bad(2, "At is NULL or not 16-byte aligned");
  if (!A || misaligned(A)) return bad(3, "A is NULL or not 16-byte aligned");
  if (lda < P->prm.m) return bad(4, "lda < m");
  DevGuard dg(P->prm.device);
  LU_CU(launch_unpack(At, A, lda, P->prm.m, P->prm.n, P->prm.b, P->p, P->q, 1, 0, P->st));
  return TQR_OK;
}

tqr_status tlu_get_u(tlu_plan* P, const double* At, double* U, int64_t ldu) {
  if (!P) return bad(1, "plan is NULL");
  if (!At || misaligned(At)) return bad(2, "At is NULL or not 16-byte aligned");
  if (!U || misaligned(U)) return bad(3, "U is NULL or not 16-byte aligned");
  if (ldu < std::min(P->prm.m, P->prm.n)) return bad(4, "ldu < min(m, n)");
  DevGuard dg(P->prm.device);
  LU_CU(launch_get_r(At, U, ldu, P->prm.m, P->prm.n, P->prm.b, P->p, P->q, 1, 0, P->st));
  return TQR_OK;
}

tqr_status tlu_getrf(tlu_plan* P, double* At, double* Wt, int32_t* piv, void* work) {
  if (!P) return bad(1, "plan is NULL");
  if (!At || misaligned(At)) return bad(2, "At is NULL or not 16-byte aligned");
  if (!Wt || misaligned(Wt)) return bad(3, "W is NULL or not 16-byte aligned");
  if (!piv || misaligned(piv)) return bad(4, "piv is NULL or not 16-byte aligned");
  if (!work || misaligned(work)) return bad(5, "work is NULL or not 16-byte aligned");
  DevGuard dg(P->prm.device);
  LU_CU(cudaMemsetAsync(P->d_ctr, 0, sizeof(int) * (P->nctr + 1), P->st));
  LuArgs a{};
  a.tasks = P->d_tasks;
  a.ntasks = P->ntasks;
  a.ticket = P->d_ctr + P->nctr;
  a.ctr = P->d_ctr;
  a.A = At;
  a.W = Wt;
  a.piv = piv;
  a.perm = (int*)work;
  a.Lw = lu_uses_ltilde(P->prm.b, P->prm.s) ? (double*)((char*)work + perm_bytes(P)) : nullptr;
  a.p = (int)P->p;
  a.q = (int)P->q;
  a.nctr = P->nctr;
  // dispatch by warp 2 during the release (tlu_exec.cu, the DISP kernel instance): throughput-bound grids only --
  // same-box C3 LU 169.0 -> 166.9 ms; the chain-bound C2 (8.80 -> 8.99 ms) and C4 (52.9 -> 53.7)
  // keep the dispatch after the release
  a.disp = P->prm.b >= 256 && std::min(P->p, P->q) >= 32;
  if (const char* e = getenv("TLU_DEV_DISP")) a.disp = atoi(e) != 0;
  a.trace = P->d_trace;
  LU_CU(launch_lu_exec(P->prm.b, P->prm.s, a, P->grid, P->st));
  return TQR_OK;
}

tqr_status tlu_sync(tlu_plan* P) {
  if (!P) return bad(1, "plan is NULL");
  DevGuard dg(P->prm.device);
  LU_CU(cudaStreamSynchronize(P->st));
  LU_CU(cudaGetLastError());
  return TQR_OK;
}

tqr_status tlu_plan_records(tlu_plan* P, int32_t* rec, int64_t cap, int64_t* n) {
  if (!P) return bad(1, "plan is NULL");
  if (!n) return bad(4, "n is NULL");
  *n = P->ntasks;
  if (rec) std::memcpy(rec, P->rec.data(), sizeof(int32_t) * (size_t)std::min<int64_t>(cap, *n) * TASK_INTS);
  return TQR_OK;
}

tqr_status tlu_schedule_records(int64_t m, int64_t n, int32_t b, int32_t s, int32_t workers, int32_t* rec, int64_t cap,
                                int64_t* ntask, int32_t* nctr) {
  if (m < 1) return bad(1, "m < 1");
  if (n < 1) return bad(2, "n < 1");
  if (!lu_supported(b, s)) return bad(3, "no kernel instance for (b, s)");
  if (workers < 1) return bad(5, "workers < 1");
  if (!ntask) return bad(8, "ntask is NULL");
  const int64_t p = (m + b - 1) / b, q = (n + b - 1) / b;
  const int w = lu_slice(b, s);
  Sched sc;
  int nc = 0;
  build_lu_sched(p, q, b, s, b / w, w, workers, sc, nc);
  if (!sc.topo_ok) {
    set_last_error("tlu: inconsistent task graph (internal error)", 0);
    return TQR_ERR_UNSUPPORTED;
  }
  const auto& v = sc.rec[0];
  *ntask = (int64_t)(v.size() / TASK_INTS);
  if (nctr) *nctr = nc;
  if (rec) std::memcpy(rec, v.data(), sizeof(int32_t) * (size_t)std::min<int64_t>(cap, *ntask) * TASK_INTS);
  return TQR_OK;
}

tqr_status tlu_trace_fetch(tlu_plan* P, int64_t* rec, int64_t cap, int64_t* n) {
  if (!P) return bad(1, "plan is NULL");
  if (!n) return bad(4, "n is NULL");
  if (!P->d_trace) {
    set_last_error("tlu_trace_fetch: plan created without TQR_FLAG_TRACE", 0);
    return TQR_ERR_UNSUPPORTED;
  }
  DevGuard dg(P->prm.device);
  *n = P->ntasks;
  if (rec && cap > 0) {
    const int64_t m = std::min<int64_t>(cap, P->ntasks);
    std::vector<unsigned long long> tr((size_t)m * 4);
    LU_CU(cudaStreamSynchronize(P->st));
    LU_CU(cudaMemcpy(tr.data(), P->d_trace, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost));
    for (int64_t t = 0; t < m; ++t) {
      const int* r = &P->rec[(size_t)t * TASK_INTS];
      int64_t* o = rec + t * 8;
      o[0] = r[0]; o[1] = r[1]; o[2] = r[2]; o[3] = r[3]; o[4] = (int64_t)tr[t * 4];
      o[5] = (int64_t)tr[t * 4 + 1]; o[6] = (int64_t)tr[t * 4 + 2]; o[7] = (int64_t)tr[t * 4 + 3];
    }
  }
  return TQR_OK;
}

}  // extern "C"
