// tqr_host.cpp -- host runtime of the tiled QR library: plan, DAG task tables, list-schedule
// dispatch order, and the C ABI declared in include/tqr.h.
//
// DAG (edges derived from each kernel's read/write sets, SPEC dag module),
// with the panel tasks split by inner block l into an apply part A and a factor part F
// (R21; P(k,i) = GEQRT(k) for i = k, TSQRT(k,i) for i > k):
//   A(k,i,l)    <- F(k,i,l-1);  A(k,i-1,l)                       (l >= 1)
//   F(k,i,l)    <- F(k,i-1,l);  A(k,i,l) | S(k-1,i,k,*) (l = 0)
//   L(k,j,sl)   <- F(k,k, last), S(k-1,k,j,sl)
//   S(k,i,j,sl) <- F(k,i, last), L(k,j,sl) | S(k,i-1,j,sl), S(k-1,i,j,sl)
// Every dependency is a chain, so it is expressed on the device as "progress counter >=
// value": PF(k,l) / PA(k,l) count the F / A parts of P(k,k), P(k,k+1), ... ; col[k][j][sl]
// counts L(k,j,sl), S(k,k+1,j,sl), ...
// The dispatch (ticket) order is a list schedule of the DAG on `workers` CTAs by bottom
// level (critical path, R10; the paper's fixed priorities G > T > L > S of
// PAPER.md:606-615 remain selectable), ties by (k, i, j, slice); it is
// topological by construction, so with all CTAs co-resident no ticket can wait forever.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tqr.h"
#include "tqr_internal.h"
#include "tqr_sched.h"

using namespace tqr;
using namespace tqr::sched;

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
}  // namespace
// error state shared with the tiled-LU runtime (tlu_host.cpp): tqr_last_error / tqr_last_bad_arg
void tqr::set_last_error(const char* what, int bad_arg_idx) {
  g_err = what;
  g_badarg = bad_arg_idx;
}
namespace {
// The caller's current device is restored on return from every entry point that touches a
// device (calls may come from a thread whose current device is another GPU).
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
// include/tqr.h: every data pointer must be 16-byte aligned (TMA bulk copies and 16-byte
// vector accesses); a misaligned pointer is an invalid argument, not a device fault
static inline bool misaligned(const void* p) { return ((uintptr_t)p & 15u) != 0; }
#define GUARD(P)                                                         \
  DevGuard dg_((P)->prm.device);                                         \
  if (dg_.err != cudaSuccess) return cuda_fail(dg_.err, "cudaSetDevice")
#define ALIGNED(ptr, idx)                                                         \
  do {                                                                            \
    if (misaligned(ptr)) return bad_arg(idx, #ptr " is not 16-byte aligned");     \
  } while (0)
#define CU(call)                                            \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);     \
  } while (0)

// Per-task durations (ns) for the list schedule only (never affect results), fitted to the
// B200 traces of the r01 executor (tools/trace_stats.py; b = 256 / 128, s = 32):
//  * update tasks (LARFB, SSRFB, apply-Q): ~2 us fixed + the task's flops at 88% (RW = 256
//    executor) / 79% (RW = 128) of the 251 GFLOP/s per-SM fp64 DMMA peak (the LARFB form
//    applies the zero rows of U above block l as well, so it costs like SSRFB without C1);
//  * panel factor part (R21 F): ~14 us fixed + s columns at (0.25 + 0.00146 b) us each
//    (TSQRT b = 256: 34 us, b = 128: 28 us, r01 v11); GEQRT + 0.04 b us;
//  * panel apply part of block l (R21 A): (1.5 + 0.012 b) us + l block applies at 78%;
//  * fused panel sub-task (no A/F split): factor part + 1 us + 1.35 x the l block applies.
struct DurModel {
  double B, Sv, W, l, s, apply;
  DurModel(int b, int s_, int w, int rwm = 128) : B(b), Sv(s_), W(w) {
    const double sm = 251.0;  // GFLOP/s per SM == flop/ns
    const double eff = (rwm >= 256 && b >= 256) ? 0.88 : 0.79;
    l = 2000 + (4.0 * B * B * W) / (eff * sm);
    s = 2000 + (4.0 * B * B * W + Sv * B * W) / (eff * sm);
    apply = 4.0 * B * Sv * Sv / (0.78 * sm);
  }
  double factor(bool geqrt) const { return 14000 + Sv * (250 + 1.46 * B) + (geqrt ? 40 * B : 0); }
  double panel(int lb, bool geqrt) const { return factor(geqrt) + 1000 + 1.35 * lb * apply; }
  double apply_part(int lb) const { return 1500 + 12 * B + lb * apply; }
  double factor_part(bool geqrt) const { return factor(geqrt); }
};

// Ranks own tile columns j == r (mod G): the panel tasks G(k), T(k,i) run on
// owner(k) and publish the panel counter on every rank; L(k,j), S(k,i,j) run on owner(j).
// Counter layout per rank: panel[k] at k (K entries, a copy on every rank), then the local
// column counters col[k][jl][sl] (jl = j / G).  `real_layout`: tile storage holds only the
// rank's own columns (storage column jl); otherwise the full global grid (column j).
// nsl: column slices per tile (one register pass each; the unit of the progress counters);
// np: register passes per update task (np | nsl); fine: 1 = the updates of the lookahead
// column k+1 run as 1-pass tasks (they feed panel k+1: a shorter chain link), 2 = also every
// update of the steps whose default-granularity task count is below two waves (the tail).
static void build_factor_sched(int64_t p, int64_t q, int b, int s, int nsl, const std::vector<int>& workers,
                               bool real_layout, bool split, Sched& out, int prio = PRIO_CLASS, double lat = 0.0,
                               int rwm = 128, double blq = 0.0, int group = 0, int np = 1, int fine = 0,
                               bool early = false, double lat_remote = 0.0, bool pipe = false,
                               bool slicedep = true, int h = 1, double gtail = 0.75) {
  const int K = (int)std::min(p, q);
  const int G = (int)workers.size();
  const int w = (b + nsl - 1) / nsl;
  // which updates join their reflector panel's group (R22): not the lookahead columns
  // (j <= k + gj) and, in mode 3, not the last (1 - gt) of the steps, where the critical path
  // decides (development knobs TQR_DEV_GROUP_J / TQR_DEV_GROUP_TAIL)
  int gj = 1;
  double gt = gtail;
  if (const char* e = getenv("TQR_DEV_GROUP_J")) gj = atoi(e);
  if (const char* e = getenv("TQR_DEV_GROUP_TAIL")) gt = atof(e);
  auto grouped = [&](int k, int j) { return j > k + gj && (group != 3 || k < gt * K); };
  const int NPT = b / s;  // panel sub-tasks per tile: one per inner block l (one output T_l)
  if (np < 1 || nsl % np != 0) np = 1;
  DurModel dm(b, s, w * np, rwm), dmf(b, s, w, rwm);
  int64_t wtot = 0;
  for (int x : workers) wtot += x;
  TaskGen T;
  auto own = [&](int64_t j) { return (int)(j % G); };
  auto qloc = [&](int r) { return r < q ? (int)((q - r + G - 1) / G) : 0; };
  auto scol = [&](int64_t j) { return real_layout ? (int)(j / G) : (int)j; };
  // Panel progress of step k, per inner block l (a copy on every rank, R21):
  //   PF(k,l): factor parts done (GEQRT(k) then TSQRT(k,k+1), ...: value i-k+1 after TSQRT(k,i))
  //   PA(k,l): apply parts done, l >= 1 (left-looking update of block l's columns; owner only)
  //   PR(k,l): R_kk's rows of block l final (a factor part's early release, owner only)
  auto PF = [&](int k, int l) { return k * 3 * NPT + l; };
  auto PA = [&](int k, int l) { return k * 3 * NPT + NPT + l; };
  auto PR = [&](int k, int l) { return k * 3 * NPT + 2 * NPT + l; };
  auto COL = [&](int k, int64_t j, int sl) {
    return K * 3 * NPT + (int)(((int64_t)k * qloc(own(j)) + j / G) * nsl + sl);
  };
  out.nctr.assign(G, 0);
  for (int r = 0; r < G; ++r) out.nctr[r] = K * 3 * NPT + (int)((int64_t)K * qloc(r) * nsl);
  // Split apply parts (units of h > 1 tile rows, R30): A(k,u,l) becomes one sub-task
  // per earlier output block lp, A(k,u,l,lp); PA2(k,l,lp) counts them over the units (owner only)
  const bool asplit = h > 1 && split;
  auto PA2 = [&](int k, int l, int lp) {
    return K * 3 * NPT + (int)((int64_t)K * qloc(own(k)) * nsl) + (k * NPT + l) * NPT + lp;
  };
  if (asplit)
    for (int r = 0; r < G; ++r) out.nctr[r] += K * NPT * NPT;
  // One panel task on tile (i,k) block l in two parts: A (apply this tile's blocks < l to
  // block l's columns: touches the rows of R_kk ABOVE the diagonal block) and F (factor: the
  // diagonal block).  A(k,i+1,l) may overlap F(k,i,l), which halves the TSQRT chain's step.
  // the column slices (register passes of the update tasks) that hold inner block l's columns:
  // a panel part only needs THOSE updated by step k-1 (R32), not the whole tile
  const int sw = (b + nsl - 1) / nsl;
  auto blk_sl0 = [&](int l) { return slicedep ? (l * s) / sw : 0; };
  auto blk_nsl = [&](int l) { return slicedep ? ((l + 1) * s - 1) / sw - (l * s) / sw + 1 : nsl; };
  // Units (R30): the tile rows below the diagonal in groups of h starting at k+1;
  // unit g covers tile rows [k+1+hg, min(p, k+1+h(g+1))) and has chain value v = g + 2 (GEQRT:
  // 1).  h = 1: the square-tile schedule (unit g = tile row k+1+g, v = i-k+1).  A step-k task
  // on tile rows up to `il` waits for step k-1's chain on its column up to the unit holding il:
  auto prevv = [&](int k, int il) { return (il - k) / h + 2; };
  // modelled durations of a two-tile unit's panel parts (R30): 2x / 3x the one-tile model (the
  // trace fit is 1.35x / 2.1x; the larger weights raise the unit chain's priority: C4 with 2b x b
  // tiles 57.9 (1x) -> 55.6 (fit) -> 53.4 ms, profiles/r02_tall_sweep.txt) -- development knobs
  // TQR_DEV_TALLF / _TALLA; TQR_DEV_PANF / _PANA scale the one-tile panel parts likewise
  double tallf = 2.0, talla = 3.0, panf = 1.0, pana = 1.0;
  if (const char* e = getenv("TQR_DEV_TALLF")) tallf = atof(e);
  if (const char* e = getenv("TQR_DEV_TALLA")) talla = atof(e);
  if (const char* e = getenv("TQR_DEV_PANF")) panf = atof(e);
  if (const char* e = getenv("TQR_DEV_PANA")) pana = atof(e);
  auto panel = [&](int kind, int k, int i, int il, int v, int cls) {
    const int ok = own(k);
    const double uf = il > i ? tallf : panf, ua = il > i ? talla : pana;
    for (int l = 0; l < NPT; ++l) {
      if (!split) {  // fused apply + factor per block (R21 without the A/F split)
        int id = T.add(kind, k, i, scol(k), l, PF(k, l), v, uf * dm.panel(l, kind == K_G), cls);
        T.t[id].rank = ok; T.t[id].kc = scol(k); T.t[id].flags = 1;
        if (early) { T.t[id].out2_idx = PR(k, l); T.t[id].flags |= (PR(k, l) + 1) << 8; }
        if (v > 1) T.dep(id, early ? PR(k, l) : PF(k, l), 1, v - 1);  // R_kk block l: previous tile
        if (l > 0) T.dep(id, PF(k, l - 1), 1, v);
        if (k > 0) T.dep(id, COL(k - 1, k, blk_sl0(l)), blk_nsl(l), prevv(k, il));  // block l's columns
        if (il > i) T.t[id].flags |= 128;
        continue;
      }
      if (l > 0 && asplit) {
        // one apply sub-task per earlier output block lp (record [4] = l | (lp + 1) << 8):
        // A(k,u,l,lp) <- F(k,u,lp), A(k,u,l,lp-1), A(k,u-1,l,lp) (R_kk rows of block lp in
        // block l's columns) -- the unit chain of each stage is one block apply long
        for (int lp = 0; lp < l; ++lp) {
          int id = T.add(kind, k, i, scol(k), l | ((lp + 1) << 8), PA2(k, l, lp), v, ua * dm.apply_part(1), cls);
          T.t[id].rank = ok; T.t[id].kc = scol(k); T.t[id].flags = 2;
          T.t[id].key[3] = l * NPT + lp;
          T.dep(id, PF(k, lp), 1, v);                            // block lp of this unit factored
          if (lp > 0) T.dep(id, PA2(k, l, lp - 1), 1, v);        // block l's columns: previous sub-apply
          if (v > 1) T.dep(id, PA2(k, l, lp), 1, v - 1);         // R_kk rows of block lp: previous unit
          if (lp == 0 && k > 0) T.dep(id, COL(k - 1, k, blk_sl0(l)), blk_nsl(l), prevv(k, il));
          if (il > i) T.t[id].flags |= 128;
        }
      } else if (l > 0) {
        int id = T.add(kind, k, i, scol(k), l, PA(k, l), v, ua * dm.apply_part(l), cls);
        T.t[id].rank = ok; T.t[id].kc = scol(k); T.t[id].flags = 2;
        T.dep(id, PF(k, l - 1), 1, v);                 // this tile's blocks < l factored
        if (v > 1) T.dep(id, PA(k, l), 1, v - 1);      // R_kk rows above block l: previous tile
        if (k > 0) T.dep(id, COL(k - 1, k, blk_sl0(l)), blk_nsl(l), prevv(k, il));  // block l's columns
        if (il > i) T.t[id].flags |= 128;
      }
      int id = T.add(kind, k, i, scol(k), l, PF(k, l), v, uf * dm.factor_part(kind == K_G), cls);
      T.t[id].rank = ok; T.t[id].kc = scol(k); T.t[id].flags = 1 | 4;
      if (early) { T.t[id].out2_idx = PR(k, l); T.t[id].flags |= (PR(k, l) + 1) << 8; }
      if (v > 1) T.dep(id, early ? PR(k, l) : PF(k, l), 1, v - 1);  // R_kk diagonal block l: previous tile
      if (l > 0) T.dep(id, asplit ? PA2(k, l, l - 1) : PA(k, l), 1, v);  // own apply part(s)
      else if (k > 0) T.dep(id, COL(k - 1, k, blk_sl0(0)), blk_nsl(0), prevv(k, il));  // block 0's columns
      if (il > i) T.t[id].flags |= 128;
    }
  };
  for (int k = 0; k < K; ++k) {
    panel(K_G, k, k, k, 1, 0);
    out.counts[0]++;
    // task granularity of step k's updates (R23)
    const bool tail = fine >= 2 && (int64_t)(q - k - 1) * (p - k) * (nsl / np) < 2 * wtot;
    auto npj = [&](int64_t j) { return (fine >= 1 && j == k + 1) || tail ? 1 : np; };
    for (int j = k + 1; j < q; ++j)
      for (int sl = 0; sl < nsl; sl += npj(j)) {
        const int n_ = npj(j);
        // lookahead (R10): updates of column k+1 feed panel k+1 -> critical path
        int id = T.add(K_L, k, k, scol(j), sl, COL(k, j, sl), 1, (n_ == np ? dm : dmf).l, j == k + 1 ? 1 : 2);
        T.t[id].rank = own(j); T.t[id].kc = scol(k);
        T.t[id].key[2] = j;
        T.t[id].np = n_; T.t[id].ocnt = n_;
        if (group && grouped(k, j)) T.t[id].group = (int64_t)k * p + k;
        T.dep(id, PF(k, NPT - 1), 1, 1);
        if (own(j) != own(k)) T.t[id].flags |= 8;  // dep 0 is published by a peer GPU
        if (pipe) T.t[id].flags |= 64;             // pipelined panel dependency (R31)
        if (k > 0) T.dep(id, COL(k - 1, j, sl), n_, 2);
        out.counts[2] += n_;  // counted per register pass (column slice)
      }
    for (int i = k + 1, v = 2; i < p; i += h, ++v) {
      const int il = (int)std::min<int64_t>(p, (int64_t)i + h) - 1;  // the unit's last tile row
      // TSQRT(k,unit) block l touches only column block l of R_kk (and the unit's tiles): a
      // wavefront over (unit, l) (R21)
      panel(K_T, k, i, il, v, 1);
      out.counts[1]++;
      for (int j = k + 1; j < q; ++j)
        for (int sl = 0; sl < nsl; sl += npj(j)) {
          const int n_ = npj(j);
          int id = T.add(K_S, k, i, scol(j), sl, COL(k, j, sl), v, (n_ == np ? dm : dmf).s * (il - i + 1),
                         j == k + 1 ? 1 : 3);
          if (il > i) T.t[id].flags |= 128;
          T.t[id].rank = own(j); T.t[id].kc = scol(k);
          T.t[id].key[2] = j;
          T.t[id].np = n_; T.t[id].ocnt = n_;
          if (group && grouped(k, j)) T.t[id].group = (int64_t)k * p + i;
          T.dep(id, PF(k, NPT - 1), 1, v);
          if (own(j) != own(k)) T.t[id].flags |= 8;  // dep 0 is published by a peer GPU
          if (pipe) T.t[id].flags |= 64;             // pipelined panel dependency (R31)
          T.dep(id, COL(k, j, sl), n_, v - 1);
          if (k > 0) T.dep(id, COL(k - 1, j, sl), n_, prevv(k, il));
          out.counts[3] += n_;
        }
    }
  }
  if (!list_schedule(T, workers, out, prio, lat, blq, lat_remote, group == 2 ? 2 : 1)) out.topo_ok = false;
}

// apply-Q^T (trans) or apply-Q to a tile-major B with qb tile columns.
//   Q^T: step k ascending: L(k,jb,sl), then S(k,i,jb,sl) for i ascending (chain on B(k,jb)).
//        cnt[k][jb][sl]: L -> 1, S(k,i) -> i-k+1.
//   Q  : step k descending: S(k,i,jb,sl) for i descending, then L(k,jb,sl).
//        cnt[k][jb][sl]: S(k,i) -> p-i, L -> p-k.
// form_q (Q applied to [I; 0], tqr_orgqr): backward accumulation leaves the tile columns
// left of step k untouched (they are still unit vectors in rows >= k b), so the tasks
// (k, jb < k) are skipped -- the DORGQR saving, half the work of a dense Q*B.
// nslf: column slices (register passes) per tile; tasks cover np of them (counters per task slice).
// Multi-rank (workers.size() = G > 1): B's tile columns are 1D block-cyclic like A's, column
// jb is applied by rank jb mod G with the packed reflectors in that rank's own workspace (every
// rank holds every panel), so the ranks never wait on each other; counters are per rank,
// indexed by the local column jb / G; `real_layout`: B holds only the rank's own columns
// (record [3] = storage column jb / G), otherwise the global grid.
static void build_orm_sched(int64_t p, int64_t q, int64_t qb, int b, int s, int nslf, bool trans,
                            const std::vector<int>& workers, bool real_layout, Sched& out, bool form_q = false,
                            int prio = PRIO_CLASS, double lat = 0.0, int rwm = 128, int np = 1) {
  const int G = (int)workers.size();
  const int K = (int)std::min(p, q);
  if (np < 1 || nslf % np != 0) np = 1;
  const int nsl = nslf / np;
  const int w = (b + nsl - 1) / nsl;
  DurModel dm(b, s, w, rwm);
  TaskGen TG;
  auto qbl = [&](int r) { return r < qb ? (int)((qb - r + G - 1) / G) : 0; };
  auto CNT = [&](int k, int64_t jb, int sl) { return (int)(((int64_t)k * qbl((int)(jb % G)) + jb / G) * nsl + sl); };
  out.nctr.assign(G, 0);
  for (int r = 0; r < G; ++r) out.nctr[r] = (int)((int64_t)K * qbl(r) * nsl);
  auto add = [&](int kind, int k, int i, int64_t jb, int sl, int val, double dur, int cls) {
    int id = TG.add(kind, k, i, real_layout ? (int)(jb / G) : (int)jb, sl, CNT(k, jb, sl), val, dur, cls);
    TG.t[id].rank = (int)(jb % G);
    TG.t[id].key[2] = (int)jb;
    return id;
  };
  for (int64_t jb = 0; jb < qb; ++jb)
    for (int sl = 0; sl < nsl; ++sl) {
      if (trans) {
        for (int k = 0; k < K; ++k) {
          int id = add(K_LQT, k, k, jb, sl, 1, dm.l, 0);
          if (k > 0) TG.dep(id, CNT(k - 1, jb, sl), 1, 2);
          for (int i = k + 1; i < p; ++i) {
            id = add(K_SQT, k, i, jb, sl, i - k + 1, dm.s, 1);
            TG.dep(id, CNT(k, jb, sl), 1, i - k);
            if (k > 0) TG.dep(id, CNT(k - 1, jb, sl), 1, i - k + 2);
          }
        }
      } else {
        for (int k = K - 1; k >= 0; --k) {
          if (form_q && jb < k) continue;                       // untouched unit columns
          const bool prev = k + 1 < K && !(form_q && jb < k + 1);  // step k+1 had tasks here
          for (int i = (int)p - 1; i > k; --i) {
            int id = add(K_SQ, k, i, jb, sl, (int)p - i, dm.s, 1);
            TG.t[id].key[0] = K - 1 - k;  // reverse order: later steps first
            TG.t[id].key[1] = (int)p - 1 - i;
            if (i < p - 1) TG.dep(id, CNT(k, jb, sl), 1, (int)p - i - 1);
            if (prev) TG.dep(id, CNT(k + 1, jb, sl), 1, (int)p - i);
          }
          int id = add(K_LQ, k, k, jb, sl, (int)p - k, dm.l, 0);
          TG.t[id].key[0] = K - 1 - k;
          if (k + 1 < p) TG.dep(id, CNT(k, jb, sl), 1, (int)p - k - 1);
        }
      }
    }
  for (auto& x : TG.t) {  // record: first register pass (column slice of width b / nslf), passes
    x.np = np;
    x.sl *= np;
  }
  if (!list_schedule(TG, workers, out, prio, lat)) out.topo_ok = false;
}

struct DevSched {
  std::vector<int*> d_tasks;  // per local rank
  std::vector<int> ntasks;
  int mode = 0;  // executor instance: 0 factorization, 1 apply Q^T, 2 apply Q
  int nctr = 0;  // counters per rank (max over the local ranks)
};

}  // namespace

// Per-rank symmetric buffer (multi-rank plans): counters | arrive flags | reflector workspace.
struct SymLayout {
  size_t ctr_off, arrive_off, yp_off, tp_off, bytes;
};

struct tqr_plan {
  tqr_params prm;
  int64_t p, q, K;
  int nsl, workers;
  int passes = 1;      // register passes per update task (policy below)
  int fine = 2;        // 1-pass tasks for the lookahead column (1) and the tail steps (2) (R23)
  int rwm = 128;       // rows-per-warp variant of the executor (policy below)
  bool split = true;   // panel A/F split (R21)
  int prio = PRIO_BLEVEL;  // list-schedule priority (policy below)
  double lat = 4000.0;     // modelled per-task handoff latency of the list schedule (ns)
  int orm_prio = PRIO_BLEVEL;  // list-schedule priority of apply-Q / form-Q
  double blq = 0.0;            // bottom-level quantum (ns) of the factorization schedule
  int group = 0;               // group the updates of one reflector panel (R22)
  double gtail = 0.75;         //   ... in the steps k < gtail * K
  bool early = true;           // factor parts release R_kk's block rows early (R24)
  bool pipe = true;            // update tasks wait for the panel block by block (R31)
  bool slicedep = true;        // panel parts wait only for their block's column slices (R32)
  cudaStream_t st;
  int G = 1, me = 0;          // job ranks, this process's rank
  bool emulate = false;       // all G ranks in this process, one launch on one device
  int h = 1;                  // tile rows per TSQRT / SSRFB unit (2: TQR_FLAG_TALL_TILES, R30)
  int* d_units = nullptr;     // h = 2: the units (i0, k, nt) whose output T blocks form_t completes
  int nunits = 0;
  bool real = false;          // G > 1, one rank per process / GPU
  int nloc = 1;               // ranks run by this process
  int nctr_max = 0;
  DevSched fact;
  std::map<std::pair<int, int64_t>, DevSched> orm;
  // device state per job rank (index = rank); local ranks own their allocations
  int* ctr[MAX_RANKS] = {};
  int* arrive[MAX_RANKS] = {};
  double* Yp[MAX_RANKS] = {};
  double* Tp[MAX_RANKS] = {};
  void* sym_own[MAX_RANKS] = {};   // allocations owned by this process (multi-rank)
  void* sym_peer[MAX_RANKS] = {};  // IPC-opened peer allocations (real multi-rank)
  SymLayout lay{};
  bool connected = false;
  int* d_ctr1 = nullptr;      // single-rank counters
  int* d_octr = nullptr;      // multi-rank plans: rank-local apply-Q counters, nloc x octr_n
  int octr_n = 0;
  int* d_ticket = nullptr;    // one per local rank
  int gen = 0;                // call generation (counter base = gen * (p + 2))
  unsigned long long* d_trace = nullptr;
  std::vector<int64_t> trace_off;  // per local rank: offset (tasks) into d_trace
  int64_t trace_cap = 0;
  bool trace_valid = false;
  long long* d_phases = nullptr;  // set by tqr_phase_counters (profiling builds)
};

// Granularity policy (measured on B200, r01):
//  * square grids, b >= 256: the RW = 256 executor (a warp holds all 256 rows of its column
//    group: no row-partial exchange) with 128-column update tasks -- C3 224 ms (70.5%),
//    C5 12.5 s (80.7%) vs 232 ms / 13.7 s with RW = 128;
//  * tall-skinny grids (p >= 4q) are bound by the TSQRT chain: the RW = 128 executor with
//    32-column update tasks and the panel A/F split (C4: 60 ms vs 77 with RW = 256);
//  * b <= 128: RW = b, 1-pass tasks, fused panel blocks (the GEQRT/TSQRT chain dominates C2);
//  * dispatch order by bottom level (critical path) with a 4 us handoff per task, not by the
//    paper's fixed classes: C3 224 -> 213 ms, C4 62.1 -> 55.2 ms, C2 7.84 -> 7.33 ms.
struct Policy {
  int rwm = 128, passes = 1, nsl = 1, fine = 2, prio = PRIO_BLEVEL, orm_prio = PRIO_BLEVEL;
  bool split = true, early = true, pipe = true, slicedep = true;
  int group = 0;
  double gtail = 0.75;  // grouped updates only in the steps k < gtail * K (R22)
  double lat = 4000.0, blq = 0.0;
  int h = 1;  // tile rows per TSQRT / SSRFB unit
};
static Policy make_policy(int64_t p, int64_t q, int b, int s, bool tall_tiles = false, bool locality = false) {
  Policy P;
  if (tall_tiles) {  // the tall-unit executor: 32-column update passes, A/F-split panels (R30)
    P.h = 2;
    P.nsl = b / exec_slice_tall();
    P.passes = 1;
    P.split = true;
    P.early = true;
    P.pipe = false;
    P.slicedep = false;
    return P;
  }
  const bool tall = p >= 4 * q;
  P.rwm = (b >= 256 && !tall) ? 256 : 128;
  P.passes = b >= 256 ? (128 / exec_slice(b, s, P.rwm)) : 1;  // 128-column tasks
  if (tall && b <= 256) P.passes = 1;
  P.split = tall;  // (square b <= 128 as well before the early R_kk release, R24: C2 7.15 -> 7.08 ms fused)
  // pipelined panel dependency (R31; the executor compiles it only for b <= 128) and per-slice
  // panel dependencies (R32): for the panel-chain-bound b <= 128 grids (C2); measured same-box,
  // the per-slice dependencies cost C3 0.3% and C4 0.5% (their dispatch order)
  P.pipe = b <= 128;
  P.slicedep = false;  // (C2: 6.749 vs 6.756 ms without; C3 +0.3%, C4 +0.5% with)
  // Reflector-panel groups (R22): square grids with b >= 256 group the updates of each panel in
  // the first half of the steps by default (measured same-box: C3 199.8 -> 198.6 ms, DRAM reads
  // 226 -> 127 GB; C5 -0.2%; C2 (+3%) and the tall-skinny C4 (+0.4%) keep the plain
  // critical-path order); TQR_FLAG_LOCALITY groups them in the first three quarters on every
  // grid (C3: 113 GB of reads, +1.1%)
  if (b >= 256 && !tall) { P.group = 3; P.gtail = 0.5; }
  // Per-edge handoff term of the bottom-level priority (R10): 4 us fits the b >= 256 grids; on
  // the panel-chain-bound b <= 128 grids a large term (the bottom level then counts chain hops)
  // raises the panel chain's priority: C2 6.85 -> 6.46 ms same-box (C3 / C4 unchanged or worse
  // with large terms, profiles/r02_lat_sweep.txt)
  if (b <= 128) P.lat = 200000.0;
  if (locality) { P.group = 3; P.gtail = 0.75; }
  if (const char* e = getenv("TQR_DEV_PASSES")) P.passes = std::max(1, atoi(e));   // development knobs
  if (const char* e = getenv("TQR_DEV_SPLIT")) P.split = atoi(e) != 0;
  if (const char* e = getenv("TQR_DEV_RW")) P.rwm = atoi(e);
  if (const char* e = getenv("TQR_DEV_PRIO")) P.prio = atoi(e);
  if (const char* e = getenv("TQR_DEV_LAT")) P.lat = atof(e);
  if (const char* e = getenv("TQR_DEV_ORM_PRIO")) P.orm_prio = atoi(e);
  if (const char* e = getenv("TQR_DEV_BLQ")) P.blq = atof(e);
  if (const char* e = getenv("TQR_DEV_GROUP")) P.group = atoi(e);
  if (const char* e = getenv("TQR_DEV_EARLY")) P.early = atoi(e) != 0;
  if (const char* e = getenv("TQR_DEV_PIPE")) P.pipe = atoi(e) != 0;
  if (const char* e = getenv("TQR_DEV_SLICEDEP")) P.slicedep = atoi(e) != 0;
  {
    const int w = exec_slice(b, s, P.rwm);  // one register pass
    P.nsl = (int)((b + w - 1) / w);
    if (P.nsl % P.passes != 0) P.passes = 1;
  }
  if (const char* e = getenv("TQR_DEV_FINE")) P.fine = atoi(e);
  return P;
}

static int64_t qloc_of(const tqr_plan* P, int r) {
  return P->real ? (r < P->q ? (P->q - r + P->G - 1) / P->G : 0) : P->q;
}

static tqr_status upload(const Sched& s, const std::vector<int>& ranks, DevSched& d) {
  d.d_tasks.assign(ranks.size(), nullptr);
  d.ntasks.assign(ranks.size(), 0);
  for (size_t li = 0; li < ranks.size(); ++li) {
    const auto& v = s.rec[ranks[li]];
    CU(cudaMalloc(&d.d_tasks[li], v.size() * sizeof(int) + 16));
    if (!v.empty()) CU(cudaMemcpy(d.d_tasks[li], v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
    d.ntasks[li] = (int)(v.size() / TASK_INTS);
  }
  return TQR_OK;
}

static void free_sched(DevSched& d) {
  for (int* t : d.d_tasks)
    if (t) cudaFree(t);
  d.d_tasks.clear();
}

static std::vector<int> local_ranks(const tqr_plan* P) {
  std::vector<int> v;
  if (P->emulate)
    for (int r = 0; r < P->G; ++r) v.push_back(r);
  else
    v.push_back(P->me);
  return v;
}

// Counter generation: counters are never reset; each call waits for / publishes base + v,
// base = gen * (p + 2) > every value of the previous call.
static tqr_status next_base(tqr_plan* P, int* base) {
  const int64_t step = P->p + 2;
  if ((int64_t)(P->gen + 2) * step >= (int64_t)INT32_MAX) {
    if (P->real) {
      g_err = "counter generations exhausted (re-create the plan)";
      return TQR_ERR_UNSUPPORTED;
    }
    for (int r = 0; r < MAX_RANKS; ++r)
      if (P->ctr[r] && (P->emulate || r == P->me))
        CU(cudaMemsetAsync(P->ctr[r], 0, sizeof(int) * (size_t)std::max(1, P->nctr_max), P->st));
    if (P->d_octr) CU(cudaMemsetAsync(P->d_octr, 0, sizeof(int) * (size_t)P->nloc * P->octr_n, P->st));
    P->gen = 0;
  }
  P->gen++;
  *base = (int)(P->gen * step);
  return TQR_OK;
}

// ctr_local (multi-rank apply-Q): rank-local counter arrays replacing the symmetric ones,
// one per local rank, indexed like local_ranks(P)
static tqr_status run(tqr_plan* P, const DevSched& d, double* A, double* T, double* Bt, void* work, bool trace,
                      int* const* ctr_local = nullptr) {
  int total = 0;
  for (int n : d.ntasks) total += n;
  if (total == 0) return TQR_OK;
  int base = 0;
  tqr_status stx = next_base(P, &base);
  if (stx != TQR_OK) return stx;
  const int nl = (int)d.d_tasks.size();
  CU(cudaMemsetAsync(P->d_ticket, 0, sizeof(int) * MAX_RANKS, P->st));
  ExecArgs a;
  std::memset(&a, 0, sizeof(a));
  a.nloc = nl;
  a.nranks = P->G;
  a.p = (int)P->p;
  a.base = base;
  a.sys = P->real ? 1 : 0;
  a.nctr = P->nctr_max;
  a.qcols = (int)std::max<int64_t>(qloc_of(P, P->me), Bt ? (int64_t)(1 << 30) : 0);  // Bt width unknown here
  a.nsl = P->nsl;
  a.phases = P->d_phases;
  if (P->G == 1) {
    a.Yp[0] = reinterpret_cast<double*>(work);
    a.Tp[0] = a.Yp[0] + (size_t)P->h * P->p * P->q * P->prm.b * P->prm.b;
    a.ctr[0] = P->d_ctr1;
  } else {
    for (int r = 0; r < P->G; ++r) {
      a.Yp[r] = P->Yp[r];
      a.Tp[r] = P->Tp[r];
      a.ctr[r] = P->ctr[r];
    }
  }
  if (trace) {
    if (P->trace_cap < total) {
      if (P->d_trace) cudaFree(P->d_trace);
      CU(cudaMalloc(&P->d_trace, sizeof(unsigned long long) * 4 * (size_t)total));
      P->trace_cap = total;
    }
    P->trace_off.assign(nl, 0);
    for (int li = 1; li < nl; ++li) P->trace_off[li] = P->trace_off[li - 1] + d.ntasks[li - 1];
    P->trace_valid = true;
  }
  const std::vector<int> lr = local_ranks(P);
  if (ctr_local) {
    for (int li = 0; li < nl; ++li) a.ctr[P->G == 1 ? 0 : lr[li]] = ctr_local[li];
    a.nctr = P->octr_n;  // (TQR_CHECKS bounds: the rank-local apply-Q counter arrays)
  }
  for (int li = 0; li < nl; ++li) {
    RankLocal& R = a.loc[li];
    R.tasks = d.d_tasks[li];
    R.ntasks = d.ntasks[li];
    R.rank = P->G == 1 ? 0 : lr[li];
    R.ticket = P->d_ticket + li;
    R.ctr = a.ctr[R.rank];
    R.A = A;
    R.T = T;
    R.Bt = Bt;
    R.trace = trace ? P->d_trace + 4 * P->trace_off[li] : nullptr;
  }
  if (P->real) CU(launch_rank_barrier(P->arrive, P->G, P->me, P->gen, P->st));
  const int grid = std::max(nl, std::min(P->workers, std::max(1, total)));
  if (P->h > 1)
    CU(launch_exec_tall(a, grid, P->st));
  else
    CU(launch_exec(P->prm.b, P->prm.s, d.mode, P->rwm, a, grid, P->st));
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

static void destroy_plan(tqr_plan* P) {
  free_sched(P->fact);
  for (auto& kv : P->orm) free_sched(kv.second);
  for (int r = 0; r < MAX_RANKS; ++r) {
    if (P->sym_peer[r]) cudaIpcCloseMemHandle(P->sym_peer[r]);
    if (P->sym_own[r]) cudaFree(P->sym_own[r]);
  }
  if (P->d_ctr1) cudaFree(P->d_ctr1);
  if (P->d_octr) cudaFree(P->d_octr);
  if (P->d_units) cudaFree(P->d_units);
  if (P->d_ticket) cudaFree(P->d_ticket);
  if (P->d_trace) cudaFree(P->d_trace);
  delete P;
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
  if (p->nranks < 1 || p->nranks > MAX_RANKS) return bad_arg(7, "nranks outside [1, 8]");
  if (p->rank < 0 || p->rank >= p->nranks) return bad_arg(8, "rank outside [0, nranks)");
  const bool emulate = (p->flags & TQR_FLAG_EMULATE_RANKS) != 0 && p->nranks > 1;
  if (emulate && p->rank != 0) return bad_arg(8, "emulated multi-rank plans run every rank: rank must be 0");
  if (!exec_supported(p->b, p->s)) {
    g_err = "no kernel instance for this (b, s)";
    return TQR_ERR_UNSUPPORTED;
  }
  const bool tall = (p->flags & TQR_FLAG_TALL_TILES) != 0;
  if (tall && (p->b != 256 || p->s != 32 || p->nranks != 1)) {
    g_err = "TQR_FLAG_TALL_TILES is built for b = 256, s = 32 on one rank";
    return TQR_ERR_UNSUPPORTED;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || p->device < 0 || p->device >= ndev)
    return bad_arg(5, "device ordinal not available");
  DevGuard dg_(p->device);
  if (dg_.err != cudaSuccess) return cuda_fail(dg_.err, "cudaSetDevice");
  tqr_plan* P = new tqr_plan();
  P->prm = *p;
  P->p = (p->m + p->b - 1) / p->b;
  P->q = (p->n + p->b - 1) / p->b;
  P->K = std::min(P->p, P->q);
  P->G = p->nranks;
  P->me = p->rank;
  P->emulate = emulate;
  P->real = P->G > 1 && !emulate;
  P->nloc = emulate ? P->G : 1;
  {
    const Policy pol = make_policy(P->p, P->q, p->b, p->s, tall, (p->flags & TQR_FLAG_LOCALITY) != 0);
    P->rwm = pol.rwm; P->passes = pol.passes; P->nsl = pol.nsl; P->fine = pol.fine; P->split = pol.split;
    P->early = pol.early; P->group = pol.group; P->prio = pol.prio; P->orm_prio = pol.orm_prio; P->lat = pol.lat;
    P->blq = pol.blq;
    P->pipe = pol.pipe;
    P->slicedep = pol.slicedep;
    P->h = pol.h;
    P->gtail = pol.gtail;
  }
  P->st = (cudaStream_t)p->stream;
  P->workers = tall ? exec_max_ctas_tall(p->device) : exec_max_ctas(p->b, p->s, P->rwm, p->device);
  if (P->workers < P->nloc) {
    destroy_plan(P);
    g_err = "executor does not fit on this device";
    return TQR_ERR_UNSUPPORTED;
  }
  if ((int64_t)P->K * P->q * P->nsl + P->K >= (1 << 24)) {
    destroy_plan(P);
    g_err = "problem too large for 24-bit counter indices";
    return TQR_ERR_UNSUPPORTED;
  }
  // worker pools: emulation splits this device's CTAs c -> rank c % G; real ranks each own a GPU
  std::vector<int> workers(P->G, P->workers);
  if (emulate)
    for (int r = 0; r < P->G; ++r) workers[r] = P->workers / P->G + (r < P->workers % P->G ? 1 : 0);
  Sched s;
  build_factor_sched(P->p, P->q, p->b, p->s, P->nsl, workers, P->real, P->split, s, P->prio, P->lat, P->rwm, P->blq, P->group, P->passes, P->fine,
                     P->early, 0.0, P->pipe, P->slicedep, P->h, P->gtail);
  if (!s.topo_ok) {
    destroy_plan(P);
    g_err = "internal: schedule is not topological";
    return TQR_ERR_UNSUPPORTED;
  }
  for (int c : s.nctr) P->nctr_max = std::max(P->nctr_max, c);
  tqr_status st = upload(s, local_ranks(P), P->fact);
  if (st != TQR_OK) { destroy_plan(P); return st; }
  if (cudaMalloc(&P->d_ticket, sizeof(int) * MAX_RANKS) != cudaSuccess) { destroy_plan(P); return TQR_ERR_OOM; }
  if (P->h > 1) {  // units whose output T blocks form_t completes: (k, k, 1) and every TSQRT unit
    std::vector<int> u;
    for (int64_t k = 0; k < P->K; ++k) {
      u.insert(u.end(), {(int)k, (int)k, 1});
      for (int64_t i = k + 1; i < P->p; i += P->h)
        u.insert(u.end(), {(int)i, (int)k, (int)(std::min<int64_t>(P->p, i + P->h) - i)});
    }
    P->nunits = (int)(u.size() / 3);
    if (cudaMalloc(&P->d_units, sizeof(int) * u.size()) != cudaSuccess) { destroy_plan(P); return TQR_ERR_OOM; }
    CU(cudaMemcpy(P->d_units, u.data(), sizeof(int) * u.size(), cudaMemcpyHostToDevice));
  }
  if (P->G == 1) {
    if (cudaMalloc(&P->d_ctr1, sizeof(int) * (size_t)std::max(1, P->nctr_max)) != cudaSuccess) {
      destroy_plan(P);
      return TQR_ERR_OOM;
    }
    CU(cudaMemset(P->d_ctr1, 0, sizeof(int) * (size_t)std::max(1, P->nctr_max)));
  } else {
    // symmetric per-rank buffer: counters | arrive | Yp (p*K tiles) | Tp (p*K slots)
    const size_t b = p->b, sb = p->s;
    SymLayout& L = P->lay;
    L.ctr_off = 0;
    L.arrive_off = ((sizeof(int) * (size_t)P->nctr_max + 255) / 256) * 256;
    L.yp_off = L.arrive_off + 256;
    L.tp_off = L.yp_off + (size_t)P->p * P->K * b * b * sizeof(double);
    L.bytes = L.tp_off + (size_t)P->p * P->K * sb * b * sizeof(double);
    for (int r : local_ranks(P)) {
      if (cudaMalloc(&P->sym_own[r], L.bytes) != cudaSuccess) { destroy_plan(P); return TQR_ERR_OOM; }
      CU(cudaMemset(P->sym_own[r], 0, L.yp_off));
      char* base = (char*)P->sym_own[r];
      P->ctr[r] = (int*)(base + L.ctr_off);
      P->arrive[r] = (int*)(base + L.arrive_off);
      P->Yp[r] = (double*)(base + L.yp_off);
      P->Tp[r] = (double*)(base + L.tp_off);
    }
    P->connected = emulate;
  }
  *out = P;
  return TQR_OK;
}

tqr_status tqr_plan_destroy(tqr_plan* P) {
  if (!P) return bad_arg(1, "plan is NULL");
  GUARD(P);
  destroy_plan(P);
  return TQR_OK;
}

// ---- real multi-GPU: peer-memory connection (CUDA IPC over NVLink / NVSwitch) ----------------
struct IpcBlob {
  char magic[8];
  int32_t rank, nranks;
  uint64_t bytes;
  int64_t m, n;
  int32_t b, s;
  cudaIpcMemHandle_t h;
};
static_assert(sizeof(IpcBlob) <= TQR_IPC_BLOB_BYTES, "blob size");

tqr_status tqr_comm_export(tqr_plan* P, void* blob) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!blob) return bad_arg(2, "blob is NULL");
  if (!P->real) {
    g_err = "tqr_comm_export: only multi-rank plans without TQR_FLAG_EMULATE_RANKS exchange peer memory";
    return TQR_ERR_UNSUPPORTED;
  }
  IpcBlob x;
  std::memset(&x, 0, sizeof(x));
  std::memcpy(x.magic, "TQRIPC1", 8);
  x.rank = P->me;
  x.nranks = P->G;
  x.bytes = P->lay.bytes;
  x.m = P->prm.m; x.n = P->prm.n; x.b = P->prm.b; x.s = P->prm.s;
  GUARD(P);
  CU(cudaIpcGetMemHandle(&x.h, P->sym_own[P->me]));
  std::memset(blob, 0, TQR_IPC_BLOB_BYTES);
  std::memcpy(blob, &x, sizeof(x));
  return TQR_OK;
}

tqr_status tqr_comm_connect(tqr_plan* P, const void* blobs) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!blobs) return bad_arg(2, "blobs is NULL");
  if (!P->real) {
    g_err = "tqr_comm_connect: not a real multi-rank plan";
    return TQR_ERR_UNSUPPORTED;
  }
  if (P->connected) return TQR_OK;
  GUARD(P);
  for (int g = 0; g < P->G; ++g) {
    IpcBlob x;
    std::memcpy(&x, (const char*)blobs + (size_t)g * TQR_IPC_BLOB_BYTES, sizeof(x));
    if (std::memcmp(x.magic, "TQRIPC1", 8) != 0 || x.rank != g || x.nranks != P->G || x.bytes != P->lay.bytes ||
        x.m != P->prm.m || x.n != P->prm.n || x.b != P->prm.b || x.s != P->prm.s)
      return bad_arg(2, "blob of some rank does not match this plan (order blobs by rank)");
    if (g == P->me) continue;
    void* ptr = nullptr;
    CU(cudaIpcOpenMemHandle(&ptr, x.h, cudaIpcMemLazyEnablePeerAccess));
    P->sym_peer[g] = ptr;
    char* base = (char*)ptr;
    P->ctr[g] = (int*)(base + P->lay.ctr_off);
    P->arrive[g] = (int*)(base + P->lay.arrive_off);
    P->Yp[g] = (double*)(base + P->lay.yp_off);
    P->Tp[g] = (double*)(base + P->lay.tp_off);
  }
  P->connected = true;
  return TQR_OK;
}

// ping slots: 8 ints right after the 8 arrive flags (same 256-byte block)
static int* ping_of(int* arrive) { return arrive ? arrive + MAX_RANKS : nullptr; }

tqr_status tqr_comm_ping(tqr_plan* P, int32_t magic) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!P->real || !P->connected) {
    g_err = "tqr_comm_ping: needs a connected real multi-rank plan";
    return TQR_ERR_UNSUPPORTED;
  }
  GUARD(P);
  int* pings[MAX_RANKS] = {};
  for (int g = 0; g < P->G; ++g) pings[g] = ping_of(P->arrive[g]);
  CU(launch_ping(pings, P->G, P->me, magic, P->st));
  CU(cudaStreamSynchronize(P->st));
  return TQR_OK;
}

tqr_status tqr_comm_flags(tqr_plan* P, int32_t* out) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!out) return bad_arg(2, "out is NULL");
  if (!P->real) {
    g_err = "tqr_comm_flags: needs a real multi-rank plan";
    return TQR_ERR_UNSUPPORTED;
  }
  CU(cudaMemcpy(out, ping_of(P->arrive[P->me]), sizeof(int32_t) * P->G, cudaMemcpyDeviceToHost));
  return TQR_OK;
}

tqr_status tqr_tiles_size(const tqr_plan* P, size_t* a, size_t* t) {
  if (!P) return bad_arg(1, "plan is NULL");
  const size_t b = (size_t)P->prm.b, s = (size_t)P->prm.s;
  const size_t ql = (size_t)qloc_of(P, P->me);
  if (a) *a = (size_t)P->p * ql * b * b;
  if (t) *t = (size_t)P->p * ql * s * b;
  return TQR_OK;
}
static size_t work_bytes(const tqr_plan* P) {
  if (P->G > 1) return 0;  // multi-rank plans own their (peer-visible) workspace
  const size_t b = (size_t)P->prm.b, s = (size_t)P->prm.s;
  return ((size_t)P->h * P->p * P->q * b * b + (size_t)P->p * P->q * s * b) * sizeof(double);
}
tqr_status tqr_workspace_size(const tqr_plan* P, size_t* bytes) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (bytes) *bytes = work_bytes(P);
  return TQR_OK;
}

static void colmap(const tqr_plan* P, int* cstride, int* coff) {
  *cstride = P->real ? P->G : 1;
  *coff = P->real ? P->me : 0;
}

tqr_status tqr_pack(tqr_plan* P, const double* A, int64_t lda, double* At) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!A) return bad_arg(2, "A is NULL");
  if (lda < P->prm.m) return bad_arg(3, "lda < m");
  if (!At) return bad_arg(4, "At is NULL");
  ALIGNED(A, 2);
  ALIGNED(At, 4);
  GUARD(P);
  int cs, co;
  colmap(P, &cs, &co);
  CU(launch_pack(A, lda, At, P->prm.m, P->prm.n, P->prm.b, P->p, qloc_of(P, P->me), cs, co, P->st));
  return TQR_OK;
}
tqr_status tqr_unpack(tqr_plan* P, const double* At, double* A, int64_t lda) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!At) return bad_arg(2, "At is NULL");
  if (!A) return bad_arg(3, "A is NULL");
  if (lda < P->prm.m) return bad_arg(4, "lda < m");
  ALIGNED(At, 2);
  ALIGNED(A, 3);
  GUARD(P);
  int cs, co;
  colmap(P, &cs, &co);
  CU(launch_unpack(At, A, lda, P->prm.m, P->prm.n, P->prm.b, P->p, qloc_of(P, P->me), cs, co, P->st));
  return TQR_OK;
}
tqr_status tqr_get_r(tqr_plan* P, const double* At, double* R, int64_t ldr) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!At) return bad_arg(2, "At is NULL");
  if (!R) return bad_arg(3, "R is NULL");
  if (ldr < std::min(P->prm.m, P->prm.n)) return bad_arg(4, "ldr < min(m, n)");
  ALIGNED(At, 2);
  ALIGNED(R, 3);
  GUARD(P);
  int cs, co;
  colmap(P, &cs, &co);
  CU(launch_get_r(At, R, ldr, P->prm.m, P->prm.n, P->prm.b, P->p, qloc_of(P, P->me), cs, co, P->st));
  return TQR_OK;
}

tqr_status tqr_geqrf(tqr_plan* P, double* At, double* T, void* work) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!At) return bad_arg(2, "At is NULL");
  if (!T) return bad_arg(3, "T is NULL");
  if (!work && P->G == 1) return bad_arg(4, "work is NULL (tqr_workspace_size bytes required)");
  ALIGNED(At, 2);
  ALIGNED(T, 3);
  ALIGNED(work, 4);
  GUARD(P);
  if (P->real && !P->connected) {
    g_err = "multi-rank plan not connected (tqr_comm_export / tqr_comm_connect)";
    return TQR_ERR_UNSUPPORTED;
  }
  size_t tsz = 0;
  tqr_tiles_size(P, nullptr, &tsz);
  if (tsz) CU(cudaMemsetAsync(T, 0, tsz * sizeof(double), P->st));
  tqr_status st = run(P, P->fact, At, T, nullptr, work, (P->prm.flags & TQR_FLAG_TRACE) != 0);
  if (st != TQR_OK) return st;
  if (P->h > 1) {  // the tall-unit executor factors with 16-column internal blocks (R16, R30)
    CU(launch_form_t_tall(At, T, P->d_units, P->nunits, (int)P->p, P->st));
  } else if (exec_inner(P->prm.b, P->prm.s) != P->prm.s) {
    int cs, co;
    colmap(P, &cs, &co);
    if (P->emulate || P->G == 1)
      CU(launch_form_t(At, T, P->prm.b, P->prm.s, P->p, P->q, 1, 0, P->st));
    else
      CU(launch_form_t(At, T, P->prm.b, P->prm.s, P->p, qloc_of(P, P->me), cs, co, P->st));
  }
  return TQR_OK;
}

// tile columns of an m x nrhs tile-major B held by this process (real multi-rank: its own)
static int64_t qb_local(const tqr_plan* P, int64_t nrhs) {
  const int64_t qb = (nrhs + P->prm.b - 1) / P->prm.b;
  if (!P->real) return qb;
  return P->me < qb ? (qb - P->me + P->G - 1) / P->G : 0;
}

static tqr_status orm_sched(tqr_plan* P, bool trans, int64_t nrhs, DevSched** out, bool form_q = false) {
  auto key = std::make_pair(trans ? 1 : (form_q ? 2 : 0), nrhs);
  auto it = P->orm.find(key);
  if (it == P->orm.end()) {
    const int64_t qb = (nrhs + P->prm.b - 1) / P->prm.b;
    if ((int64_t)P->K * qb * P->nsl >= (1 << 24)) {
      g_err = "nrhs too large for 24-bit counter indices";
      return TQR_ERR_UNSUPPORTED;
    }
    // worker pools as for the factorization (emulation splits this device's CTAs by rank)
    std::vector<int> workers(P->G, P->workers);
    if (P->emulate)
      for (int r = 0; r < P->G; ++r) workers[r] = P->workers / P->G + (r < P->workers % P->G ? 1 : 0);
    Sched s;
    build_orm_sched(P->p, P->q, qb, P->prm.b, P->prm.s, P->nsl, trans, workers, P->real, s, form_q, P->orm_prio,
                    P->lat, P->rwm, P->passes);
    if (!s.topo_ok) {
      g_err = "internal: apply-Q schedule is not topological";
      return TQR_ERR_UNSUPPORTED;
    }
    DevSched d;
    d.mode = trans ? 1 : 2;
    for (int r : local_ranks(P)) d.nctr = std::max(d.nctr, s.nctr[r]);
    if (P->G == 1 && d.nctr > P->nctr_max) {
      // grow the single-rank counter array (fresh zeros; the generation base stays valid)
      int* nc = nullptr;
      CU(cudaMalloc(&nc, sizeof(int) * (size_t)d.nctr));
      CU(cudaMemset(nc, 0, sizeof(int) * (size_t)d.nctr));
      CU(cudaStreamSynchronize(P->st));
      cudaFree(P->d_ctr1);
      P->d_ctr1 = nc;
      P->nctr_max = d.nctr;
    }
    if (P->G > 1 && d.nctr > P->octr_n) {  // rank-local apply-Q counters (never touched by peers)
      int* nc = nullptr;
      CU(cudaMalloc(&nc, sizeof(int) * (size_t)P->nloc * d.nctr));
      CU(cudaMemset(nc, 0, sizeof(int) * (size_t)P->nloc * d.nctr));
      CU(cudaStreamSynchronize(P->st));
      if (P->d_octr) cudaFree(P->d_octr);
  if (P->d_units) cudaFree(P->d_units);
      P->d_octr = nc;
      P->octr_n = d.nctr;
    }
    tqr_status st = upload(s, local_ranks(P), d);
    if (st != TQR_OK) return st;
    it = P->orm.emplace(key, d).first;
  }
  *out = &it->second;
  return TQR_OK;
}

// Packed reflector panels of the factors (At, T) into the workspace(s) the apply-Q tasks
// stream from.  1 GPU: the caller's `work`.  Emulated ranks: every rank's workspace (global
// At / T).  Real multi-rank: each rank packs the tile columns k it owns into EVERY rank's
// workspace over NVLink peer stores -- the only exchange of apply-Q -- between two
// device-side rank barriers (nobody still reads the old panels; nobody reads before all
// ranks' panels have landed, the second barrier being run()'s entry barrier).
static tqr_status stage_factors(tqr_plan* P, const double* At, const double* T, void* work) {
  const int b = P->prm.b, s = P->prm.s;
  if (P->G == 1) {
    double* Yp = reinterpret_cast<double*>(work);
    double* Tp = Yp + (size_t)P->p * P->q * b * b;
    CU(launch_pack_factors(At, T, &Yp, &Tp, 1, b, s, P->p, P->K, P->q, 1, 0, false, P->st));
    return TQR_OK;
  }
  if (P->emulate) {
    CU(launch_pack_factors(At, T, P->Yp, P->Tp, P->G, b, s, P->p, P->K, P->q, 1, 0, false, P->st));
    return TQR_OK;
  }
  int base = 0;
  tqr_status st = next_base(P, &base);
  if (st != TQR_OK) return st;
  CU(launch_rank_barrier(P->arrive, P->G, P->me, P->gen, P->st));
  CU(launch_pack_factors(At, T, P->Yp, P->Tp, P->G, b, s, P->p, P->K, qloc_of(P, P->me), P->G, P->me, true, P->st));
  return TQR_OK;
}

static tqr_status ormqr_impl(tqr_plan* P, char trans, const double* At, const double* T, double* Bt, int64_t nrhs,
                             void* work, bool form_q) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (trans != 'T' && trans != 'N' && trans != 't' && trans != 'n') return bad_arg(2, "trans must be 'T' or 'N'");
  if (!At) return bad_arg(3, "At is NULL");
  if (!T) return bad_arg(4, "T is NULL");
  if (!Bt) return bad_arg(5, "Bt is NULL");
  if (nrhs < 1) return bad_arg(6, "nrhs < 1");
  if (!work && P->G == 1) return bad_arg(7, "work is NULL (tqr_workspace_size bytes required)");
  ALIGNED(At, 3);
  ALIGNED(T, 4);
  ALIGNED(Bt, 5);
  ALIGNED(work, 7);
  GUARD(P);
  if (P->real && !P->connected) {
    g_err = "multi-rank plan not connected (tqr_comm_export / tqr_comm_connect)";
    return TQR_ERR_UNSUPPORTED;
  }
  if (P->h > 1) {
    g_err = "apply-Q / form-Q are not built for TQR_FLAG_TALL_TILES plans";
    return TQR_ERR_UNSUPPORTED;
  }
  DevSched* d = nullptr;
  tqr_status st = orm_sched(P, trans == 'T' || trans == 't', nrhs, &d, form_q);
  if (st != TQR_OK) return st;
  st = stage_factors(P, At, T, work);
  if (st != TQR_OK) return st;
  if (P->G == 1) return run(P, *d, const_cast<double*>(At), const_cast<double*>(T), Bt, work, false);
  int* ctrs[MAX_RANKS] = {};
  for (int li = 0; li < P->nloc; ++li) ctrs[li] = P->d_octr + (size_t)li * P->octr_n;
  return run(P, *d, const_cast<double*>(At), const_cast<double*>(T), Bt, work, false, ctrs);
}

tqr_status tqr_ormqr(tqr_plan* P, char trans, const double* At, const double* T, double* Bt, int64_t nrhs,
                     void* work) {
  return ormqr_impl(P, trans, At, T, Bt, nrhs, work, false);
}

tqr_status tqr_orgqr(tqr_plan* P, const double* At, const double* T, int64_t k, double* Qt, void* work) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!At) return bad_arg(2, "At is NULL");
  if (!T) return bad_arg(3, "T is NULL");
  if (k < 1 || k > P->prm.m) return bad_arg(4, "k outside [1, m]");
  if (!Qt) return bad_arg(5, "Qt is NULL");
  if (!work && P->G == 1) return bad_arg(6, "work is NULL (tqr_workspace_size bytes required)");
  ALIGNED(At, 2);
  ALIGNED(T, 3);
  ALIGNED(Qt, 5);
  ALIGNED(work, 6);
  GUARD(P);
  int cs, co;
  colmap(P, &cs, &co);
  CU(launch_eye_tiles(Qt, P->prm.m, k, P->prm.b, P->p, qb_local(P, k), cs, co, P->st));
  return ormqr_impl(P, 'N', At, T, Qt, k, work, true);
}

tqr_status tqr_sync(tqr_plan* P) {
  if (!P) return bad_arg(1, "plan is NULL");
  GUARD(P);
  CU(cudaStreamSynchronize(P->st));
  CU(cudaGetLastError());
  return TQR_OK;
}

static tqr_status inspect(int64_t p, int64_t q, int32_t nslice, int32_t workers, int32_t nranks, Sched& s,
                          int h = 1) {
  g_badarg = 0;
  if (p < 1) return bad_arg(1, "p < 1");
  if (q < 1) return bad_arg(2, "q < 1");
  if (nslice < 1) return bad_arg(3, "nslice < 1");
  if (workers < 1) return bad_arg(4, "workers < 1");
  if (nranks < 1 || nranks > MAX_RANKS) return bad_arg(5, "nranks outside [1, 8]");
  // both panel forms, both priorities and every task-granularity policy are exercised by the
  // inspected shapes
  build_factor_sched(p, q, 64 * nslice, 32 * nslice, nslice, std::vector<int>(nranks, workers), nranks > 1,
                     (p + q) % 2 == 0, s, p % 2 == 0 ? PRIO_BLEVEL : PRIO_CLASS, 4000.0, 128, 0.0, false,
                     nslice % 2 == 0 ? 2 : 1, (int)(q % 3), (p + 2 * q) % 3 != 0, 0.0, (p + q) % 3 != 1, true, h);
  if (!s.topo_ok) {
    g_err = "schedule is not a topological order";
    return TQR_ERR_UNSUPPORTED;
  }
  return TQR_OK;
}

tqr_status tqr_schedule_inspect(int64_t p, int64_t q, int32_t nslice, int32_t workers, int64_t counts[4],
                                int64_t* n_edges) {
  Sched s;
  tqr_status st = inspect(p, q, nslice, workers, 1, s);
  if (counts)
    for (int c = 0; c < 4; ++c) counts[c] = s.counts[c];
  if (n_edges) *n_edges = s.nedges;
  return st;
}

tqr_status tqr_schedule_records(int64_t p, int64_t q, int32_t nslice, int32_t workers, int32_t nranks, int32_t rank,
                                int32_t* rec, int64_t cap, int64_t* n, int32_t* nctr) {
  return tqr_schedule_records_h(p, q, nslice, workers, nranks, rank, 1, rec, cap, n, nctr);
}

tqr_status tqr_schedule_records_h(int64_t p, int64_t q, int32_t nslice, int32_t workers, int32_t nranks,
                                  int32_t rank, int32_t h, int32_t* rec, int64_t cap, int64_t* n, int32_t* nctr) {
  if (rank < 0 || rank >= nranks) return bad_arg(6, "rank outside [0, nranks)");
  if (h < 1 || h > 4) return bad_arg(7, "h outside [1, 4]");
  if (!n) return bad_arg(10, "n is NULL");
  Sched s;
  tqr_status st = inspect(p, q, nslice, workers, nranks, s, h);
  if (st != TQR_OK) return st;
  const auto& v = s.rec[rank];
  *n = (int64_t)(v.size() / TASK_INTS);
  if (nctr) *nctr = s.nctr[rank];
  if (rec) std::memcpy(rec, v.data(), sizeof(int32_t) * (size_t)std::min<int64_t>(cap, *n) * TASK_INTS);
  return TQR_OK;
}

tqr_status tqr_schedule_records_policy(int64_t m, int64_t n, int32_t b, int32_t s, int32_t nranks, int32_t rank,
                                       int32_t workers, uint32_t flags, int32_t* rec, int64_t cap, int64_t* ntask,
                                       int32_t* nctr, int32_t info[4]) {
  g_badarg = 0;
  if (m < 1) return bad_arg(1, "m < 1");
  if (n < 1) return bad_arg(2, "n < 1");
  if (!exec_supported(b, s)) return bad_arg(3, "no kernel instance for (b, s)");
  if (nranks < 1 || nranks > MAX_RANKS) return bad_arg(5, "nranks outside [1, 8]");
  if (rank < 0 || rank >= nranks) return bad_arg(6, "rank outside [0, nranks)");
  if (workers < 1) return bad_arg(7, "workers < 1");
  const bool tall = (flags & TQR_FLAG_TALL_TILES) != 0;
  if (tall && (b != 256 || s != 32 || nranks != 1)) return bad_arg(8, "TQR_FLAG_TALL_TILES: b = 256, s = 32, one rank");
  if (!ntask) return bad_arg(11, "ntask is NULL");
  const int64_t p = (m + b - 1) / b, q = (n + b - 1) / b;
  const Policy pol = make_policy(p, q, b, s, tall, (flags & TQR_FLAG_LOCALITY) != 0);
  Sched sc;
  build_factor_sched(p, q, b, s, pol.nsl, std::vector<int>(nranks, workers), nranks > 1, pol.split, sc, pol.prio,
                     pol.lat, pol.rwm, pol.blq, pol.group, pol.passes, pol.fine, pol.early, 0.0, pol.pipe,
                     pol.slicedep, pol.h, pol.gtail);
  if (!sc.topo_ok) {
    g_err = "schedule is not a topological order";
    return TQR_ERR_UNSUPPORTED;
  }
  const auto& v = sc.rec[rank];
  *ntask = (int64_t)(v.size() / TASK_INTS);
  if (nctr) *nctr = sc.nctr[rank];
  if (info) {
    info[0] = b / s;                                                  // panel blocks per tile
    info[1] = tall ? exec_slice_tall() : exec_slice(b, s, pol.rwm);   // columns per register pass
    info[2] = pol.nsl;
    info[3] = pol.h;
  }
  if (rec) std::memcpy(rec, v.data(), sizeof(int32_t) * (size_t)std::min<int64_t>(cap, *ntask) * TASK_INTS);
  return TQR_OK;
}

tqr_status tqr_schedule_model(int64_t m, int64_t n, int32_t b, int32_t s, int32_t nranks, int32_t workers,
                              double remote_ns, double* makespan_ns, double* busy) {
  g_badarg = 0;
  if (m < 1) return bad_arg(1, "m < 1");
  if (n < 1) return bad_arg(2, "n < 1");
  if (!exec_supported(b, s)) return bad_arg(3, "no kernel instance for (b, s)");
  if (nranks < 1 || nranks > MAX_RANKS) return bad_arg(5, "nranks outside [1, 8]");
  if (workers < 1) return bad_arg(6, "workers < 1");
  if (remote_ns < 0.0) return bad_arg(7, "remote_ns < 0");
  if (!makespan_ns) return bad_arg(8, "makespan_ns is NULL");
  const int64_t p = (m + b - 1) / b, q = (n + b - 1) / b;
  const Policy pol = make_policy(p, q, b, s);
  Sched sc;
  build_factor_sched(p, q, b, s, pol.nsl, std::vector<int>(nranks, workers), nranks > 1, pol.split, sc, pol.prio,
                     pol.lat, pol.rwm, pol.blq, pol.group, pol.passes, pol.fine, pol.early, remote_ns, pol.pipe,
                     pol.slicedep, 1, pol.gtail);
  if (!sc.topo_ok) {
    g_err = "schedule is not a topological order";
    return TQR_ERR_UNSUPPORTED;
  }
  *makespan_ns = sc.makespan;
  if (busy) *busy = sc.busy;
  return TQR_OK;
}

tqr_status tqr_plan_records(tqr_plan* P, int32_t local, int32_t* rec, int64_t cap, int64_t* n) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (local < 0 || local >= (int32_t)P->fact.d_tasks.size()) return bad_arg(2, "local rank index out of range");
  if (!rec && cap > 0) return bad_arg(3, "rec is NULL");
  if (!n) return bad_arg(5, "n is NULL");
  *n = P->fact.ntasks[local];
  const int64_t c = std::min<int64_t>(cap, *n);
  if (c > 0)
    CU(cudaMemcpy(rec, P->fact.d_tasks[local], sizeof(int32_t) * (size_t)c * TASK_INTS, cudaMemcpyDeviceToHost));
  return TQR_OK;
}

tqr_status tqr_plan_info(const tqr_plan* P, int32_t info[16]) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!info) return bad_arg(2, "info is NULL");
  info[0] = P->rwm;
  info[1] = P->passes;
  info[2] = P->nsl;
  info[3] = P->split ? 1 : 0;
  info[4] = P->early ? 1 : 0;
  info[5] = P->workers;
  info[6] = P->prio;
  info[7] = P->fine;
  info[8] = exec_inner(P->prm.b, P->prm.s);
  info[9] = P->G;
  info[10] = P->nloc;
  info[11] = P->h > 1 ? exec_slice_tall() : exec_slice(P->prm.b, P->prm.s, P->rwm);
  info[12] = P->h;
  info[13] = info[14] = info[15] = 0;
  if (P->h > 1) info[8] = 16;  // (the tall-unit executor's internal block)
  return TQR_OK;
}

tqr_status tqr_trace_fetch(tqr_plan* P, int64_t* rec, int64_t cap, int64_t* n) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (!rec && cap > 0) return bad_arg(2, "rec is NULL");
  if (!n) return bad_arg(4, "n is NULL");
  *n = 0;
  if (!P->d_trace || !P->trace_valid) return TQR_OK;
  CU(cudaStreamSynchronize(P->st));
  int64_t w = 0;
  for (size_t li = 0; li < P->fact.d_tasks.size() && w < cap; ++li) {
    const int64_t cnt = std::min<int64_t>(cap - w, P->fact.ntasks[li]);
    std::vector<unsigned long long> raw((size_t)cnt * 4);
    std::vector<int> tasks((size_t)cnt * TASK_INTS);
    CU(cudaMemcpy(raw.data(), P->d_trace + 4 * P->trace_off[li], raw.size() * sizeof(unsigned long long),
                  cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(tasks.data(), P->fact.d_tasks[li], tasks.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < cnt; ++r) {
      const int* t = &tasks[(size_t)r * TASK_INTS];
      int64_t* o = rec + (w + r) * 8;
      o[0] = t[0]; o[1] = t[1]; o[2] = t[2]; o[3] = t[3];
      o[4] = (int64_t)(t[4] & 0xFFFF) | ((int64_t)(t[14] & 0xFF) << 16);  // slice | task flags << 16
      o[5] = (int64_t)(raw[r * 4] >> 32);
      o[6] = (int64_t)raw[r * 4 + 2];
      o[7] = (int64_t)raw[r * 4 + 3];
    }
    w += cnt;
  }
  *n = w;
  return TQR_OK;
}

tqr_status tqr_profile_tasks(tqr_plan* P, int32_t kind, int64_t count, double* At, double* T, void* work) {
  if (!P) return bad_arg(1, "plan is NULL");
  if (kind < 0 || kind > 9) return bad_arg(2, "kind outside [0, 9]");
  if (count < 1 || count > (1 << 24)) return bad_arg(3, "count outside [1, 2^24]");
  if (!At) return bad_arg(4, "At is NULL");
  if (!T) return bad_arg(5, "T is NULL");
  if (!work) return bad_arg(6, "work is NULL");
  if (P->p < 2 || P->q < 2 || P->G > 1 || P->h > 1) {
    g_err = "profiling needs a single-rank square-tile plan with p >= 2 and q >= 2";
    return TQR_ERR_UNSUPPORTED;
  }
  GUARD(P);
  Sched s;
  s.rec.assign(1, std::vector<int>((size_t)count * TASK_INTS, 0));
  for (int64_t t = 0; t < count; ++t) {
    int* q = &s.rec[0][(size_t)t * TASK_INTS];
    const int i = 1 + (int)(t % (P->p - 1));
    const int j = 1 + (int)((t / (P->p - 1)) % (P->q - 1));
    // kinds 8 / 9: the factor part F(k,i,l) alone of a GEQRT / TSQRT (R21), block
    // l = t mod (b/s): the panel column loop, Gram, T_l and the V/Y/T stores, no left-looking apply
    const bool fpart = kind >= 8;
    if (fpart) kind -= 8;
    q[0] = kind;
    q[1] = kind == 0 ? (int)(t % P->K) : 0;
    const bool lkind = kind == 2 || kind == 4 || kind == 6;
    q[2] = (kind == 0 || lkind) ? q[1] : i;
    q[3] = (kind == 0 || kind == 1) ? q[1] : j;
    if (kind == 1) {  // TSQRT: distinct tiles (i, k), i > k, as long as there are enough of them
      const int64_t np_ = std::max<int64_t>(1, (int64_t)P->K * P->p - P->K * (P->K + 1) / 2);
      int64_t x = (fpart ? t / (P->prm.b / P->prm.s) : t) % np_;
      int kk = 0;
      while (x >= P->p - kk - 1) { x -= P->p - kk - 1; ++kk; }
      q[1] = kk; q[2] = kk + 1 + (int)x; q[3] = kk;
    }
    // -1: a panel task over the whole tile; update tasks: first register pass, P->passes passes
    q[4] = (kind == 0 || kind == 1) ? (fpart ? (int)(t % (P->prm.b / P->prm.s)) : -1)
                                    : (int)(t % (P->nsl / P->passes)) * P->passes;
    q[14] = fpart ? 4 : 0;
    q[15] = P->passes | (1 << 8);
    if (fpart) kind += 8;
    q[5] = 0;
    q[6] = 1;
    q[7] = q[1];
  }
  DevSched d;
  d.mode = (kind >= 6 && kind <= 7) ? 2 : ((kind >= 4 && kind <= 7) ? 1 : 0);
  tqr_status st = upload(s, std::vector<int>{0}, d);
  if (st != TQR_OK) return st;
  st = run(P, d, At, T, At, work, false);
  cudaStreamSynchronize(P->st);
  free_sched(d);
  return st;
}

// Profiling builds (-DTQR_PROFILE_PHASES): attach a device array of 16 int64 phase-cycle
// totals (NULL detaches).
tqr_status tqr_phase_counters(tqr_plan* P, long long* d_counters) {
  if (!P) return bad_arg(1, "plan is NULL");
  P->d_phases = d_counters;
  return TQR_OK;
}

}  // extern "C"
