// tqr_exec.cu -- persistent DAG executor and layout kernels (sm_100a).
//
// The paper runs the tasks of Algorithm 1 out of order on CPU
// threads that pick ready tasks by priority.  Here one persistent
// CTA per SM (co-resident cooperative launch) takes tickets in a host-computed
// topological order (a list schedule by critical-path priority, R10) and waits
// on per-chain monotone progress counters (acquire) before running the task; on
// completion it publishes its counter(s) (release).  Task granularity: GEQRT(k) and
// TSQRT(k,i) run as one single-CTA task per inner block l (fused, or split into an apply
// and a factor part, R21); LARFB and SSRFB tasks cover np register passes of a
// tile's columns (one 8-column group per warp, register resident; R23).
#include <cstdio>

#include "tqr_device.cuh"
#include "tqr_internal.h"

namespace tqr {

// End-of-task publication: __syncthreads, then thread 0 releases the task's counter(s)
// (st.release.gpu: cumulative over the CTA's stores ordered before it by the barrier).
// TQR_RELEASE_FENCE=1 adds an explicit fence.sc.gpu before the release (experiment knob).
// Per-instance features, measured same-box against r01 (tools/ab3.sh):
// the pipelined panel dependency (R31) and the blocked T_l (R26) pay off only where the panel
// chain bounds the factorization (b <= 128, C2: 7.09 -> 6.75 ms); in the b >= 256 instances
// their extra code in the executor costs 0.3-1% (C3, C4), so it is compiled out there.
// TQR_PF_CALL=1 calls the panel column loop instead of inlining it in the b = 256 RW = 128
// instance (the loop itself 58k -> 46k cycles, but C4 0.9% slower overall): off.
#ifndef TQR_PF_CALL
#define TQR_PF_CALL 0
#endif
template <int B>
struct Feat {
  static constexpr bool PIPE = B <= 128;      // pipelined panel dependency (R31)
  static constexpr bool TBLOCKED = B <= 128;  // T_l by 8 x 8 DMMA blocks (R26)
};
#ifndef TQR_PANEL_NEXT  // panel tasks take their successor ticket before factoring (section 5)
#define TQR_PANEL_NEXT 0  // (measured: C2 +1.4%, C4 -0.1%: off)
#endif
#ifndef TQR_RELEASE_FENCE
#define TQR_RELEASE_FENCE 1
#endif

#ifndef TQR_POLL_NS
#define TQR_POLL_NS 200  // back-off between polls of an unresolved dependency counter
#endif

// Optional phase timing (build with -DTQR_PROFILE_PHASES): warp 0 of every CTA accumulates
// clock64 deltas per phase; totals are added to ExecArgs::phases at kernel exit.
#ifdef TQR_PROFILE_PHASES
constexpr int NPH = 16;
__shared__ long long s_ph[NPH];  // per-CTA phase totals (thread 0)
__shared__ long long s_pht;      // thread 0's last mark
#define PH_T0                                 \
  do {                                        \
    if (threadIdx.x == 0) s_pht = clock64();  \
  } while (0)
#define PH_MARK(idx)                          \
  do {                                        \
    if (threadIdx.x == 0) {                   \
      long long ph_n = clock64();             \
      s_ph[idx] += ph_n - s_pht;              \
      s_pht = ph_n;                           \
    }                                         \
  } while (0)
#else
#define PH_T0 do {} while (0)
#define PH_MARK(idx) do {} while (0)
#endif

template <int B, int S, int RWM>
struct Layout {
  using C = Cfg<B, S, RWM>;
  static constexpr int YSZ = B * S;          // one Y buffer (swizzled panel)
  static constexpr int TSZ = S * S;
  // Y0 T0 | Y1 T1: the panel tasks overlay P (ld B+4) on the contiguous (Y1, T1) region
  static constexpr int Y0 = 0, T0 = YSZ, Y1 = YSZ + TSZ, T1 = 2 * YSZ + TSZ;
  static constexpr int LDP = B + 4;
  static_assert(LDP * S <= YSZ + TSZ, "P overlay");
  // W partials (RS > 1): one per warp, double-buffered by block parity -- a warp rewrites a
  // buffer two blocks later, after its partner has passed the next block's exchange barrier,
  // so one named barrier per block suffices (group_apply BAR2 = false)
  static constexpr int XBUF = 2 * YSZ + 2 * TSZ;
  static constexpr int XSZ = C::RS > 1 ? 2 * C::NWARP * C::XW : 0;
  static constexpr int C1S = XBUF + XSZ;          // C1 blocks, 2 buffers x GPS groups
  static constexpr int C1SZ = C::GPS * C::C1W;
  // panel-only scratch (Rb, Z, tau; Rb reused for the plain T_l), aliased onto the partial /
  // C1 buffers, which the panel task uses only in its left-looking phase
  static constexpr int RB = XBUF, ZZ = RB + TSZ, TAU = ZZ + TSZ;
  static constexpr int PANEL_END = TAU + S;
  static constexpr int UPD_END = C1S + 2 * C1SZ;
  // 2 "full" mbarriers (8 B each) + 2 int32 "done" counters
  static constexpr int MBAR = (PANEL_END > UPD_END ? PANEL_END : UPD_END);
  // S mbarriers of the panel column handoff (panel_factor), initialised once per launch
  static constexpr int PMB = MBAR + 4;
  static constexpr int TOTAL = PMB + S;  // doubles
  static constexpr size_t BYTES = (size_t)TOTAL * sizeof(double);
  static_assert(BYTES <= 232448, "shared memory budget");
  static_assert((T0 % 2) == 0 && (Y1 % 2) == 0 && (MBAR % 1) == 0, "16-byte aligned TMA destinations");
};

__device__ __forceinline__ double* tile_ptr(double* base, int i, int j, int p, int B) {
  return base + ((size_t)i + (size_t)j * p) * (size_t)B * B;
}
__device__ __forceinline__ double* tslot_ptr(double* base, int i, int k, int p, int B, int S) {
  return base + ((size_t)i + (size_t)k * p) * (size_t)S * B;
}
// Workspace: packed copies of every reflector panel, written once by the panel
// task that creates it, read by every update task through TMA bulk copies.
//   Yp tile (i,k), panel l: B*S doubles at tile_ptr(Yp, i, k) + l*B*S, swy<B> layout;
//     diagonal tiles hold U_l (0 above the block, unit-lower top block, V below).
//   Tp slot (i,k), block l: S*S doubles at tslot_ptr(Tp, i, k) + l*S*S, swz<S> layout.

// Stage panel l (Y_l: B*S doubles, T_l: S*S) from the packed workspace into buffer `buf`
// with two TMA bulk copies completing on mbarrier full[buf].  One thread.  No proxy fence
// here: the generic-proxy writes of the packed panels are ordered before these async-proxy
// reads by the fence.proxy.async after the dependency acquire (or after panel_block), and a
// buffer refill after generic reads (WAR) needs none.  (A fence here also waited for the
// thread's outstanding acc loads -- 6% of C3 time.)
template <int B, int S, int RWM>
__device__ __forceinline__ void issue_panel(double* sm, const double* Yp, const double* Tp, int l, int buf) {
  using L = Layout<B, S, RWM>;
  constexpr unsigned YB = B * S * 8, TB = S * S * 8;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + L::MBAR);
  mbar_expect_tx(full + buf, YB + TB);
  bulk_g2s(sm + (buf ? L::Y1 : L::Y0), Yp + (size_t)l * B * S, YB, full + buf);
  bulk_g2s(sm + (buf ? L::T1 : L::T0), Tp + (size_t)l * S * S, TB, full + buf);
}

// Update phase shared by every task kind (one inlined copy per executor instance):
// load the column groups [col0, col0 + 8*gact) of tile Ct into registers, then apply the
// nb packed reflector blocks (Yp, Tp) to them -- blocks 0..nb-1 (DESC: nb-1..0) -- each
// as W = [C1] + Y^T C; W <- T^{T|1} W; [C1 -= W]; C -= Y W, with the C1 rows of block l
// taken from tile C1 (nullptr: LARFB / GEQRT type).
// Pipeline: two buffers; blocks 0 and 1 are issued at phase start; the LAST warp to finish
// with a buffer (shared-memory counter) issues its refill two blocks ahead, so there is no
// __syncthreads inside the block loop and every refill overlaps a whole block of math.
// C1 is fetched one block ahead by the group's rpart-0 warp (cp.async).
// `pf(li, nb)` is called by thread 0 once per block (cross-task prefetch hook).
// Pipelined panel dependency (R31): `pp` (not null) points at the panel progress
// counters PF(k, 0..) of the reflectors being applied; internal block l may only be staged
// once PF(k, l / SPO) >= pp_val (SPO internal blocks per output T block); blocks < pp_ready
// are known to be ready.  The thread that stages a block waits for it (acquire + proxy fence);
// block 1, if not ready at phase start, is staged by the last reader of block 0.
struct PanelDep {
  const int* ctr = nullptr;  // PF(k, 0) on this rank (nullptr: every block ready)
  int val = 0;
  int ready = 1 << 30;       // internal blocks known ready
  int spo = 1;               // internal blocks per output block
  bool sys = false;          // a peer GPU publishes the counter
};
__device__ __forceinline__ bool panel_block_ready(const PanelDep& pd, int l) {
  if (l < pd.ready) return true;
  const int* c = pd.ctr + l / pd.spo;
  return (pd.sys ? ld_acquire_sys(c) : ld_acquire(c)) >= pd.val;
}
__device__ __forceinline__ void panel_block_wait(const PanelDep& pd, int l) {
  if (l < pd.ready) return;
  const int* c = pd.ctr + l / pd.spo;
  if ((pd.sys ? ld_acquire_sys(c) : ld_acquire(c)) < pd.val) {
    const unsigned long long t0w = globaltimer();
    while ((pd.sys ? ld_acquire_sys(c) : ld_acquire(c)) < pd.val) {
      __nanosleep(TQR_POLL_NS);
      if (globaltimer() - t0w > 20ull * 1000000000ull) __trap();
    }
  }
  fence_proxy_async();  // the producer's generic stores -> our TMA reads
}

template <int B, int S, int RWM, bool QT, bool DESC, class PF>
__device__ __forceinline__ void update_phase(double* sm, double (&acc)[Cfg<B, S, RWM>::RW / 8][2], const double* Yp,
                                             const double* Tp, int lb0, int nbe, double* C1, const double* Ct,
                                             int col0, int gact, PF&& pf, bool keep = false,
                                             const PanelDep& pd = PanelDep()) {
  // blocks lb0 .. nbe-1 (DESC: nbe-1 .. 0, lb0 must be 0)
  const int nb = nbe - lb0;
  using C = Cfg<B, S, RWM>;
  using L = Layout<B, S, RWM>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gi = warp / C::RS, rpart = warp % C::RS, t0 = rpart * (C::RW / 8);
  const int cg0 = col0 + gi * 8;
  const bool active = gi < gact;
  const bool top_owner = C1 != nullptr && active && rpart == 0;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + L::MBAR);
  int* done = reinterpret_cast<int*>(full + 2);  // done[0], done[1]; done[2]: block 1 deferred
  double* c1s0 = sm + L::C1S + gi * C::C1W;           // C1 buffer for even li
  double* c1s1 = sm + L::C1S + L::C1SZ + gi * C::C1W;  // C1 buffer for odd li
  if (nb > 0 && threadIdx.x == 0) {  // staging first: nothing outstanding to wait for
    mbar_init(full, 1);
    mbar_init(full + 1, 1);
    done[0] = 0;
    done[1] = 0;
    done[2] = 0;
    fence_mbar_init();
    fence_proxy_async();
    issue_panel<B, S, RWM>(sm, Yp, Tp, DESC ? nb - 1 : lb0, 0);  // (block 0: waited by the task)
    if (nb > 1) {
      if constexpr (Feat<B>::PIPE) {
        if (DESC || panel_block_ready(pd, lb0 + 1)) {
          fence_proxy_async();
          issue_panel<B, S, RWM>(sm, Yp, Tp, DESC ? nb - 2 : lb0 + 1, 1);
        } else {
          done[2] = 1;  // staged by the last reader of block 0
        }
      } else {
        issue_panel<B, S, RWM>(sm, Yp, Tp, DESC ? nb - 2 : lb0 + 1, 1);
      }
    }
  }
  if (active) {
    load_cols<B, C::RW>(acc, Ct, cg0, t0, keep);
  } else {
    // a def on every path: otherwise acc stays live (for the compiler) across the panel code
    // of a panel task, which then rematerialises its indices (RW = 256: +40% instructions
    // in the column loop)
#pragma unroll
    for (int t = 0; t < C::RW / 8; ++t) { acc[t][0] = 0.0; acc[t][1] = 0.0; }
  }
  if (nb <= 0) return;
  if (top_owner) c1_fetch<B, S>(c1s0, C1, (DESC ? nb - 1 : lb0) * S, cg0);
  __syncthreads();
  PH_MARK(14);
  for (int li = 0; li < nb; ++li) {
    const int l = DESC ? nb - 1 - li : lb0 + li;
    const int buf = li & 1;
    if (top_owner) {
      cp_async_wait<0>();  // this block's C1
      __syncwarp();
      if (li + 1 < nb) c1_fetch<B, S>(buf ? c1s0 : c1s1, C1, (DESC ? l - 1 : l + 1) * S, cg0);
    }
    if (li == 0) PH_MARK(15);
    mbar_wait(full + buf, (li >> 1) & 1);
    if (li == 0) PH_MARK(0);
    if (threadIdx.x == 0) pf(li, nb);
    if (active)
      group_apply<B, S, C::RW, C::RS, QT, false>(acc, sm + (buf ? L::Y1 : L::Y0), sm + (buf ? L::T1 : L::T0),
                                                buf ? c1s1 : c1s0, C1, l * S, cg0, t0, gi, rpart,
                                                sm + L::XBUF + (li & 1) * (C::NWARP * C::XW) + gi * C::RS * C::XW);
    __syncwarp();
if constexpr (Feat<B>::PIPE) {
    if (lane == 0 && (li + 2 < nb || (li == 0 && nb > 1))) {
      if (atomicAdd(done + buf, 1) == C::NWARP - 1) {  // last reader of this buffer: refill it
        done[buf] = 0;
        if (li == 0 && done[2]) {  // deferred block 1 (pipelined panel dependency)
          done[2] = 0;
          panel_block_wait(pd, l + 1);
          issue_panel<B, S, RWM>(sm, Yp, Tp, l + 1, 1);
        }
        if (li + 2 < nb) {
          if (!DESC) panel_block_wait(pd, l + 2);
          issue_panel<B, S, RWM>(sm, Yp, Tp, DESC ? l - 2 : l + 2, buf);
        }
      }
    }
} else {
    if (lane == 0 && li + 2 < nb) {
      if (atomicAdd(done + buf, 1) == C::NWARP - 1) {  // last reader of this buffer: refill it
        done[buf] = 0;
        issue_panel<B, S, RWM>(sm, Yp, Tp, DESC ? l - 2 : l + 2, buf);
      }
    }
}
  }
  __syncthreads();  // every staged buffer consumed before anyone reuses the staging space
}

// ---------------------------------------------------------------------------------------
// Panel block l of GEQRT(k) (ts = false) or TSQRT(k,i) (PAPER.md:404-428,
// ts = true).  The panel task is left-looking inside the tile: for block l the update
// phase has already applied this task's blocks 0..l-1 to the block's columns (acc); here
// they go to shared memory, the block is factored (panel_factor), V / R / T are written
// out and the packed Y_l / T_l are published for blocks l+1.. and for every update task.
// TSQRT reads and writes only the upper triangle of A(k,k).
// ---------------------------------------------------------------------------------------
// The panel column loop as a called function, register-allocated on its own instead of inside
// the whole executor: used by the tall-skinny b = 256 instance (RW = 128), whose inlined loop
// measured 1880 clk per column vs 1440 called (tools/prof_tasks.py, r02 phase profiles); the
// other instances keep it inlined (called: 3-9% slower there).
template <int B, int S, int NW, int LDP, bool TS>
__device__ __noinline__ void panel_factor_call(double* P, int c0, double* Rb, double* tau, unsigned long long* pmb,
                                               unsigned parity) {
  panel_factor<B, S, NW, LDP>(P, c0, Rb, tau, TS, pmb, parity);
}

template <int B, int S, int SO, int RWM, bool ts>
__device__ __forceinline__ void panel_block(double* sm, const double (&acc)[Cfg<B, S, RWM>::RW / 8][2],
                                            double* Akk, double* Ab, double* Tslot, const ExecArgs& a, size_t yoff,
                                            size_t toff, int l, bool more, int rlo, unsigned& pf_gen,
                                            int* pr_ctr, int pr_val) {
  using C = Cfg<B, S, RWM>;
  using L = Layout<B, S, RWM>;
  constexpr int LDP = L::LDP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gi = warp / C::RS, rpart = warp % C::RS, t0 = rpart * (C::RW / 8);
  const int c0 = l * S;
  double* P = sm + L::Y1;
  double* Ys = sm + L::Y0;
  double* Rb = sm + L::RB;
  double* Tp = sm + L::RB;  // after Rb is written back
  double* Z = sm + L::ZZ;
  double* tau = sm + L::TAU;
  // block columns -> P (shared memory); GEQRT: rows above the block are final R -- written
  // back only from row rlo: rows above the task's first block belong to the apply part,
  // which the next tile's apply part (TSQRT A(k,k+1,.)) may already be updating (R21)
  if (gi < S / 8) {
    const int col = 8 * gi + (lane >> 2);
#pragma unroll
    for (int t = 0; t < C::RW / 8; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * (t0 + t) + 2 * (lane & 3) + h;
        if (ts || r >= c0) P[r + col * LDP] = acc[t][h];
        else if (r >= rlo) __stcg(Ab + (size_t)(c0 + col) * B + r, acc[t][h]);
      }
  }
  if (ts)
    for (int e = tid; e < S * S; e += C::NT) {
      const int r = e % S, c = e / S;
      Rb[e] = (r <= c) ? __ldcg(Akk + (size_t)(c0 + c) * B + c0 + r) : 0.0;
    }
  __syncthreads();
  PH_MARK(8);
  if constexpr (TQR_PF_CALL && B == 256 && RWM == 128)
    panel_factor_call<B, S, C::NWARP, LDP, ts>(P, c0, Rb, tau, reinterpret_cast<unsigned long long*>(sm + L::PMB),
                                               pf_gen & 1);
  else
    panel_factor<B, S, C::NWARP, LDP>(P, c0, Rb, tau, ts, reinterpret_cast<unsigned long long*>(sm + L::PMB),
                                      pf_gen & 1);
  ++pf_gen;  // every call completes each column mbarrier once
  PH_MARK(9);
  // V / R out, packed Y_l (Ys), Gram -> T_l, packed T_l
  for (int e = tid; e < B * S; e += C::NT) {
    const int r = e % B, c = e / B;
    double y = 0.0;
    if (ts) {
      y = P[r + c * LDP];
      __stcg(Ab + (size_t)(c0 + c) * B + r, y);
    } else if (r >= c0) {
      const double v = P[r + c * LDP];
      __stcg(Ab + (size_t)(c0 + c) * B + r, v);
      y = (r - c0 == c) ? 1.0 : (r - c0 > c ? v : 0.0);
    }
    Ys[swy<B>(r, c)] = y;
  }
  if (ts)
    for (int e = tid; e < S * S; e += C::NT) {
      const int r = e % S, c = e / S;
      if (r <= c) __stcg(Akk + (size_t)(c0 + c) * B + c0 + r, Rb[e]);
    }
  __syncthreads();
  // early release (R24): R_kk's rows of this block are final (V/R out above), which
  // is all the next tile's factor part of this block reads -- it need not wait for the Gram,
  // T and packed-panel work below
  if (pr_ctr && !more && threadIdx.x == 0) {
    __threadfence();
    st_release(pr_ctr, pr_val);
  }
  PH_MARK(10);
  gram_upper<B, S, C::NWARP>(Ys, Z);
  __syncthreads();
  PH_MARK(11);
  // T_l by 8 x 8 blocks on warps 0 .. S/8 - 1 (scratch: the P overlay, no longer read)
  constexpr int NTW = S / 8 < C::NWARP ? S / 8 : C::NWARP;
  // the packed Y_l into every rank's workspace (the V broadcast of SURVEY 8(e), fused into
  // the panel task: peer stores over NVLink on a multi-GPU job, local stores otherwise).  One
  // flat loop over (rank, 16-byte chunk), so the stores to all G ranks are in flight together.
  auto store_y = [&](int t0, int nt) __attribute__((always_inline)) {
    constexpr int NV2 = B * S / 2;
    const double2* ys2 = reinterpret_cast<const double2*>(Ys);
    for (int e = tid - t0; e < a.nranks * NV2; e += nt) {
      const int g = e / NV2, x = e - g * NV2;
      __stcg(reinterpret_cast<double2*>(a.Yp[g] + yoff + (size_t)l * B * S) + x, ys2[x]);
    }
  };
if constexpr (Feat<B>::TBLOCKED) {
  if (warp < NTW) build_t_blocked<S>(Tp, tau, Z, P, 14);
  else store_y(32 * NTW, C::NT - 32 * NTW);  // meanwhile, on the other warps
  __syncthreads();
  if constexpr (NTW == C::NWARP) {
    store_y(0, C::NT);
    __syncthreads();
  }
} else {
  constexpr int NTW1 = (S + 31) / 32;
  if (warp < NTW1) build_t<S>(Tp, tau, Z);
  else store_y(32 * NTW1, C::NT - 32 * NTW1);
  __syncthreads();
}
  PH_MARK(12);
  // output slot: T_L (SO x SO) in columns [L*SO, L*SO+SO); this SI-block is its diagonal
  // block m (the off-diagonal blocks of SO > SI are formed after the factorization)
  constexpr int RB_ = SO / S;
  const int Lo = l / RB_, mo = (l % RB_) * S;
  for (int e = tid; e < S * S; e += C::NT) {
    const int r = e % S, c = e / S;
    __stcg(Tslot + ((size_t)Lo * SO + mo + c) * SO + mo + r, Tp[e]);
  }
  for (int e = tid; e < a.nranks * S * S; e += C::NT) {  // packed T_l to every rank, flat
    const int g = e / (S * S), x = e - g * (S * S);
    const int r = x % S, c = x / S;
    __stcg(a.Tp[g] + toff + (size_t)l * S * S + swz<S>(r, c), Tp[x]);
  }
  if (a.sys) __threadfence_system();  // peer stores ordered before the counter release
  // packed panels (generic stores) -> TMA reads of the next block of THIS task; a later task
  // orders them with its own fence after acquiring the panel counter
  if (more) fence_proxy_async();
  __syncthreads();
  PH_MARK(13);
}

// L2 prefetch of the inputs of a (not yet started) task record q: the tile column slice it
// updates (+ its C1 slice), or the tile a panel task factors, and its first two packed
// reflector blocks.  Safe before the task's dependencies hold (L2 is coherent).
template <int B, int S, int SO, int RWM, int MODE>
__device__ __forceinline__ void prefetch_task(const int* q, const RankLocal& R, const double* Yme, int p) {
  using C = Cfg<B, S, RWM>;
  const int kind = q[0], k = q[1], i = q[2], j = q[3], sl = q[4], kc = q[7];
  if (MODE == 0 && (kind == K_G || kind == K_T)) {
    prefetch_l2(tile_ptr(R.A, kind == K_T ? i : k, kc, p, B), (unsigned)(B * B * 8));
    return;
  }
  const bool lkind = kind == K_L || kind == K_LQT || kind == K_LQ;
  double* Bt = MODE == 0 ? R.A : R.Bt;
  const size_t off = (size_t)sl * C::SLICE * B;
  const unsigned bytes = (unsigned)(C::SLICE * B * 8);  // the first pass's columns
  prefetch_l2(tile_ptr(Bt, lkind ? k : i, j, p, B) + off, bytes, lkind);       // C2 (LARFB: the C1 row tile)
  if (!lkind) prefetch_l2(tile_ptr(Bt, k, j, p, B) + off, bytes, true);          // C1: kept in L2
  const int vrow = lkind ? k : i;
  const double* Y = Yme + ((size_t)vrow + (size_t)k * p) * (size_t)B * B;
  constexpr int NL = B / S;
  const int l0 = MODE == 2 ? (NL >= 2 ? NL - 2 : 0) : 0;
  prefetch_l2(Y + (size_t)l0 * B * S, (unsigned)((NL >= 2 ? 2 : 1) * B * S * 8), true);
}

// ---------------------------------------------------------------------------------------
// Persistent executor.
// ---------------------------------------------------------------------------------------
// MODE 0: factorization; MODE 1: apply Q^T; MODE 2: apply Q.  No device-function calls:
// every task kind runs through ONE inlined update phase (plus the panel block for GEQRT /
// TSQRT), so ptxas allocates the column-group accumulators once, without spills.
template <int B, int SO, int MODE, int RWM>
__global__ void __launch_bounds__(Cfg<B, Inner<B, SO>::SI, RWM>::NT, 1) exec_kernel(const __grid_constant__ ExecArgs a) {
  constexpr int S = Inner<B, SO>::SI;  // internal inner block (== SO up to b = 256)
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_task[TASK_INTS];
  __shared__ int s_ticket;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const RankLocal& R = a.loc[blockIdx.x % a.nloc];  // the rank this CTA serves
  double* const Yme = a.Yp[R.rank];
  double* const Tme = a.Tp[R.rank];
#ifdef TQR_PROFILE_PHASES
  if (tid < NPH) s_ph[tid] = 0;
  __syncthreads();
#endif
  // Cross-task pipelining (thread 0): half-way through the last pass of an update the next
  // ticket is taken, one block later its record is fetched (cp.async), one more block later
  // its input tiles are prefetched into L2, so the next prologue (acc / C1 loads, first
  // TMA) reads from L2 and the dispatch round trips overlap math.  Holding one ticket ahead cannot
  // deadlock: every wait is on a smaller ticket, and the smallest unfinished ticket is running.
  __shared__ __align__(16) int s_next[TASK_INTS];
  __shared__ int s_have;
  // panel column handoff mbarriers (panel_factor): one init per launch, parity by call count
  unsigned pf_gen = 0;
  if (MODE == 0) {
    if (tid < S) mbar_init(reinterpret_cast<unsigned long long*>(sm + Layout<B, S, RWM>::PMB) + tid, 1);
    fence_mbar_init();
    __syncthreads();
  }
  int next_tk = -1, rec_for = -1;  // thread 0
  for (;;) {
    PH_T0;
    if (tid == 0) {
      if (next_tk < 0) next_tk = atomicAdd(R.ticket, 1);
      cp_async_wait<0>();  // a prefetched record has landed
      s_ticket = next_tk;
      s_have = rec_for == next_tk;
      next_tk = -1;
    }
    __syncthreads();
    const int tk = s_ticket;
#ifdef TQR_PROFILE_PHASES
    if (tk >= R.ntasks) {
      if (tid < NPH && a.phases) atomicAdd((unsigned long long*)&a.phases[tid], (unsigned long long)s_ph[tid]);
      return;
    }
#else
    if (tk >= R.ntasks) return;
#endif
    if (tid < TASK_INTS) s_task[tid] = s_have ? s_next[tid] : R.tasks[(size_t)tk * TASK_INTS + tid];
    __syncthreads();
    PH_MARK(1);
    unsigned long long t_grab = 0, t_start = 0;
    if (R.trace && tid == 0) t_grab = globaltimer();
    if (warp == 0) {
#pragma unroll
      for (int d = 0; d < TASK_NDEP; ++d) {
        const int code = s_task[8 + 2 * d], val = a.base + s_task[9 + 2 * d];
        // pipelined panel dependency (record [14] bit 6, R31): dependency 0 names the
        // LAST block's counter PF(k, NPT-1); the task starts on block 0's, PF(k, 0), and waits
        // for each later block just before staging it (update_phase)
        const int pipe = (Feat<B>::PIPE && d == 0 && (s_task[14] & 64)) ? B / SO - 1 : 0;
        const int cnt = (int)((unsigned)code >> 24), idx = (code & 0xFFFFFF) - pipe;
        // system scope only for a counter a peer GPU publishes (record [14] bit 3 + d); the
        // rank-local chains (column counters, apply / early-release parts) stay at gpu scope
        const bool sysd = a.sys && ((s_task[14] >> (3 + d)) & 1);
        for (int x = lane; x < cnt; x += 32) {
          const int* c = R.ctr + idx + x;
          if ((sysd ? ld_acquire_sys(c) : ld_acquire(c)) >= val) continue;
          const unsigned long long t0w = globaltimer();
          while ((sysd ? ld_acquire_sys(c) : ld_acquire(c)) < val) {
            __nanosleep(TQR_POLL_NS);
            // watchdog: a dependency that never resolves is a schedule bug; fail loudly
            if (globaltimer() - t0w > 20ull * 1000000000ull) __trap();
          }
        }
      }
      __syncwarp();
      fence_proxy_async();  // producer data (generic-proxy stores) -> our TMA reads
    }
    __syncthreads();
    PH_MARK(6);
    if (R.trace && tid == 0) t_start = globaltimer();
    const int kind = s_task[0], k = s_task[1], i = s_task[2], j = s_task[3], sl = s_task[4], kc = s_task[7];
#ifdef TQR_CHECKS
    // checked build: every field of the record and every counter range in bounds
    if (tid == 0) {
      bool bad = kind < 0 || kind > 7 || k < 0 || k >= a.p || i < k || i >= a.p || kc < 0 || kc >= a.qcols ||
                 j < 0 || j >= a.qcols || sl < -1 || sl >= (kind >= K_L ? a.nsl : B / SO) ||
                 (kind >= K_L && ((s_task[15] & 0xFF) < 1 || sl + (s_task[15] & 0xFF) > a.nsl)) ||
                 s_task[5] < 0 || s_task[5] + ((s_task[15] >> 8) & 0xFF) > a.nctr || (MODE == 0) != (kind <= K_S);
      for (int d = 0; d < TASK_NDEP; ++d) {
        const int code = s_task[8 + 2 * d], cnt = (int)((unsigned)code >> 24), idx = code & 0xFFFFFF;
        if (cnt && (idx + cnt > a.nctr)) bad = true;
      }
      const int pr = (s_task[14] >> 8) - 1;  // early-release counter of a panel factor part
      if (pr >= a.nctr || (pr >= 0 && !(kind == K_G || kind == K_T))) bad = true;
      if (bad) {
        printf("tqr checked build: bad task record %d: kind %d k %d i %d j %d sl %d kc %d out %d\n", tk, kind, k, i,
               j, sl, kc, s_task[5]);
        __trap();
      }
    }
#endif
    const int p = a.p;
    {
      constexpr int NL = B / S;
      const bool panel = MODE == 0 && (kind == K_G || kind == K_T);
      const bool ts = kind == K_T;
      const bool lkind = kind == K_L || kind == K_LQT || kind == K_LQ;
      double* Bt = MODE == 0 ? R.A : R.Bt;
      double* Akk = tile_ptr(R.A, k, kc, p, B);
      double* Ab = ts ? tile_ptr(R.A, i, kc, p, B) : Akk;  // panel tasks: the tile being factored
      const int vrow = (panel && !ts) || lkind ? k : i;     // tile row of the reflectors applied
      double* Tslot = tslot_ptr(R.T, vrow, kc, p, B, SO);
      // reflector workspace, indexed by the global step k (every rank holds every panel);
      // T slots of SO*B doubles holding the B/S internal S x S blocks
      const size_t yoff = ((size_t)vrow + (size_t)k * p) * (size_t)B * B;
      const size_t toff = ((size_t)vrow + (size_t)k * p) * (size_t)SO * B;
      const double* Ypt = Yme + yoff;
      const double* Tps = Tme + toff;
      // panel task: inner blocks [sub0, sub1) of the tile (one output T block per task, or the
      // whole tile when sl < 0); update task: np register passes from pass sl
      constexpr int SPT = SO / S;  // internal blocks per output T block
      const int sub0 = panel ? (sl < 0 ? 0 : sl * SPT) : 0;
      // update tasks: passes [sl, sl + np) of SLICE columns each (record [15] = np | ocnt << 8)
      const int np = s_task[15] & 0xFF;
      const int nsub = panel ? (sl < 0 ? NL : sub0 + SPT) : np;
      // panel split (R21): flags bit 1 = apply part only (left-looking update of the
      // block columns with this tile's earlier blocks, stored back), bit 2 = factor part only
      const bool a_part = panel && (s_task[14] & 2), f_part = panel && (s_task[14] & 4);
      for (int sub = sub0; sub < nsub; ++sub) {
        double acc[Cfg<B, S, RWM>::RW / 8][2];
        double* C1;
        double* Ct;
        int col0, nb, gact, lb0 = 0;
        if (panel) {
          C1 = ts ? Akk : nullptr;
          Ct = Ab;
          col0 = sub * S;
          nb = a_part ? sub0 : sub;   // A: blocks < sub0; F: this task's blocks [sub0, sub)
          lb0 = f_part ? sub0 : 0;
          gact = S / 8;
        } else {
          C1 = lkind ? nullptr : tile_ptr(Bt, k, j, p, B);
          Ct = lkind ? tile_ptr(Bt, k, j, p, B) : tile_ptr(Bt, i, j, p, B);
          col0 = (sl + sub) * Cfg<B, S, RWM>::SLICE;  // (update tasks: sl >= 0)
          nb = NL;
          gact = (B - col0) / 8 < Cfg<B, S, RWM>::GPS ? (B - col0) / 8 : Cfg<B, S, RWM>::GPS;
        }
        auto pf = [&](int li, int nbb) {
          if (!panel && sub + 1 < nsub && li == nbb / 2) {  // next register pass of this task
            const size_t nxt_off = (size_t)(col0 + Cfg<B, S, RWM>::SLICE) * B;
            prefetch_l2(Ct + nxt_off, (unsigned)(Cfg<B, S, RWM>::SLICE * B * 8), lkind);
            if (C1) prefetch_l2(C1 + nxt_off, (unsigned)(Cfg<B, S, RWM>::SLICE * B * 8), true);
          }
          if (sub != nsub - 1 || nbb < 4) return;  // (nbb: blocks this pass applies)
          const int l0 = nbb / 2;
          if (li == l0) next_tk = atomicAdd(R.ticket, 1);  // next ticket, half a pass early
          if (li == l0 + 1 && next_tk < R.ntasks) {       // its record -> s_next (async)
#pragma unroll
            for (int x = 0; x < TASK_INTS; x += 4)  // 4 x 16 bytes
              cp_async16(s_next + x, R.tasks + (size_t)next_tk * TASK_INTS + x);
            cp_async_commit();
            rec_for = next_tk;
          }
          if (li == l0 + 2 && rec_for == next_tk && next_tk < R.ntasks) {
            cp_async_wait<0>();
            prefetch_task<B, S, SO, RWM, MODE>(s_next, R, Yme, p);
          }
        };
        // L2 policy of the target (section 5): C1 row tiles (LARFB targets) and panel tiles are
        // re-read soon (evict_last); SSRFB C2 slices stream (evict_first) -- TQR_L2HINT builds
        const bool keep = panel || lkind;
        PanelDep pd;
        if (Feat<B>::PIPE && MODE == 0 && !panel && (s_task[14] & 64) && sub == sub0) {
          pd.ctr = R.ctr + (s_task[8] & 0xFFFFFF) - (B / SO - 1);
          pd.val = a.base + s_task[9];
          pd.spo = SO / S;
          pd.sys = a.sys && (s_task[14] & 8);
          pd.ready = pd.spo;  // output block 0: waited for above
          if (panel_block_ready(pd, NL - 1)) pd.ready = NL;  // the whole panel is already done
        }
        update_phase<B, S, RWM, MODE != 2, MODE == 2>(sm, acc, Ypt, Tps, lb0, nb, C1, Ct, col0, gact, pf, keep, pd);
        if (panel) PH_MARK(7); else PH_MARK(4);
        if (TQR_PANEL_NEXT && panel && sub == nsub - 1 && tid == 0 && next_tk < 0) {
          // a panel task's last block: take the next ticket and fetch its record now, so both
          // round trips overlap the factorization (update tasks do this half-way through their
          // last pass); holding it early cannot deadlock (every wait is on a smaller ticket)
          next_tk = atomicAdd(R.ticket, 1);
          if (next_tk < R.ntasks) {
#pragma unroll
            for (int x = 0; x < TASK_INTS; x += 4) cp_async16(s_next + x, R.tasks + (size_t)next_tk * TASK_INTS + x);
            cp_async_commit();
            rec_for = next_tk;
          }
        }
        if (a_part) {
          if (warp / Cfg<B, S, RWM>::RS < gact)
            store_cols<B, Cfg<B, S, RWM>::RW>(acc, Ct, col0 + 8 * (warp / Cfg<B, S, RWM>::RS),
                                         (warp % Cfg<B, S, RWM>::RS) * (Cfg<B, S, RWM>::RW / 8), true);
        } else if (panel) {
          // TS as a template argument: each flavour is register-allocated on its own
          const int rlo = f_part ? sub0 * S : 0;
          const int pr = (s_task[14] >> 8) - 1;  // early-release counter (or -1)
          int* const prc = pr >= 0 ? R.ctr + pr : nullptr;
          const int prv = a.base + s_task[6];
          if (ts)
            panel_block<B, S, SO, RWM, true>(sm, acc, Akk, Ab, Tslot, a, yoff, toff, sub, sub + 1 < nsub, rlo, pf_gen,
                                             prc, prv);
          else
            panel_block<B, S, SO, RWM, false>(sm, acc, Akk, Ab, Tslot, a, yoff, toff, sub, sub + 1 < nsub, rlo, pf_gen,
                                              prc, prv);
        } else if (warp / Cfg<B, S, RWM>::RS < gact) {
          store_cols<B, Cfg<B, S, RWM>::RW>(acc, Ct, col0 + 8 * (warp / Cfg<B, S, RWM>::RS),
                                       (warp % Cfg<B, S, RWM>::RS) * (Cfg<B, S, RWM>::RW / 8), keep);
        }
        if (!panel) PH_MARK(5);
      }
    }
    __syncthreads();
    PH_MARK(2);
    if (tid == 0) {
#if TQR_RELEASE_FENCE
      __threadfence();
#endif
      fence_proxy_async();
      const int oidx = s_task[5], oval = a.base + s_task[6];
      if ((s_task[14] >> 8) != 0 && s_task[6] > 1) {
        // Ordered publication of an early-releasing factor part (R24): the next
        // tile's factor part of this block may have started on our early release and may
        // finish first; PF(k,l) must still advance v-1 -> v -> v+1 (a consumer of PF >= v
        // reads this task's Y_l / T_l), so wait for the previous tile's publication.  That
        // task is past its own early release and waits on nothing: no deadlock.
        const int* c = R.ctr + oidx;  // (this rank's copy, published by this rank: gpu scope)
        if (ld_acquire(c) < oval - 1) {
          const unsigned long long t0w = globaltimer();
          while (ld_acquire(c) < oval - 1) {
            __nanosleep(TQR_POLL_NS);
            if (globaltimer() - t0w > 20ull * 1000000000ull) __trap();
          }
        }
      }
      if ((s_task[14] & 1) && a.nranks > 1) {
        // panel progress: release on every rank (the V/T tiles it covers are already there)
        if (a.sys) {
          __threadfence_system();
          for (int g = 0; g < a.nranks; ++g) st_release_sys(a.ctr[g] + oidx, oval);
        } else {
          for (int g = 0; g < a.nranks; ++g) st_release(a.ctr[g] + oidx, oval);
        }
      } else {
        const int ocnt = (s_task[15] >> 8) & 0xFF;  // update tasks: one counter per pass
        for (int x = 0; x < (ocnt > 0 ? ocnt : 1); ++x) st_release(R.ctr + oidx + x, oval);
      }
      PH_MARK(3);
      if (R.trace) {
        unsigned long long* tr = R.trace + (size_t)tk * 4;
        tr[0] = ((unsigned long long)smid() << 32) | (unsigned)tk;
        tr[1] = t_grab;
        tr[2] = t_start;
        tr[3] = globaltimer();
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// Tall-unit executor (R30; "2b x b blocks"): the tile rows below
// the diagonal are grouped in units of two b x b tiles (the last unit of a step may be one
// tile); TSQRT / SSRFB work on the (2b) x b stack of a unit.  b = 256, s = 32 only: a unit is
// 512 rows, so the executor runs the 512-row register configuration of the b = 512 instance
// (RW = 256 rows per warp, two warps per column group, SI = 16 internal blocks: a 512 x 16
// packed panel, double-buffered, fits shared memory) on 256-column tiles whose leading
// dimension is 256: warp rpart of a column group holds tile i0 + rpart.  GEQRT / LARFB tasks
// (the diagonal tile) are units whose second tile is absent (zero rows, not stored).
// Records: [2] = the unit's first tile row i0, [14] bit 7 = the unit has a second tile.
// Workspace: the packed panels of unit (i0, k) at (i0 + k p) * 2 b^2 doubles (TR x SI per
// internal block), T blocks as for square tiles.
// ---------------------------------------------------------------------------------------
namespace tall {
constexpr int TB = 256, TR = 512, SO = 32, S = Inner<TR, SO>::SI, RWM = 256;
using C = Cfg<TR, S, RWM>;
using L = Layout<TR, S, RWM>;
static_assert(S == 16 && C::RS == 2 && C::RW == TB, "tall-unit configuration");
constexpr int NL = TB / S;   // internal blocks per tile (16)
constexpr int SPT = SO / S;  // internal blocks per output T block (2)

__device__ __forceinline__ double* unit_panel(double* base, int i0, int k, int p) {
  return base + ((size_t)i0 + (size_t)k * p) * 2 * (size_t)TB * TB;
}

// update phase on a unit: warp rpart of column group gi holds tile Ct[rpart] (nullptr: absent
// rows -- zeros, still part of the group's W exchange)
template <class PF>
__device__ __forceinline__ void update_phase(double* sm, double (&acc)[C::RW / 8][2], const double* Yp,
                                             const double* Tp, int lb0, int nbe, double* C1, double* const (&Ct)[2],
                                             int col0, int gact, PF&& pf) {
  const int nb = nbe - lb0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gi = warp / C::RS, rpart = warp % C::RS, t0 = rpart * (C::RW / 8);
  const int cg0 = col0 + gi * 8;
  const bool active = gi < gact;
  const bool rows = active && Ct[rpart] != nullptr;
  const bool top_owner = C1 != nullptr && active && rpart == 0;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + L::MBAR);
  int* done = reinterpret_cast<int*>(full + 2);
  double* c1s0 = sm + L::C1S + gi * C::C1W;
  double* c1s1 = sm + L::C1S + L::C1SZ + gi * C::C1W;
  if (nb > 0 && threadIdx.x == 0) {
    mbar_init(full, 1);
    mbar_init(full + 1, 1);
    done[0] = 0;
    done[1] = 0;
    fence_mbar_init();
    fence_proxy_async();
    issue_panel<TR, S, RWM>(sm, Yp, Tp, lb0, 0);
    if (nb > 1) issue_panel<TR, S, RWM>(sm, Yp, Tp, lb0 + 1, 1);
  }
  if (rows) {
    load_cols<TB, C::RW>(acc, Ct[rpart], cg0, 0);
  } else {
#pragma unroll
    for (int t = 0; t < C::RW / 8; ++t) { acc[t][0] = 0.0; acc[t][1] = 0.0; }
  }
  if (nb <= 0) return;
  if (top_owner) c1_fetch<TB, S>(c1s0, C1, lb0 * S, cg0);
  __syncthreads();
  for (int li = 0; li < nb; ++li) {
    const int l = lb0 + li;
    const int buf = li & 1;
    if (top_owner) {
      cp_async_wait<0>();
      __syncwarp();
      if (li + 1 < nb) c1_fetch<TB, S>(buf ? c1s0 : c1s1, C1, (l + 1) * S, cg0);
    }
    mbar_wait(full + buf, (li >> 1) & 1);
    if (threadIdx.x == 0) pf(li, nb);
    if (active)
      group_apply<TR, S, C::RW, C::RS, true, false, TB>(acc, sm + (buf ? L::Y1 : L::Y0), sm + (buf ? L::T1 : L::T0),
                                                        buf ? c1s1 : c1s0, C1, l * S, cg0, t0, gi, rpart,
                                                        sm + L::XBUF + (li & 1) * (C::NWARP * C::XW) +
                                                            gi * C::RS * C::XW);
    __syncwarp();
    if (lane == 0 && li + 2 < nb) {
      if (atomicAdd(done + buf, 1) == C::NWARP - 1) {
        done[buf] = 0;
        issue_panel<TR, S, RWM>(sm, Yp, Tp, l + 2, buf);
      }
    }
  }
  __syncthreads();
}

// Panel block l of GEQRT(k) (ts = false; Ab = {A(k,k), nullptr}) or TSQRT(k, unit) (ts = true;
// Ab = the unit's tiles): as ::panel_block on the 512-row staged block, V / R written back to
// the unit's tiles, packed Y_l (512 x SI) / T_l to the workspace.
template <bool ts>
__device__ __forceinline__ void panel_block(double* sm, const double (&acc)[C::RW / 8][2], double* Akk,
                                            double* const (&Ab)[2], double* Tslot, double* Yunit, double* Tunit,
                                            int l, bool more, int rlo, unsigned& pf_gen, int* pr_ctr, int pr_val) {
  constexpr int LDP = L::LDP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gi = warp / C::RS, rpart = warp % C::RS, t0 = rpart * (C::RW / 8);
  const int c0 = l * S;
  double* P = sm + L::Y1;
  double* Ys = sm + L::Y0;
  double* Rb = sm + L::RB;
  double* Tp = sm + L::RB;
  double* Z = sm + L::ZZ;
  double* tau = sm + L::TAU;
  if (gi < S / 8) {
    const int col = 8 * gi + (lane >> 2);
#pragma unroll
    for (int t = 0; t < C::RW / 8; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * (t0 + t) + 2 * (lane & 3) + h;  // unit row (rows >= TB: tile 2)
        if (ts || r >= c0) P[r + col * LDP] = acc[t][h];
        else if (r >= rlo) __stcg(Akk + (size_t)(c0 + col) * TB + r, acc[t][h]);  // (GEQRT: r < TB)
      }
  }
  if (ts)
    for (int e = tid; e < S * S; e += C::NT) {
      const int r = e % S, c = e / S;
      Rb[e] = (r <= c) ? __ldcg(Akk + (size_t)(c0 + c) * TB + c0 + r) : 0.0;
    }
  __syncthreads();
  panel_factor<TR, S, C::NWARP, LDP>(P, c0, Rb, tau, ts, reinterpret_cast<unsigned long long*>(sm + L::PMB),
                                     pf_gen & 1);
  ++pf_gen;
  for (int e = tid; e < TR * S; e += C::NT) {
    const int r = e % TR, c = e / TR;
    double y = 0.0;
    if (ts) {
      y = P[r + c * LDP];
      double* t = Ab[r / TB];
      if (t) __stcg(t + (size_t)(c0 + c) * TB + r % TB, y);
    } else if (r >= c0 && r < TB) {
      const double v = P[r + c * LDP];
      __stcg(Akk + (size_t)(c0 + c) * TB + r, v);
      y = (r - c0 == c) ? 1.0 : (r - c0 > c ? v : 0.0);
    }
    Ys[swy<TR>(r, c)] = y;
  }
  if (ts)
    for (int e = tid; e < S * S; e += C::NT) {
      const int r = e % S, c = e / S;
      if (r <= c) __stcg(Akk + (size_t)(c0 + c) * TB + c0 + r, Rb[e]);
    }
  __syncthreads();
  if (pr_ctr && !more && threadIdx.x == 0) {  // early release of R_kk's block rows (R24)
    __threadfence();
    st_release(pr_ctr, pr_val);
  }
  gram_upper<TR, S, C::NWARP>(Ys, Z);
  __syncthreads();
  if (warp == 0) {
    build_t<S>(Tp, tau, Z);
  } else {
    const double2* ys2 = reinterpret_cast<const double2*>(Ys);
    for (int e = tid - 32; e < TR * S / 2; e += C::NT - 32)
      __stcg(reinterpret_cast<double2*>(Yunit + (size_t)l * TR * S) + e, ys2[e]);
  }
  __syncthreads();
  const int Lo = l / SPT, mo = (l % SPT) * S;
  for (int e = tid; e < S * S; e += C::NT) {
    const int r = e % S, c = e / S;
    __stcg(Tslot + ((size_t)Lo * SO + mo + c) * SO + mo + r, Tp[e]);
    __stcg(Tunit + (size_t)l * S * S + swz<S>(r, c), Tp[e]);
  }
  if (more) fence_proxy_async();
  __syncthreads();
}

// Persistent executor for tall-unit factorizations (one rank; same ticket / counter protocol
// as ::exec_kernel, including the ordered end-of-task publication of R25).
__global__ void __launch_bounds__(C::NT, 1) exec_kernel(const __grid_constant__ ExecArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_task[TASK_INTS];
  __shared__ int s_ticket;
  __shared__ __align__(16) int s_next[TASK_INTS];
  __shared__ int s_have;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const RankLocal& R = a.loc[0];
  double* const Yme = a.Yp[0];
  double* const Tme = a.Tp[0];
  unsigned pf_gen = 0;
  if (tid < S) mbar_init(reinterpret_cast<unsigned long long*>(sm + L::PMB) + tid, 1);
  fence_mbar_init();
  __syncthreads();
  int next_tk = -1, rec_for = -1;
  const int p = a.p;
  for (;;) {
    if (tid == 0) {
      if (next_tk < 0) next_tk = atomicAdd(R.ticket, 1);
      cp_async_wait<0>();
      s_ticket = next_tk;
      s_have = rec_for == next_tk;
      next_tk = -1;
    }
    __syncthreads();
    const int tk = s_ticket;
    if (tk >= R.ntasks) return;
    if (tid < TASK_INTS) s_task[tid] = s_have ? s_next[tid] : R.tasks[(size_t)tk * TASK_INTS + tid];
    __syncthreads();
    unsigned long long t_grab = 0, t_start = 0;
    if (R.trace && tid == 0) t_grab = globaltimer();
    if (warp == 0) {
#pragma unroll
      for (int d = 0; d < TASK_NDEP; ++d) {
        const int code = s_task[8 + 2 * d], val = a.base + s_task[9 + 2 * d];
        const int cnt = (int)((unsigned)code >> 24), idx = code & 0xFFFFFF;
        for (int x = lane; x < cnt; x += 32) {
          const int* c = R.ctr + idx + x;
          if (ld_acquire(c) >= val) continue;
          const unsigned long long t0w = globaltimer();
          while (ld_acquire(c) < val) {
            __nanosleep(TQR_POLL_NS);
            if (globaltimer() - t0w > 20ull * 1000000000ull) __trap();
          }
        }
      }
      __syncwarp();
      fence_proxy_async();
    }
    __syncthreads();
    if (R.trace && tid == 0) t_start = globaltimer();
    const int kind = s_task[0], k = s_task[1], i0 = s_task[2], j = s_task[3];
    const int sl = s_task[4] & 0xFF, lsub = (s_task[4] >> 8) - 1;  // apply sub-task: output block lsub
    const bool two = (s_task[14] & 128) != 0;
    {
      const bool panel = kind == K_G || kind == K_T;
      const bool ts = kind == K_T;
      const bool lkind = kind == K_L;
      double* Akk = tile_ptr(R.A, k, k, p, TB);
      const int urow = (panel && !ts) || lkind ? k : i0;  // the unit whose reflectors are applied
      double* Tslot = tslot_ptr(R.T, urow, k, p, TB, SO);
      double* Yunit = unit_panel(Yme, urow, k, p);
      double* Tunit = Tme + ((size_t)urow + (size_t)k * p) * (size_t)SO * TB;
      const int sub0 = panel ? sl * SPT : 0;
      const int np = s_task[15] & 0xFF;
      const int nsub = panel ? sub0 + SPT : np;
      const bool a_part = panel && (s_task[14] & 2), f_part = panel && (s_task[14] & 4);
      for (int sub = sub0; sub < nsub; ++sub) {
        double acc[C::RW / 8][2];
        double* C1;
        double* Ct[2];
        int col0, nb, gact, lb0 = 0;
        if (panel) {
          C1 = ts ? Akk : nullptr;
          Ct[0] = ts ? tile_ptr(R.A, i0, k, p, TB) : Akk;
          Ct[1] = ts && two ? tile_ptr(R.A, i0 + 1, k, p, TB) : nullptr;
          col0 = sub * S;
          nb = a_part ? (lsub >= 0 ? (lsub + 1) * SPT : sub0) : sub;  // (apply sub-task: blocks of lsub)
          lb0 = f_part ? sub0 : (lsub >= 0 ? lsub * SPT : 0);
          gact = S / 8;
        } else {
          C1 = lkind ? nullptr : tile_ptr(R.A, k, j, p, TB);
          Ct[0] = lkind ? tile_ptr(R.A, k, j, p, TB) : tile_ptr(R.A, i0, j, p, TB);
          Ct[1] = !lkind && two ? tile_ptr(R.A, i0 + 1, j, p, TB) : nullptr;
          col0 = (sl + sub) * C::SLICE;
          nb = NL;
          gact = (TB - col0) / 8 < C::GPS ? (TB - col0) / 8 : C::GPS;
        }
        auto pf = [&](int li, int nbb) {
          if (sub != nsub - 1 || nbb < 4) return;
          const int l0 = nbb / 2;
          if (li == l0) next_tk = atomicAdd(R.ticket, 1);
          if (li == l0 + 1 && next_tk < R.ntasks) {
#pragma unroll
            for (int x = 0; x < TASK_INTS; x += 4) cp_async16(s_next + x, R.tasks + (size_t)next_tk * TASK_INTS + x);
            cp_async_commit();
            rec_for = next_tk;
          }
          if (li == l0 + 2 && rec_for == next_tk && next_tk < R.ntasks) {
            cp_async_wait<0>();
            const int* q = s_next;
            const int qk = q[1], qi = q[2], qj = q[3];
            if (q[0] == K_S) {  // the next update's C2 / C1 column slices and first reflector blocks
              const size_t off = (size_t)q[4] * C::SLICE * TB;
              prefetch_l2(tile_ptr(R.A, qi, qj, p, TB) + off, (unsigned)(C::SLICE * TB * 8));
              if (q[14] & 128) prefetch_l2(tile_ptr(R.A, qi + 1, qj, p, TB) + off, (unsigned)(C::SLICE * TB * 8));
              prefetch_l2(tile_ptr(R.A, qk, qj, p, TB) + off, (unsigned)(C::SLICE * TB * 8));
              prefetch_l2(unit_panel(Yme, qi, qk, p), (unsigned)(2 * TR * S * 8));
            }
          }
        };
        update_phase(sm, acc, Yunit, Tunit, lb0, nb, C1, Ct, col0, gact, pf);
        if (TQR_PANEL_NEXT && panel && sub == nsub - 1 && tid == 0 && next_tk < 0) {  // (as ::exec_kernel)
          next_tk = atomicAdd(R.ticket, 1);
          if (next_tk < R.ntasks) {
#pragma unroll
            for (int x = 0; x < TASK_INTS; x += 4) cp_async16(s_next + x, R.tasks + (size_t)next_tk * TASK_INTS + x);
            cp_async_commit();
            rec_for = next_tk;
          }
        }
        if (a_part) {
          const int gi = warp / C::RS, rp = warp % C::RS;
          if (gi < gact && Ct[rp]) {
            if (!ts && lsub >= 0) {
              // a GEQRT apply sub-task changes only rows >= lsub*SO of block l's columns (U is zero
              // above): store only those -- the TSQRT sub-applies of unit 0 already update R_kk's
              // rows of earlier blocks in these columns while this sub-task runs
              const int rmin = lsub * SO;
              double2* col = reinterpret_cast<double2*>(Ct[rp] + (size_t)(col0 + 8 * gi + (lane >> 2)) * TB +
                                                        2 * (lane & 3));
#pragma unroll
              for (int t = 0; t < C::RW / 8; ++t)
                if (8 * t >= rmin) __stcg(col + 4 * t, make_double2(acc[t][0], acc[t][1]));
            } else {
              store_cols<TB, C::RW>(acc, Ct[rp], col0 + 8 * gi, 0);
            }
          }
        } else if (panel) {
          const int rlo = f_part ? sub0 * S : 0;
          const int pr = (s_task[14] >> 8) - 1;
          int* const prc = pr >= 0 ? R.ctr + pr : nullptr;
          const int prv = a.base + s_task[6];
          if (ts)
            panel_block<true>(sm, acc, Akk, Ct, Tslot, Yunit, Tunit, sub, sub + 1 < nsub, rlo, pf_gen, prc, prv);
          else
            panel_block<false>(sm, acc, Akk, Ct, Tslot, Yunit, Tunit, sub, sub + 1 < nsub, rlo, pf_gen, prc, prv);
        } else {
          const int gi = warp / C::RS, rp = warp % C::RS;
          if (gi < gact && Ct[rp]) store_cols<TB, C::RW>(acc, Ct[rp], col0 + 8 * gi, 0);
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      fence_proxy_async();
      const int oidx = s_task[5], oval = a.base + s_task[6];
      if ((s_task[14] >> 8) != 0 && s_task[6] > 1) {  // ordered publication (R25)
        const int* c = R.ctr + oidx;
        if (ld_acquire(c) < oval - 1) {
          const unsigned long long t0w = globaltimer();
          while (ld_acquire(c) < oval - 1) {
            __nanosleep(TQR_POLL_NS);
            if (globaltimer() - t0w > 20ull * 1000000000ull) __trap();
          }
        }
      }
      const int ocnt = (s_task[15] >> 8) & 0xFF;
      for (int x = 0; x < (ocnt > 0 ? ocnt : 1); ++x) st_release(R.ctr + oidx + x, oval);
      if (R.trace) {
        unsigned long long* tr = R.trace + (size_t)tk * 4;
        tr[0] = ((unsigned long long)smid() << 32) | (unsigned)tk;
        tr[1] = t_grab;
        tr[2] = t_start;
        tr[3] = globaltimer();
      }
    }
  }
}

// Off-diagonal SI x SI blocks of the output T_L (SO x SO) of every unit (as ::form_t_kernel,
// with the reflectors of a unit spanning its two tiles).  One CTA per (unit (i0, k), L).
__global__ void __launch_bounds__(256) form_t_kernel(const double* __restrict__ A, double* __restrict__ T,
                                                     const int* __restrict__ units, int nunits, int p) {
  constexpr int NLO = TB / SO, RC = 64;
  extern __shared__ double fsm[];
  double(*U)[SO + 1] = reinterpret_cast<double(*)[SO + 1]>(fsm);
  double* Z = fsm + RC * (SO + 1);
  double* tau = Z + SO * SO;
  double* Tf = fsm;
  const int L = blockIdx.x % NLO, u = blockIdx.x / NLO;
  if (u >= nunits) return;
  const int i0 = units[3 * u], k = units[3 * u + 1], nt = units[3 * u + 2];
  const bool diag = i0 == k;
  double* Ts = T + ((size_t)i0 + (size_t)k * p) * (size_t)SO * TB + (size_t)L * SO * SO;
  const int c0 = L * SO, tid = threadIdx.x;
  const int a = tid % SO, bg = tid / SO, NBG = 256 / SO;
  double acc[SO / (256 / SO)];
#pragma unroll
  for (int x = 0; x < SO / NBG; ++x) acc[x] = 0.0;
  const int rows = nt * TB;
  for (int r0 = diag ? c0 : 0; r0 < rows; r0 += RC) {
    __syncthreads();
    for (int e = tid; e < RC * SO; e += 256) {
      const int rr = e % RC, c = e / RC, r = r0 + rr, gc = c0 + c;
      double uv = 0.0;
      if (r < rows) {
        const double* At = A + ((size_t)(i0 + r / TB) + (size_t)k * p) * TB * TB;
        const int rt = r % TB;
        uv = diag ? (rt < gc ? 0.0 : (rt == gc ? 1.0 : At[(size_t)gc * TB + rt])) : At[(size_t)gc * TB + rt];
      }
      U[rr][c] = uv;
    }
    __syncthreads();
    for (int rr = 0; rr < RC; ++rr) {
      const double ua = U[rr][a];
#pragma unroll
      for (int x = 0; x < SO / NBG; ++x) acc[x] += ua * U[rr][bg + NBG * x];
    }
  }
#pragma unroll
  for (int x = 0; x < SO / NBG; ++x) Z[a + (bg + NBG * x) * SO] = acc[x];
  if (tid < SO) tau[tid] = Ts[(size_t)tid * SO + tid];
  __syncthreads();
  if (tid < 32 * ((SO + 31) / 32)) build_t<SO>(Tf, tau, Z);
  __syncthreads();
  for (int e = tid; e < SO * SO; e += 256) {
    const int r = e % SO, c = e / SO;
    if (r / S < c / S) Ts[e] = Tf[e];
  }
}
}  // namespace tall

cudaError_t launch_exec_tall(const ExecArgs& a, int grid, cudaStream_t st) {
  constexpr int NDEV = 64;
  static bool attr[NDEV] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= NDEV || !attr[dev]) {
    e = cudaFuncSetAttribute(tall::exec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tall::L::BYTES);
    if (e != cudaSuccess) return e;
    if (dev < NDEV) attr[dev] = true;
  }
  ExecArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((const void*)tall::exec_kernel, dim3(grid), dim3(tall::C::NT), params,
                                     tall::L::BYTES, st);
}
int exec_max_ctas_tall(int device) {
  int per_sm = 0, sms = 0;
  cudaFuncSetAttribute(tall::exec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tall::L::BYTES);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tall::exec_kernel, tall::C::NT, tall::L::BYTES) !=
      cudaSuccess)
    return 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return per_sm * sms;
}
int exec_slice_tall() { return tall::C::SLICE; }
cudaError_t launch_form_t_tall(const double* A, double* T, const int* d_units, int nunits, int p, cudaStream_t st) {
  if (nunits == 0) return cudaSuccess;
  constexpr size_t smem = (size_t)(64 * (tall::SO + 1) + tall::SO * tall::SO + tall::SO) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(tall::form_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  tall::form_t_kernel<<<(unsigned)(nunits * (tall::TB / tall::SO)), 256, smem, st>>>(A, T, d_units, nunits, p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Instances and dispatch.  (b, s) pairs built: the BASELINE.json configs (64,16),
// (128,32), (256,32) plus small/test shapes and s == b (the paper's unblocked kernels).
// ---------------------------------------------------------------------------------------
#define TQR_INSTANCES(X) \
  X(16, 8) X(16, 16) X(32, 8) X(32, 32) X(64, 16) X(64, 64) X(128, 32) X(256, 32) X(512, 64)

// RWM: rows per warp cap (Cfg::RW = min(B, RWM)).  b >= 256 tiles are built twice: RWM = 256
// (one warp holds a whole 256-row column group: no row-partial exchange, 64-column passes --
// square grids) and RWM = 128 (32-column passes -- tall-skinny grids want the finer tasks);
// the plan chooses (tqr_host.cpp).  b <= 128 has RW = B either way.
template <int B, int S, int MODE, int RWM>
static cudaError_t launch_mode(const ExecArgs& a, int grid, cudaStream_t st) {
  using L = Layout<B, Inner<B, S>::SI, RWM>;
  // the shared-memory attribute is per device: cache it per device ordinal
  constexpr int NDEV = 64;
  static bool attr[NDEV] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= NDEV || !attr[dev]) {
    e = cudaFuncSetAttribute(exec_kernel<B, S, MODE, RWM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    if (e != cudaSuccess) return e;
    if (dev < NDEV) attr[dev] = true;
  }
  ExecArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((const void*)exec_kernel<B, S, MODE, RWM>, dim3(grid),
                                     dim3(Cfg<B, Inner<B, S>::SI, RWM>::NT), params, L::BYTES, st);
}
template <int B, int S, int RWM>
static cudaError_t launch_one(const ExecArgs& a, int mode, int grid, cudaStream_t st) {
  if (mode == 1) return launch_mode<B, S, 1, RWM>(a, grid, st);
  if (mode == 2) return launch_mode<B, S, 2, RWM>(a, grid, st);
  return launch_mode<B, S, 0, RWM>(a, grid, st);
}

template <int B, int S, int RWM>
static int max_ctas_one(int device) {
  using L = Layout<B, Inner<B, S>::SI, RWM>;
  int per_sm = 0, sms = 0, worst = 1 << 30;
  const void* fns[3] = {(const void*)exec_kernel<B, S, 0, RWM>, (const void*)exec_kernel<B, S, 1, RWM>,
                        (const void*)exec_kernel<B, S, 2, RWM>};
  for (const void* f : fns) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, Cfg<B, Inner<B, S>::SI, RWM>::NT, L::BYTES) !=
        cudaSuccess)
      return 0;
    worst = per_sm < worst ? per_sm : worst;
  }
  per_sm = worst;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return per_sm * sms;
}

bool exec_supported(int b, int s) {
#define X(BB, SS) if (b == BB && s == SS) return true;
  TQR_INSTANCES(X)
#undef X
  return false;
}
int exec_rw_variant(int b, int rwm) { return (b >= 256 && rwm >= 256) ? 256 : 128; }

cudaError_t launch_exec(int b, int s, int mode, int rwm, const ExecArgs& a, int grid, cudaStream_t st) {
#define X(BB, SS)                                                              \
  if (b == BB && s == SS) {                                                    \
    if constexpr (BB >= 256)                                                   \
      if (exec_rw_variant(b, rwm) == 256) return launch_one<BB, SS, 256>(a, mode, grid, st); \
    return launch_one<BB, SS, 128>(a, mode, grid, st);                         \
  }
  TQR_INSTANCES(X)
#undef X
  return cudaErrorInvalidValue;
}

int exec_slice(int b, int s, int rwm) {
#define X(BB, SS)                                                                         \
  if (b == BB && s == SS)                                                                 \
    return exec_rw_variant(b, rwm) == 256 ? Cfg<BB, Inner<BB, SS>::SI, 256>::SLICE        \
                                          : Cfg<BB, Inner<BB, SS>::SI, 128>::SLICE;
  TQR_INSTANCES(X)
#undef X
  return 0;
}

int exec_max_ctas(int b, int s, int rwm, int device) {
#define X(BB, SS)                                                          \
  if (b == BB && s == SS) {                                                \
    if constexpr (BB >= 256)                                               \
      if (exec_rw_variant(b, rwm) == 256) return max_ctas_one<BB, SS, 256>(device); \
    return max_ctas_one<BB, SS, 128>(device);                              \
  }
  TQR_INSTANCES(X)
#undef X
  return 0;
}

// ---------------------------------------------------------------------------------------
// Layout kernels (Block Data Layout).  HBM-bound copies, organised by
// RUNS: a run is column cc of tile (i, jl) -- B contiguous doubles in the tile-major array
// and rows [i*B, i*B + B) of global column c = (coff + jl*cstride)*B + cc in the
// column-major array.  Runs are numbered (jl*B + cc)*p + i, so consecutive runs continue one
// column of the column-major side.  A warp moves a run (B >= 64) or 32/(B/2) runs (B < 64)
// per iteration with 16-byte accesses, all of a lane's loads issued before its stores; the
// index arithmetic (64-bit div/mod) is per run, not per element.  A run cropped at m / n,
// or whose column-major start is not 16-byte aligned (odd leading dimension), goes scalar.
// get_r skips the reads of runs wholly below the diagonal (zeros).
// ---------------------------------------------------------------------------------------
enum RunOp { OP_PACK = 0, OP_UNPACK = 1, OP_GETR = 2, OP_EYE = 3 };

template <int B, int OP>
__global__ void __launch_bounds__(256) runs_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t ld,
                                                   int64_t m, int64_t n, int64_t p, int cstride, int coff,
                                                   int64_t nruns) {
  constexpr int NV = B / 2;                     // double2 per run
  constexpr int RPW = NV >= 32 ? 1 : 32 / NV;   // runs per warp iteration
  constexpr int VPL = NV >= 32 ? NV / 32 : 1;   // double2 per lane per run
  const int lane = threadIdx.x & 31;
  const int sub = NV >= 32 ? 0 : lane / NV, x0 = NV >= 32 ? lane : lane % NV;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t kmin = m < n ? m : n;  // rows of R (GETR)
  for (int64_t run = warp * RPW + sub; run < nruns; run += nw * RPW) {
    const int64_t i = run % p, col = run / p;
    const int64_t jl = col / B;
    const int cc = (int)(col - jl * B);
    const int64_t c = ((int64_t)coff + jl * cstride) * B + cc;  // global column
    const int64_t r0 = i * B;                                   // global first row
    const int64_t toff = ((i + jl * p) * B + cc) * B;           // run start, tile-major
    if (OP == OP_EYE) {  // dst tile-major, columns < n (= k) and rows < m hold I
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int e = 2 * (x0 + 32 * v);
        const double2 z = make_double2((r0 + e == c && c < n && r0 + e < m) ? 1.0 : 0.0,
                                       (r0 + e + 1 == c && c < n && r0 + e + 1 < m) ? 1.0 : 0.0);
        reinterpret_cast<double2*>(dst + toff)[x0 + 32 * v] = z;
      }
      continue;
    }
    const int64_t rows = OP == OP_GETR ? kmin : m;  // rows of the column-major side
    const bool in_col = c < n;
    const bool full = in_col && r0 + B <= rows;
    const bool al = ((c * ld) & 1) == 0;            // 16-byte aligned column-major run start
    const double* s_ = OP == OP_PACK ? src + c * ld + r0 : src + toff;
    double* d_ = OP == OP_PACK ? dst + toff : dst + c * ld + r0;
    if (OP != OP_PACK && !in_col) continue;         // nothing to write
    if (OP == OP_GETR && r0 > c) {                  // wholly below the diagonal: zeros, no read
      if (full && al) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) reinterpret_cast<double2*>(d_)[x0 + 32 * v] = make_double2(0.0, 0.0);
      } else {
        for (int e = x0; e < B; e += (NV >= 32 ? 32 : NV))
          if (r0 + e < rows) d_[e] = 0.0;
      }
      continue;
    }
    if (OP == OP_PACK && !in_col) {                 // padding column
#pragma unroll
      for (int v = 0; v < VPL; ++v) reinterpret_cast<double2*>(d_)[x0 + 32 * v] = make_double2(0.0, 0.0);
      continue;
    }
    if (full && al) {
      double2 t[VPL];
#pragma unroll
      for (int v = 0; v < VPL; ++v) t[v] = __ldcs(reinterpret_cast<const double2*>(s_) + x0 + 32 * v);
      if (OP == OP_GETR && r0 + B - 1 > c) {        // diagonal run: zeros below row c
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const int64_t r = r0 + 2 * (x0 + 32 * v);
          if (r > c) t[v].x = 0.0;
          if (r + 1 > c) t[v].y = 0.0;
        }
      }
#pragma unroll
      for (int v = 0; v < VPL; ++v) reinterpret_cast<double2*>(d_)[x0 + 32 * v] = t[v];
    } else {                                         // cropped or unaligned run: scalar
      for (int e = x0; e < B; e += (NV >= 32 ? 32 : NV)) {
        const int64_t r = r0 + e;
        if (OP == OP_PACK) d_[e] = r < m ? s_[e] : 0.0;
        else if (r < rows) d_[e] = (OP == OP_GETR && r > c) ? 0.0 : s_[e];
      }
    }
  }
}

template <int OP>
static cudaError_t launch_runs(int b, const double* src, double* dst, int64_t ld, int64_t m, int64_t n, int64_t p,
                               int64_t qloc, int cstride, int coff, cudaStream_t st) {
  const int64_t nruns = p * qloc * (int64_t)b;
  if (nruns == 0) return cudaSuccess;
  const int rpw = b >= 64 ? 1 : 32 / (b / 2);
  int64_t g = ((nruns + rpw - 1) / rpw + 7) / 8;   // 8 warps per block
  if (g > 148 * 8) g = 148 * 8;                    // 8 resident 256-thread blocks per SM
#define RUNS_B(BB) \
  if (b == BB) { runs_kernel<BB, OP><<<(unsigned)g, 256, 0, st>>>(src, dst, ld, m, n, p, cstride, coff, nruns); return cudaGetLastError(); }
  RUNS_B(16) RUNS_B(32) RUNS_B(64) RUNS_B(128) RUNS_B(256) RUNS_B(512)
#undef RUNS_B
  return cudaErrorInvalidValue;
}

// Packed reflector panels for apply-Q from the boundary factors (At, T): the same Yp/Tp
// contents the factorization writes, one thread per element of the lower tile triangle.
// The internal S x S blocks are the diagonal blocks of the output T_L (SO x SO).  The source
// holds storage columns kc of global tile column k = coff + kc*cstride; every element goes to
// all nd destination workspaces (multi-rank: this rank's panels into every rank's workspace).
struct DPtrs {
  double* p[MAX_RANKS];
};
template <int B, int SO>
__global__ void pack_factors_kernel(const double* __restrict__ A, const double* __restrict__ T, DPtrs Yd, DPtrs Td,
                                    int nd, int p, int K, int64_t qloc, int cstride, int coff, int sys_fence) {
  constexpr int S = Inner<B, SO>::SI, RB_ = SO / S;
  const int64_t bb = (int64_t)B * B;
  const int64_t total = (int64_t)p * qloc * bb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = e / bb;
    const int in = (int)(e % bb);
    const int i = (int)(tile % p), kc = (int)(tile / p);
    const int k = coff + kc * cstride;
    if (k >= K || i < k) continue;
    // element `in` of the packed tile: panel l, swizzled position -> (r, c) of the panel
    const int l = in / (B * S), q = in % (B * S);
    const int blk = q >> 6, w = q & 63;
    const int cb = blk / (B / 8), rb = blk % (B / 8);
    const int cc = w >> 3;
    const int c = cb * 8 + cc, r = rb * 8 + ((w & 7) ^ xy(cc));
    const double* At = A + tile * bb;
    const int gc = l * S + c;  // column inside the tile
    double y;
    if (i > k) {
      y = At[(size_t)gc * B + r];
    } else {
      y = r < gc ? 0.0 : (r == gc ? 1.0 : At[(size_t)gc * B + r]);
    }
    const int64_t gtile = (int64_t)i + (int64_t)k * p;  // workspace index: global step k
    for (int d = 0; d < nd; ++d) Yd.p[d][gtile * bb + in] = y;
    if (q < S * S) {  // internal T block l of slot (i, k) in swz<S>
      const int tb = q >> 6, tw = q & 63;
      const int tcb = tb / (S / 8), trb = tb % (S / 8);
      const int tc = tcb * 8 + (tw >> 3), tr = trb * 8 + ((tw & 7) ^ (tc & 6));
      const int Lo = l / RB_, mo = (l % RB_) * S;
      const double tv = T[tile * (int64_t)SO * B + ((int64_t)Lo * SO + mo + tc) * SO + mo + tr];
      for (int d = 0; d < nd; ++d) Td.p[d][gtile * (int64_t)SO * B + (int64_t)l * S * S + q] = tv;
    }
  }
  if (sys_fence) __threadfence_system();  // peer stores visible before the next rank barrier
}

// Output T_L blocks when the executor ran with SI < SO (b = 512, s = 64): the off-diagonal
// SI x SI blocks of T_L = (diag(1/tau) + striu(Z))^{-1}, Z = U_L^T U_L (the forward
// column-wise DLARFT recurrence over SO columns; build_t).  The diagonal
// blocks -- what the factorization applied -- are kept as written; tau_j = T_L[j][j].
// One CTA per (slot (i, k), L); Z accumulated over 64-row chunks of the reflectors.
template <int B, int SO>
__global__ void __launch_bounds__(256) form_t_kernel(const double* __restrict__ A, double* __restrict__ T, int p,
                                                     int qloc, int cstride, int coff) {
  constexpr int SI = Inner<B, SO>::SI, NLO = B / SO, RC = 64;
  extern __shared__ double fsm[];
  double(*U)[SO + 1] = reinterpret_cast<double(*)[SO + 1]>(fsm);  // RC x (SO+1)
  double* Z = fsm + RC * (SO + 1);
  double* tau = Z + SO * SO;
  double* Tf = fsm;  // aliases U once Z is complete
  int64_t idx = blockIdx.x;
  const int L = (int)(idx % NLO);
  idx /= NLO;
  const int i = (int)(idx % p), kc = (int)(idx / p);
  const int k = coff + kc * cstride;  // global tile column
  if (i < k || kc >= qloc) return;
  const double* At = A + ((size_t)i + (size_t)kc * p) * B * B;
  double* Ts = T + ((size_t)i + (size_t)kc * p) * (size_t)SO * B + (size_t)L * SO * SO;
  const bool diag = i == k;
  const int c0 = L * SO, tid = threadIdx.x;
  const int a = tid % SO, bg = tid / SO, NBG = 256 / SO;
  double acc[SO / (256 / SO)];
#pragma unroll
  for (int x = 0; x < SO / NBG; ++x) acc[x] = 0.0;
  for (int r0 = diag ? c0 : 0; r0 < B; r0 += RC) {
    __syncthreads();
    for (int e = tid; e < RC * SO; e += 256) {
      const int rr = e % RC, c = e / RC, r = r0 + rr, gc = c0 + c;
      double u = 0.0;
      if (r < B) u = diag ? (r < gc ? 0.0 : (r == gc ? 1.0 : At[(size_t)gc * B + r])) : At[(size_t)gc * B + r];
      U[rr][c] = u;
    }
    __syncthreads();
    for (int rr = 0; rr < RC; ++rr) {
      const double ua = U[rr][a];
#pragma unroll
      for (int x = 0; x < SO / NBG; ++x) acc[x] += ua * U[rr][bg + NBG * x];
    }
  }
#pragma unroll
  for (int x = 0; x < SO / NBG; ++x) Z[a + (bg + NBG * x) * SO] = acc[x];
  if (tid < SO) tau[tid] = Ts[(size_t)tid * SO + tid];
  __syncthreads();  // (U no longer read: Tf may overwrite it)
  if (tid < 32 * ((SO + 31) / 32)) build_t<SO>(Tf, tau, Z);
  __syncthreads();
  for (int e = tid; e < SO * SO; e += 256) {
    const int r = e % SO, c = e / SO;
    if (r / SI < c / SI) Ts[e] = Tf[e];
  }
}

struct RankPtrs {
  int* p[MAX_RANKS];
};

static int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (int)g;
}

cudaError_t launch_pack(const double* A, int64_t lda, double* At, int64_t m, int64_t n, int b, int64_t p,
                        int64_t qloc, int cstride, int coff, cudaStream_t st) {
  return launch_runs<OP_PACK>(b, A, At, lda, m, n, p, qloc, cstride, coff, st);
}
cudaError_t launch_unpack(const double* At, double* A, int64_t lda, int64_t m, int64_t n, int b, int64_t p,
                          int64_t qloc, int cstride, int coff, cudaStream_t st) {
  return launch_runs<OP_UNPACK>(b, At, A, lda, m, n, p, qloc, cstride, coff, st);
}
cudaError_t launch_get_r(const double* At, double* R, int64_t ldr, int64_t m, int64_t n, int b, int64_t p,
                         int64_t qloc, int cstride, int coff, cudaStream_t st) {
  return launch_runs<OP_GETR>(b, At, R, ldr, m, n, p, qloc, cstride, coff, st);
}

// Cross-rank entry barrier (real multi-GPU): every rank publishes `gen` into arrive[me] of
// every rank, then waits for all ranks' arrivals in its own array.  A rank therefore starts
// call `gen` only after every rank has finished call gen-1 (stream order), so no panel of
// call gen can overwrite a workspace another rank is still reading.
__global__ void rank_barrier_kernel(RankPtrs arr, int nranks, int me, int gen) {
  const int g = threadIdx.x;
  if (g < nranks) {
    __threadfence_system();
    st_release_sys(arr.p[g] + me, gen);
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(arr.p[me] + g) < gen) {
      __nanosleep(500);
      if (globaltimer() - t0 > 60ull * 1000000000ull) __trap();  // a rank never arrived
    }
  }
}
// Connectivity check of the peer mappings (no waiting): rank `me` stores magic + me into
// slot me of every rank's ping array (system-scope release, over NVLink on a real job).
__global__ void ping_kernel(RankPtrs arr, int nranks, int me, int magic) {
  const int g = threadIdx.x;
  if (g < nranks) st_release_sys(arr.p[g] + me, magic + me);
}
cudaError_t launch_ping(int* const* ping_all, int nranks, int me, int magic, cudaStream_t st) {
  RankPtrs arr;
  for (int g = 0; g < MAX_RANKS; ++g) arr.p[g] = g < nranks ? ping_all[g] : nullptr;
  ping_kernel<<<1, 32, 0, st>>>(arr, nranks, me, magic);
  return cudaGetLastError();
}
cudaError_t launch_rank_barrier(int* const* arrive_all, int nranks, int me, int gen, cudaStream_t st) {
  RankPtrs arr;
  for (int g = 0; g < MAX_RANKS; ++g) arr.p[g] = g < nranks ? arrive_all[g] : nullptr;
  rank_barrier_kernel<<<1, 32, 0, st>>>(arr, nranks, me, gen);
  return cudaGetLastError();
}
cudaError_t launch_pack_factors(const double* A, const double* T, double* const* Yp, double* const* Tp, int nd, int b,
                                int s, int64_t p, int64_t K, int64_t qloc, int cstride, int coff, bool sys_fence,
                                cudaStream_t st) {
  const int64_t total = p * qloc * (int64_t)b * b;
  if (total == 0) return cudaSuccess;
  DPtrs Yd{}, Td{};
  for (int d = 0; d < nd && d < MAX_RANKS; ++d) { Yd.p[d] = Yp[d]; Td.p[d] = Tp[d]; }
#define X(BB, SS)                                                                                         \
  if (b == BB && s == SS) {                                                                               \
    pack_factors_kernel<BB, SS><<<grid_for(total), 256, 0, st>>>(A, T, Yd, Td, nd, (int)p, (int)K, qloc,   \
                                                                 cstride, coff, sys_fence ? 1 : 0);      \
    return cudaGetLastError();                                                                            \
  }
  TQR_INSTANCES(X)
#undef X
  return cudaErrorInvalidValue;
}

int exec_inner(int b, int s) {
#define X(BB, SS) if (b == BB && s == SS) return Inner<BB, SS>::SI;
  TQR_INSTANCES(X)
#undef X
  return 0;
}
template <int B, int SO>
static cudaError_t form_t_one(const double* A, double* T, int64_t p, int64_t qloc, int cstride, int coff,
                              cudaStream_t st) {
  if constexpr (Inner<B, SO>::SI == SO) {
    return cudaSuccess;
  } else {
    const int64_t nblk = p * qloc * (B / SO);
    if (nblk == 0) return cudaSuccess;
    constexpr size_t smem = (size_t)(64 * (SO + 1) + SO * SO + SO) * sizeof(double);
    static_assert(64 * (SO + 1) >= SO * SO, "Tf alias");
    cudaError_t e = cudaFuncSetAttribute(form_t_kernel<B, SO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    form_t_kernel<B, SO><<<(unsigned)nblk, 256, smem, st>>>(A, T, (int)p, (int)qloc, cstride, coff);
    return cudaGetLastError();
  }
}
cudaError_t launch_form_t(const double* A, double* T, int b, int s, int64_t p, int64_t qloc, int cstride, int coff,
                          cudaStream_t st) {
#define X(BB, SS) if (b == BB && s == SS) return form_t_one<BB, SS>(A, T, p, qloc, cstride, coff, st);
  TQR_INSTANCES(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_eye_tiles(double* Qt, int64_t m, int64_t k, int b, int64_t p, int64_t qloc, int cstride, int coff,
                             cudaStream_t st) {
  return launch_runs<OP_EYE>(b, nullptr, Qt, 0, m, k, p, qloc, cstride, coff, st);
}

}  // namespace tqr
