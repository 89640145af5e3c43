// tlu_exec.cu -- B200 executor of the tiled LU factorization ("an algorithm
// that is analogous to the QR one"; kernels = DESIGN.md readings LU1-LU9).
//
// One persistent launch per factorization, one 8-warp CTA per SM, tickets in the host's
// list-schedule order and "progress counter >= value" dependencies (the tiled-QR executor's
// protocol, tqr_exec.cu).  Task kinds:
//   G  GETRF(k)        panel: in-tile LU with partial pivoting, block by block (LU1)
//   T  TSTRF(k,i)      panel: LU with pairwise pivoting of [U_kk; A_ik] (LU3)
//   L  GESSM(k,j,sl)   update of a 64-column slice of A_kj (LU2)
//   S  SSSSM(k,i,j,sl) update of a 64-column slice of [A_kj; A_ij] (LU4)
// Update blocks (apply_block, per inner block l): the target slice Y lives in shared memory
// (column-major, ld b + 4: conflict-free 8x8 accumulator fragments); the block's interchanges
// are one gather/scatter of at most 2s rows (the net permutation the panel precomputed, so no
// serial swap chain in the update); X_l = W_l X_l by DMMA (W_l = the inverse of the block's
// unit-lower factor, computed once by the panel, LU8); Y -= L_l X_l by DMMA.8x8x4 with the
// multipliers streamed from L2 straight into A fragments.  Bound: the fp64 DMMA pipe
// (2 b s w flops per block against (b + s) w x 16 bytes of shared-memory traffic).
// Panels: row-per-thread (thread r holds row r of the block's s columns in registers), one
// block-wide argmax (warp shuffles + 8 partials) and one interchange per column.
#include <cuda_runtime.h>

#include "tlu_internal.h"
#include "tqr_device.cuh"
#include "tqr_internal.h"

namespace tqr {
namespace lu {

constexpr int NT = 256;
constexpr int W = 64;  // update slice width (columns)
#ifndef LU_KU
#define LU_KU 8  // unroll of the update GEMM's k-steps (C3 LU: 2 -> 180.8 ms, 4 -> 180.9, 8 -> 178.0)
#endif
#ifndef LU_PF
#define LU_PF 1  // L2 prefetch of the task this many ticket rounds ahead (0: off; development knob;
                 // same-box C3 LU: off 178.1-178.4 ms, 1 round 176.1, 2 rounds 178.8, 4 rounds 177.0)
#endif
#ifndef LU_NEXT
#define LU_NEXT 0  // cross-task pipelining of the dispatch (as the QR executor): half-way through an
                   // update task thread 0 takes the next ticket, one block later fetches its record
                   // (cp.async), so both round trips overlap the GEMMs (0: off; 2: also the L2
                   // prefetch of that task's slice one more block later)
#endif
constexpr int NX_TK = TASK_INTS, NX_REC = TASK_INTS + 1;  // s_next: the held ticket / its record's ticket
#define LU_STR(x) #x
#define LU_UNROLL(n) _Pragma(LU_STR(unroll n))

template <int B, int S>
struct LCfg {
  static_assert(B % 64 == 0 || B == 64, "b: 64, 128, 256");
  static_assert(S % 8 == 0 && B % S == 0 && S <= 32, "s: 8 | s, s | b, s <= 32");
  static constexpr int NB = B / S;
  // LU12: the update forms Y -= (L_l W_l) X_l next to X_l <- W_l X_l (b = 256: C3 LU 190.9 ->
  // 180.8 ms); at b <= 128 the panel chain bounds the run and the panels' Ltilde products cost
  // more than the updates gain (C2 LU 8.74 -> 9.22 ms), so those instances keep L_l
  static constexpr bool LT = B >= 256;
  // LT: the workspace holds each block's L_l W_l in the shared-memory layout (S columns at ld
  // LDL), so one bulk copy per block brings it in (one thread, completion on an mbarrier)
  static constexpr int LTT = LT ? B * (B + 4) : 0;  // doubles per workspace tile
  static constexpr int LDX = W + 4;          // X_l: S rows x W, row-major (two buffers)
  static constexpr int LDW = S + 4;          // W_l: S x S column-major (two buffers)
  static constexpr int LDL = B + 4;          // L_l: B x S column-major (two buffers)
  static constexpr int LDST = W + 2;         // interchange staging: 2S rows x W, row-major
  static constexpr int LUT = S + 1;          // panel top block, row-major
  static constexpr int PL = 4 + 4 * S;       // pair list (count, -, -, -, dst, src, ...)
  static constexpr int SLT = B + S;          // slot tables: row -> its pair as source / destination
  static constexpr int PLW = PL + 2 * SLT;   // per-block workspace ints (16-byte multiple)
  static constexpr int RPW = B / 8;          // GEMM rows per warp
  static constexpr int MT = RPW / 8;         // 8-row m-tiles per warp
  // shared memory (doubles)
  static constexpr int OFF_ST = 0;                       // staging (2S x LDST); the panel's Ut aliases it
  static constexpr int OFF_UT = OFF_ST;
  static constexpr int OFF_L = OFF_ST + 2 * S * LDST;    // 2 x S x LDL
  static constexpr int OFF_X = OFF_L + 2 * S * LDL;      // 2 x S x LDX
  static constexpr int OFF_W = OFF_X + 2 * S * LDX;      // 2 x S x LDW
  static constexpr int OFF_BUF = OFF_W + 2 * S * LDW;    // 2 x S (GETRF row interchange)
  static constexpr int OFF_RED = OFF_BUF + 2 * S;        // 8 warp maxima
  static constexpr int NDBL = (OFF_RED + 8 + 1) & ~1;
  static_assert(S * LUT + S * S <= 2 * S * LDST, "Ut and the panel's W_l copy fit the staging area");
  // ints after the doubles
  static constexpr int IOFF_RIDX = 0;                // 8 warp argmax rows
  static constexpr int IOFF_PIV = 8;                 // S pivots of the current block
  static constexpr int IOFF_CUR = IOFF_PIV + S;      // B (GETRF net-permutation simulation)
  static constexpr int IOFF_CNT = IOFF_CUR + B;      // 1
  static constexpr int IOFF_BLK = (IOFF_CNT + 4 + 3) & ~3;  // 2 x PLW: the blocks' pair lists + slot tables
  static constexpr int IOFF_MB = (IOFF_BLK + 2 * PLW + 1) & ~1;  // LT: 2 mbarriers (L_l W_l bulk copies) ...
  static constexpr int IOFF_USE = IOFF_MB + 4;                    // ... and their completed-phase counts
  static constexpr int NINT = IOFF_USE + 2;
  static constexpr size_t SMEM = (size_t)NDBL * 8 + (size_t)NINT * 4;
};

__device__ __forceinline__ double* wslot_ptr(double* W_, int i, int k, int p, int B, int S) {
  return W_ + ((size_t)i + (size_t)k * p) * (size_t)S * B;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}

// ---- GESSM (SS = false) / SSSSM (SS = true) on one column slice, inner blocks [l0, l1) ----
// The slice's accumulators stay in registers for the whole run (warp w owns rows
// [w RPW, (w + 1) RPW) x W columns as 8x8 DMMA fragments).  A block's interchanges move only the
// rows its pair list names (<= 2S): each row's owner stores it to a staging row if it is a
// source and reloads it if it is a destination (the precomputed slot tables give the pair; the
// register index is static -- every m-tile is visited with a per-lane predicate), so no pass
// moves the whole slice.  Each block's inputs -- L_l (B x S multipliers; GESSM: rows >= c0 + S),
// W_l, the pair list and slot tables, SSSSM: X_l = C1's rows [c0, c0 + S) -- are double-buffered
// and prefetched by cp.async one block ahead, so their L2 latency hides behind the previous
// block's GEMM.  Y: the target tile (GESSM: A_kj, SSSSM: A_ij); L: the multipliers' tile (A_kk /
// A_ik); Wsl / wsp: the W slot and workspace slot of those factors; C1 (SSSSM): A_kj.  Rows
// [r_lo, B) of the slice are stored back (GETRF's trailing update: LU11).
// element e of an R x W row-major shared tile <-> column-major global: 8-row x 4-column warp
// tiles (global: 4 runs of 64 bytes; shared at ld W + 4: the minimum number of wavefronts)
__device__ __forceinline__ void io_rc(int e, int& r, int& c) {
  const int lane = e & 31, t = e >> 5;
  constexpr int CT = W / 4;
  r = 8 * (t / CT) + (lane >> 2);
  c = 4 * (t % CT) + (lane & 3);
}

template <int B, int S, bool SS>
__device__ __forceinline__ void issue_inputs(double* sm, int* ism, int l, const double* __restrict__ L,
                                             const double* __restrict__ Wsl, const int* __restrict__ wsp,
                                             const double* C1, int cl, int nc) {
  using C = LCfg<B, S>;
  const int tid = threadIdx.x, bf = l & 1, c0 = l * S;
  double* Ls = sm + C::OFF_L + bf * S * C::LDL;
  double* Xs = sm + C::OFF_X + bf * S * C::LDX;
  double* Ws = sm + C::OFF_W + bf * S * C::LDW;
  int* blk = ism + C::IOFF_BLK + bf * C::PLW;
  if constexpr (C::LT) {  // L_l W_l: one bulk copy of the block (rows < r_lo unused by GESSM)
    if (tid == 0) {
      unsigned long long* bar = reinterpret_cast<unsigned long long*>(ism + C::IOFF_MB) + bf;
      constexpr unsigned bytes = S * C::LDL * 8;
      fence_proxy_async();  // the panel's generic stores (acquired / barrier-ordered) before the async read
      mbar_expect_tx(bar, bytes);
      bulk_g2s(Ls, L + (size_t)c0 * C::LDL, bytes, bar);
    }
  } else {
    const int r_lo = SS ? 0 : c0 + S;
    const int nv = (B - r_lo) / 2;  // 16-byte granules per column
    for (int e = tid; e < nv * S; e += NT) {
      const int v = e % nv, cc = e / nv;
      cp_async16(Ls + cc * C::LDL + r_lo + 2 * v, L + r_lo + 2 * v + (size_t)(c0 + cc) * B);
    }
  }
  const double* Wl = Wsl + (size_t)l * S * S;
  for (int e = tid; e < S * S / 2; e += NT) {
    const int r2 = e % (S / 2), cc = e / (S / 2);
    cp_async16(Ws + cc * C::LDW + 2 * r2, Wl + cc * S + 2 * r2);
  }
  const int* pl = wsp + l * C::PLW;
  for (int e = tid; e < C::PLW / 4; e += NT) cp_async16(blk + 4 * e, pl + 4 * e);
  if (SS) {
    for (int e = tid; e < S * W; e += NT) {
      int r, cc;
      io_rc(e, r, cc);
      if (cc < nc) cp_async8(Xs + r * C::LDX + cc, C1 + (c0 + r) + (size_t)(cl + cc) * B);
    }
  }
  cp_async_commit();
}

template <int B, int S>
__device__ __forceinline__ void lu_prefetch(const LuArgs& a, const int* q);

// pa / s_next (update tasks over all NB blocks only): the dispatch pipelining of LU_NEXT.  Holding
// one ticket ahead cannot deadlock: every wait is on a smaller ticket, and the smallest
// unfinished ticket is some CTA's current task.
template <int B, int S, bool SS>
__device__ __noinline__ void update_run(double* sm, int* ism, double* Y, const double* __restrict__ L,
                                        const double* __restrict__ Wsl, const int* __restrict__ wsp, double* C1,
                                        int cl, int nc, int l0, int l1, int r_lo, const LuArgs* pa = nullptr,
                                        int* s_next = nullptr) {
  using C = LCfg<B, S>;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int r0 = warp * C::RPW;
  double* St = sm + C::OFF_ST;
  issue_inputs<B, S, SS>(sm, ism, l0, L, Wsl, wsp, C1, cl, nc);
  int ntk = -1;  // thread 0: the next ticket (LU_NEXT)
  // the slice into registers (fragment rows r0 + 8 mt + g, columns 8 nt + 2 t4, + 1)
  double2 acc[C::MT][W / 8];
#pragma unroll
  for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < W / 8; ++nt) {
      const int row = r0 + 8 * mt + g, col = 8 * nt + 2 * t4;
      acc[mt][nt].x = col < nc ? __ldcg(Y + row + (size_t)(cl + col) * B) : 0.0;
      acc[mt][nt].y = col + 1 < nc ? __ldcg(Y + row + (size_t)(cl + col + 1) * B) : 0.0;
    }
#pragma unroll 1
  for (int l = l0; l < l1; ++l) {
    const int bf = l & 1, c0 = l * S;
    double* Ls = sm + C::OFF_L + bf * S * C::LDL;
    double* Xs = sm + C::OFF_X + bf * S * C::LDX;
    const double* Ws = sm + C::OFF_W + bf * S * C::LDW;
    const int* blk = ism + C::IOFF_BLK + bf * C::PLW;
    const int* srcs = blk + C::PL;
    const int* dsts = srcs + C::SLT;
    cp_async_wait<0>();
    if constexpr (C::LT)
      mbar_wait(reinterpret_cast<unsigned long long*>(ism + C::IOFF_MB) + bf, ism[C::IOFF_USE + bf] & 1);
    __syncthreads();  // block l's inputs landed; every thread is past block l - 1
    if (C::LT && tid == 0) ++ism[C::IOFF_USE + bf];  // read again only after the next barrier
    if (l + 1 < l1) issue_inputs<B, S, SS>(sm, ism, l + 1, L, Wsl, wsp, C1, cl, nc);
    if (LU_NEXT > 0 && pa && tid == 0) {  // (pa: l1 - l0 = NB >= 4, so all three blocks below exist)
      const int lm = l0 + (l1 - l0) / 2 - 1;
      if (l == lm) ntk = atomicAdd(pa->ticket, 1);
      if (l == lm + 1) {
        s_next[NX_TK] = ntk;
        if (ntk < pa->ntasks) {
#pragma unroll
          for (int x = 0; x < TASK_INTS; x += 4) cp_async16(s_next + x, pa->tasks + (size_t)ntk * TASK_INTS + x);
          cp_async_commit();
          s_next[NX_REC] = ntk;
        }
      }
      if (LU_NEXT > 1 && l == lm + 2 && ntk < pa->ntasks) lu_prefetch<B, S>(*pa, s_next);  // (landed: wait above)
    }
    // (1) sources -> staging
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt) {
      const int sl = srcs[r0 + 8 * mt + g];
      if (sl >= 0) {
#pragma unroll
        for (int nt = 0; nt < W / 8; ++nt)
          *reinterpret_cast<double2*>(St + sl * C::LDST + 8 * nt + 2 * t4) = acc[mt][nt];
      }
    }
    if (SS) {
      for (int e = tid; e < S * W / 2; e += NT) {
        const int r = e / (W / 2), c2 = e % (W / 2);
        const int sl = srcs[B + r];
        if (sl >= 0)
          *reinterpret_cast<double2*>(St + sl * C::LDST + 2 * c2) =
              *reinterpret_cast<const double2*>(Xs + r * C::LDX + 2 * c2);
      }
    }
    __syncthreads();
    // (2) destinations <- staging
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt) {
      const int sl = dsts[r0 + 8 * mt + g];
      if (sl >= 0) {
#pragma unroll
        for (int nt = 0; nt < W / 8; ++nt)
          acc[mt][nt] = *reinterpret_cast<const double2*>(St + sl * C::LDST + 8 * nt + 2 * t4);
      }
    }
    if (SS) {
      for (int e = tid; e < S * W / 2; e += NT) {
        const int r = e / (W / 2), c2 = e % (W / 2);
        const int sl = dsts[B + r];
        if (sl >= 0)
          *reinterpret_cast<double2*>(Xs + r * C::LDX + 2 * c2) =
              *reinterpret_cast<const double2*>(St + sl * C::LDST + 2 * c2);
      }
    } else if (r0 >= c0 && r0 < c0 + S) {  // GESSM: X_l = Y's rows [c0, c0 + S) (this warp's band)
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < W / 8; ++nt)
          *reinterpret_cast<double2*>(Xs + (r0 - c0 + 8 * mt + g) * C::LDX + 8 * nt + 2 * t4) = acc[mt][nt];
    }
    __syncthreads();
    if constexpr (C::LT) {
    // (3) X_l <- W_l X_l and (4) Y -= Ltilde_l X_l, both from the interchanged X_l (Ltilde_l =
    // L_l W_l, formed once by the panel: LU12), so neither waits for the other and no barrier
    // separates them.  SSSSM: warp w forms the X_l fragments f = w + 8x (M = S, N = W, K = S) and
    // stores them straight to C1's rows [c0, c0 + S); GESSM: the band warps (rows [c0, c0 + S))
    // form their own rows of W_l X_l, the others update.
    if (SS) {
      constexpr int SMT = S / 8, NNT = W / 8, PER = SMT * NNT / 8;
      double d[PER][2];
#pragma unroll
      for (int x = 0; x < PER; ++x) d[x][0] = d[x][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < S / 4; ++ks)
#pragma unroll
        for (int x = 0; x < PER; ++x) {
          const int f = warp + 8 * x, mt = f % SMT, nt = f / SMT;
          dmma(d[x], Ws[(4 * ks + t4) * C::LDW + 8 * mt + g], Xs[(4 * ks + t4) * C::LDX + 8 * nt + g]);
        }
      LU_UNROLL(LU_KU)
      for (int ks = 0; ks < S / 4; ++ks) {
        double a[C::MT];
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) a[mt] = -Ls[(4 * ks + t4) * C::LDL + r0 + 8 * mt + g];
#pragma unroll
        for (int nt = 0; nt < W / 8; ++nt) {
          const double bb = Xs[(4 * ks + t4) * C::LDX + 8 * nt + g];
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt) {
            double d2[2] = {acc[mt][nt].x, acc[mt][nt].y};
            dmma(d2, a[mt], bb);
            acc[mt][nt] = make_double2(d2[0], d2[1]);
          }
        }
      }
      // (5) X_l back to C1's rows [c0, c0 + S), from the fragments' registers
#pragma unroll
      for (int x = 0; x < PER; ++x) {
        const int f = warp + 8 * x, mt = f % SMT, nt = f / SMT;
        const int row = c0 + 8 * mt + g, col = 8 * nt + 2 * t4;
        if (col < nc) C1[row + (size_t)(cl + col) * B] = d[x][0];
        if (col + 1 < nc) C1[row + (size_t)(cl + col + 1) * B] = d[x][1];
      }
    } else if (r0 >= c0 + S) {
      LU_UNROLL(LU_KU)
      for (int ks = 0; ks < S / 4; ++ks) {
        double a[C::MT];
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) a[mt] = -Ls[(4 * ks + t4) * C::LDL + r0 + 8 * mt + g];
#pragma unroll
        for (int nt = 0; nt < W / 8; ++nt) {
          const double bb = Xs[(4 * ks + t4) * C::LDX + 8 * nt + g];
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt) {
            double d2[2] = {acc[mt][nt].x, acc[mt][nt].y};
            dmma(d2, a[mt], bb);
            acc[mt][nt] = make_double2(d2[0], d2[1]);
          }
        }
      }
    } else if (r0 >= c0) {  // GESSM band rows: acc <- (W_l X_l)'s rows r0 - c0 + [0, RPW)
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < W / 8; ++nt) acc[mt][nt] = make_double2(0.0, 0.0);
#pragma unroll 2
      for (int ks = 0; ks < S / 4; ++ks) {
        double a[C::MT];
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) a[mt] = Ws[(4 * ks + t4) * C::LDW + (r0 - c0) + 8 * mt + g];
#pragma unroll
        for (int nt = 0; nt < W / 8; ++nt) {
          const double bb = Xs[(4 * ks + t4) * C::LDX + 8 * nt + g];
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt) {
            double d2[2] = {acc[mt][nt].x, acc[mt][nt].y};
            dmma(d2, a[mt], bb);
            acc[mt][nt] = make_double2(d2[0], d2[1]);
          }
        }
      }
    }
    } else {  // b < 256: W_l X_l first, then Y -= L_l X_l (the panels skip Ltilde, LU12)
    // (3) X_l <- W_l X_l  (M = S, N = W, K = S; in registers until every warp has read X_l)
    {
      constexpr int SMT = S / 8, NNT = W / 8, PER = SMT * NNT / 8;
      double d[PER][2];
#pragma unroll
      for (int x = 0; x < PER; ++x) d[x][0] = d[x][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < S / 4; ++ks)
#pragma unroll
        for (int x = 0; x < PER; ++x) {
          const int f = warp + 8 * x, mt = f % SMT, nt = f / SMT;
          dmma(d[x], Ws[(4 * ks + t4) * C::LDW + 8 * mt + g], Xs[(4 * ks + t4) * C::LDX + 8 * nt + g]);
        }
      __syncthreads();
#pragma unroll
      for (int x = 0; x < PER; ++x) {
        const int f = warp + 8 * x, mt = f % SMT, nt = f / SMT;
        *reinterpret_cast<double2*>(Xs + (8 * mt + g) * C::LDX + 8 * nt + 2 * t4) = make_double2(d[x][0], d[x][1]);
      }
    }
    __syncthreads();
    // (4) Y -= L_l X_l (GESSM: only rows >= c0 + S; the band rows [c0, c0 + S) take X_l)
    if (SS || r0 >= c0 + S) {
#pragma unroll 2
      for (int ks = 0; ks < S / 4; ++ks) {
        double a[C::MT];
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) a[mt] = -Ls[(4 * ks + t4) * C::LDL + r0 + 8 * mt + g];
#pragma unroll
        for (int nt = 0; nt < W / 8; ++nt) {
          const double bb = Xs[(4 * ks + t4) * C::LDX + 8 * nt + g];
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt) {
            double d2[2] = {acc[mt][nt].x, acc[mt][nt].y};
            dmma(d2, a[mt], bb);
            acc[mt][nt] = make_double2(d2[0], d2[1]);
          }
        }
      }
    } else if (!SS && r0 >= c0) {
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < W / 8; ++nt)
          acc[mt][nt] = *reinterpret_cast<const double2*>(Xs + (r0 - c0 + 8 * mt + g) * C::LDX + 8 * nt + 2 * t4);
    }
    if (SS) {  // (5) X_l back to C1's rows [c0, c0 + S)
      for (int e = tid; e < S * W; e += NT) {
        int r, cc;
        io_rc(e, r, cc);
        if (cc < nc) C1[(c0 + r) + (size_t)(cl + cc) * B] = Xs[r * C::LDX + cc];
      }
    }
    }
  }
  // the slice back (rows >= r_lo)
#pragma unroll
  for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < W / 8; ++nt) {
      const int row = r0 + 8 * mt + g, col = 8 * nt + 2 * t4;
      if (row >= r_lo) {
        if (col < nc) Y[row + (size_t)(cl + col) * B] = acc[mt][nt].x;
        if (col + 1 < nc) Y[row + (size_t)(cl + col + 1) * B] = acc[mt][nt].y;
      }
    }
  __syncthreads();
}

// block-wide argmax of v (ties: the smaller index); every thread gets (value, index)
template <int B, int S>
__device__ __forceinline__ void block_argmax(double* sm, int* ism, double v, int idx, double& bv, int& bi) {
  using C = LCfg<B, S>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
  if (lane == 0) { sm[C::OFF_RED + warp] = v; ism[C::IOFF_RIDX + warp] = idx; }
  __syncthreads();
  bv = sm[C::OFF_RED];
  bi = ism[C::IOFF_RIDX];
#pragma unroll
  for (int w = 1; w < 8; ++w) {  // warps hold increasing row ranges: strict > keeps the smaller row
    const double x = sm[C::OFF_RED + w];
    if (x > bv) { bv = x; bi = ism[C::IOFF_RIDX + w]; }
  }
}

// W_l = (I + strict lower of Ut)^{-1} (unit lower; LU8), column c = thread c, stored column-major
template <int B, int S>
__device__ __forceinline__ void build_w(const double* Ut, double* Wl, double* Wsm) {
  using C = LCfg<B, S>;
  const int tid = threadIdx.x;
  if (tid < S) {
    double w[S];
#pragma unroll
    for (int r = 0; r < S; ++r) w[r] = r == tid ? 1.0 : 0.0;
#pragma unroll
    for (int r = 1; r < S; ++r) {
      if (r > tid) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < r; ++t) acc = fma(Ut[r * C::LUT + t], w[t], acc);
        w[r] = -acc;
      }
    }
#pragma unroll
    for (int r = 0; r < S; ++r) {
      Wl[tid * S + r] = w[r];
      Wsm[tid * S + r] = w[r];
    }
  }
}

// Ltilde_l = L_l W_l for rows [r_lo, B) of the block's multipliers (thread r holds row r in x;
// W_l unit lower, column-major in Wsm, 16-byte aligned), into the workspace tile Lt: the update tasks then form
// Y -= Ltilde_l X_l from the interchanged X_l, independent of X_l <- W_l X_l (LU12)
template <int B, int S>
__device__ __forceinline__ void store_ltilde(const double (&x)[S], const double* Wsm, double* Lt, int c0, int r_lo) {
  const int tid = threadIdx.x;
  if (tid >= r_lo && tid < B) {
#pragma unroll
    for (int c = 0; c < S; ++c) {  // column c of W_l is stored whole (zeros above, 1 on the diagonal)
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int t = c & ~1; t < S; t += 2) {  // 16-byte broadcast loads of W_l
        const double2 w2 = *reinterpret_cast<const double2*>(Wsm + c * S + t);
        a0 = fma(x[t], w2.x, a0);
        a1 = fma(x[t + 1], w2.y, a1);
      }
      Lt[tid + (size_t)(c0 + c) * (B + 4)] = a0 + a1;  // the update's shared layout (LDL = B + 4)
    }
  }
}

// the block's slot tables from its pair list (written by this CTA just before): row -> the
// index of the pair that has it as source / destination, -1 if none (rows [0, B): Y, [B, B + S): X)
template <int B, int S>
__device__ __forceinline__ void build_slots(int* pl) {
  using C = LCfg<B, S>;
  int* srcs = pl + C::PL;
  int* dsts = srcs + C::SLT;
  for (int e = threadIdx.x; e < C::SLT; e += NT) srcs[e] = dsts[e] = -1;
  __syncthreads();
  const int np = __ldcg(pl);
  for (int e = threadIdx.x; e < np; e += NT) {
    dsts[__ldcg(pl + 4 + 2 * e)] = e;
    srcs[__ldcg(pl + 5 + 2 * e)] = e;
  }
  __syncthreads();
}

// GETRF(k) on tile Akk (LU1)
template <int B, int S>
__device__ __noinline__ void getrf_task(double* sm, int* ism, double* Akk, double* Lkk, double* Wsl, int* pivs,
                                        int* perms, int l0, int l1) {
  using C = LCfg<B, S>;
  const int tid = threadIdx.x;
  double* Ut = sm + C::OFF_UT;
  double* bufA = sm + C::OFF_BUF;
  double* bufB = bufA + S;
  int* spiv = ism + C::IOFF_PIV;
  int* cur = ism + C::IOFF_CUR;
  for (int l = l0; l < l1; ++l) {
    const int c0 = l * S;
    double x[S];
    __syncthreads();  // the previous block's trailing stores
#pragma unroll
    for (int c = 0; c < S; ++c) x[c] = (tid < B) ? __ldcg(Akk + tid + (size_t)(c0 + c) * B) : 0.0;
#pragma unroll
    for (int jj = 0; jj < S; ++jj) {
      const int c = c0 + jj;
      double bv;
      int pr;
      block_argmax<B, S>(sm, ism, (tid >= c && tid < B) ? fabs(x[jj]) : -1.0, tid, bv, pr);
      if (tid == c) {
#pragma unroll
        for (int cc = 0; cc < S; ++cc) bufA[cc] = x[cc];
      }
      if (tid == pr) {
#pragma unroll
        for (int cc = 0; cc < S; ++cc) bufB[cc] = x[cc];
      }
      if (tid == 0) spiv[jj] = pr;
      __syncthreads();
      if (pr != c) {
        if (tid == c) {
#pragma unroll
          for (int cc = 0; cc < S; ++cc) x[cc] = bufB[cc];
        } else if (tid == pr) {
#pragma unroll
          for (int cc = 0; cc < S; ++cc) x[cc] = bufA[cc];
        }
      }
      if (tid > c && tid < B) {  // multipliers and the rank-1 update of the block's later columns
        const double d = bufB[jj];
        if (d != 0.0) x[jj] = x[jj] / d;
#pragma unroll
        for (int cc = jj + 1; cc < S; ++cc) x[cc] = fma(-x[jj], bufB[cc], x[cc]);
      }
    }
    if (tid >= c0 && tid < B) {
#pragma unroll
      for (int c = 0; c < S; ++c) Akk[tid + (size_t)(c0 + c) * B] = x[c];
    }
    if (tid >= c0 && tid < c0 + S) {  // L11 of the block
#pragma unroll
      for (int c = 0; c < S; ++c) Ut[(tid - c0) * C::LUT + c] = c < tid - c0 ? x[c] : 0.0;
    }
    for (int e = tid; e < B; e += NT) cur[e] = e;
    if (tid == 0) ism[C::IOFF_CNT] = 0;
    __syncthreads();
    double* Wl = Wsl + (size_t)l * S * S;
    int* pl = perms + l * C::PLW;
    double* Wsm = Ut + S * C::LUT;
    build_w<B, S>(Ut, Wl, Wsm);
    if (tid < S) pivs[c0 + tid] = spiv[tid];
    if (tid == 0) {  // net permutation of the block's interchanges (at most 2S rows move)
      for (int jj = 0; jj < S; ++jj) {
        const int a = c0 + jj, bb = spiv[jj];
        const int t = cur[a];
        cur[a] = cur[bb];
        cur[bb] = t;
      }
    }
    __syncthreads();
    if constexpr (C::LT) store_ltilde<B, S>(x, Wsm, Lkk, c0, c0 + S);
    if (tid < B && cur[tid] != tid) {
      const int e = atomicAdd(ism + C::IOFF_CNT, 1);
      pl[4 + 2 * e] = tid;
      pl[5 + 2 * e] = cur[tid];
    }
    __syncthreads();
    if (tid == 0) pl[0] = ism[C::IOFF_CNT];
    __syncthreads();
    build_slots<B, S>(pl);
    for (int cl = c0 + S; cl < B; cl += W)
      update_run<B, S, false>(sm, ism, Akk, Lkk, Wsl, perms, nullptr, cl, min(W, B - cl), l, l + 1, c0);
  }
}

// TSTRF(k,i) on [U_kk; A_ik] (LU3)
template <int B, int S>
__device__ __noinline__ void tstrf_task(double* sm, int* ism, double* Ukk, double* Aik, double* Lik, double* Wsl, int* pivs,
                                        int* perms, int l0, int l1) {
  using C = LCfg<B, S>;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* Ut = sm + C::OFF_UT;
  int* spiv = ism + C::IOFF_PIV;
  for (int l = l0; l < l1; ++l) {
    const int c0 = l * S;
    double x[S];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < S; ++c) x[c] = (tid < B) ? __ldcg(Aik + tid + (size_t)(c0 + c) * B) : 0.0;
    for (int e = tid; e < S * S; e += NT) {
      const int r = e % S, c = e / S;
      Ut[r * C::LUT + c] = c >= r ? __ldcg(Ukk + (c0 + r) + (size_t)(c0 + c) * B) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < S; ++jj) {
      double bv;
      int br;
      block_argmax<B, S>(sm, ism, tid < B ? fabs(x[jj]) : -1.0, tid, bv, br);
      const int pr = bv > fabs(Ut[jj * C::LUT + jj]) ? br : -1;  // ties: U_kk's row (LU5)
      if (tid == 0) spiv[jj] = pr;
      if (tid == pr) {  // interchange with U's row jj in the block's columns; L part -> Ltilde
#pragma unroll
        for (int cc = 0; cc < S; ++cc) {
          if (cc < jj) {
            Ut[jj * C::LUT + cc] = x[cc];
            x[cc] = 0.0;
          } else {
            const double t = Ut[jj * C::LUT + cc];
            Ut[jj * C::LUT + cc] = x[cc];
            x[cc] = t;
          }
        }
      }
      __syncthreads();
      if (tid < B) {
        const double d = Ut[jj * C::LUT + jj];
        if (d != 0.0) x[jj] = x[jj] / d;
#pragma unroll
        for (int cc = jj + 1; cc < S; ++cc) x[cc] = fma(-x[jj], Ut[jj * C::LUT + cc], x[cc]);
      }
    }
    if (tid < B) {
#pragma unroll
      for (int c = 0; c < S; ++c) Aik[tid + (size_t)(c0 + c) * B] = x[c];
    }
    for (int e = tid; e < S * S; e += NT) {  // U's block (upper part only: A_kk's strict lower holds GETRF's L)
      const int r = e % S, c = e / S;
      if (c >= r) Ukk[(c0 + r) + (size_t)(c0 + c) * B] = Ut[r * C::LUT + c];
    }
    double* Wl = Wsl + (size_t)l * S * S;
    int* pl = perms + l * C::PLW;
    double* Wsm = Ut + S * C::LUT;
    build_w<B, S>(Ut, Wl, Wsm);
    if (tid < S) pivs[c0 + tid] = spiv[tid];
    if (warp == 0) {  // net permutation: X row j <- (previous X row with the same A row) or A row; A row <- last X row
      const int r = lane < S ? spiv[lane] : -1;
      const bool act = r >= 0;
      const unsigned same = __match_any_sync(0xffffffffu, act ? r : -1 - lane);
      const unsigned below = same & ((1u << lane) - 1u);
      const int prev = below ? 31 - __clz(below) : -1;
      const int last = 31 - __clz(same);
      const int n1 = act ? 1 : 0, n2 = (act && lane == last) ? 1 : 0;
      const unsigned m1 = __ballot_sync(0xffffffffu, n1), m2 = __ballot_sync(0xffffffffu, n2);
      const unsigned lt = (1u << lane) - 1u;
      int pos = __popc(m1 & lt) + __popc(m2 & lt);
      if (n1) {
        pl[4 + 2 * pos] = B + lane;
        pl[5 + 2 * pos] = prev >= 0 ? B + prev : r;
        ++pos;
      }
      if (n2) {
        pl[4 + 2 * pos] = r;
        pl[5 + 2 * pos] = B + lane;
      }
      if (lane == 0) pl[0] = __popc(m1) + __popc(m2);
    }
    __syncthreads();
    if constexpr (C::LT) store_ltilde<B, S>(x, Wsm, Lik, c0, 0);
    build_slots<B, S>(pl);
    for (int cl = c0 + S; cl < B; cl += W)
      update_run<B, S, true>(sm, ism, Aik, Lik, Wsl, perms, Ukk, cl, min(W, B - cl), l, l + 1, 0);
  }
}

// GESSM(k,j,sl) (SS = false) / SSSSM(k,i,j,sl) (SS = true): one 64-column slice, every block
template <int B, int S, bool SS>
__device__ __noinline__ void update_task(double* sm, const LuArgs& a, int k, int i, int j, int sl, int* s_next) {
  using C = LCfg<B, S>;
  const int p = a.p;
  const int vr = SS ? i : k;  // tile row of the multipliers / W / interchange lists applied
  double* Y = a.A + ((size_t)(SS ? i : k) + (size_t)j * p) * B * B;
  const double* L = C::LT ? a.Lw + ((size_t)vr + (size_t)k * p) * C::LTT : a.A + ((size_t)vr + (size_t)k * p) * B * B;
  const double* Wsl = wslot_ptr(a.W, vr, k, p, B, S);
  const int* perms = a.perm + ((size_t)vr + (size_t)k * p) * C::NB * C::PLW;
  double* C1 = a.A + ((size_t)k + (size_t)j * p) * B * B;
  const int cl = sl * W;
  update_run<B, S, SS>(sm, reinterpret_cast<int*>(sm + C::NDBL), Y, L, Wsl, perms, SS ? C1 : nullptr, cl,
                       min(W, B - cl), 0, C::NB, 0, LU_NEXT > 0 && C::NB >= 4 ? &a : nullptr, s_next);
}

// L2 prefetch of the target of task record q (update: its tile-column slice, 128 KiB contiguous;
// panel: its block's columns), issued LU_PF ticket rounds ahead (148 tickets per round).  A hint only: L2 is coherent,
// so prefetching before the task's dependencies hold is safe; the slice loads at the start of
// an update task then hit L2 instead of HBM.
template <int B, int S>
__device__ __forceinline__ void lu_prefetch(const LuArgs& a, const int* q) {
  const int kind = q[0], k = q[1], i = q[2], j = q[3], sl = q[4];
  const int p = a.p;
  if (kind == LK_S || kind == LK_L) {
    const double* Y = a.A + ((size_t)(kind == LK_S ? i : k) + (size_t)j * p) * B * B;
    const int cl = sl * W, nc = min(W, B - cl);
    prefetch_l2(Y + (size_t)cl * B, (unsigned)(nc * B * 8));
  } else {
    const double* T = a.A + ((size_t)(kind == LK_T ? i : k) + (size_t)k * p) * B * B;
    const int l0 = sl < 0 ? 0 : sl, nb = sl < 0 ? B / S : 1;
    prefetch_l2(T + (size_t)l0 * S * B, (unsigned)(nb * S * B * 8));
  }
}

template <int B, int S, bool DISP>
__global__ void __launch_bounds__(NT, 1) lu_exec_kernel(const __grid_constant__ LuArgs a) {
  using C = LCfg<B, S>;
  extern __shared__ __align__(16) double sm[];
  int* ism = reinterpret_cast<int*>(sm + C::NDBL);
  __shared__ int s_task[TASK_INTS];
  __shared__ int s_ticket;
  __shared__ __align__(16) int s_next[TASK_INTS + 4];  // a prefetched record, [NX_TK], [NX_REC] (LU_NEXT)
  __shared__ int s_have;
  __shared__ unsigned long long s_tgrab;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int p = a.p;
  if (tid == 0) s_next[NX_TK] = s_next[NX_REC] = -1;
  if (C::LT && tid < 2) {
    mbar_init(reinterpret_cast<unsigned long long*>(ism + C::IOFF_MB) + tid, 1);
    ism[C::IOFF_USE + tid] = 0;
  }
  fence_mbar_init();
  __syncthreads();
  for (;;) {
    int tk;
    unsigned long long t_grab = 0, t_start = 0;
    if constexpr (DISP) {
      // Dispatch by warp 2 (thread 0 of the previous task is still in its fence + release): the
      // ticket, its record and the dependency poll follow one another in one warp, one barrier.
      if (warp == 2) {
        int nt = 0;
        if (lane == 0) nt = atomicAdd(a.ticket, 1);
        nt = __shfl_sync(0xffffffffu, nt, 0);
        if (lane == 0) {
          s_ticket = nt;
          if (a.trace) s_tgrab = globaltimer();
        }
        if (nt < a.ntasks) {
          int rv = lane < TASK_INTS ? a.tasks[(size_t)nt * TASK_INTS + lane] : 0;
          if (lane < TASK_INTS) s_task[lane] = rv;
#pragma unroll
          for (int d = 0; d < TASK_NDEP; ++d) {
            const int code = __shfl_sync(0xffffffffu, rv, 8 + 2 * d), val = __shfl_sync(0xffffffffu, rv, 9 + 2 * d);
            const int cnt = (int)((unsigned)code >> 24), idx = code & 0xFFFFFF;
            for (int x = lane; x < cnt; x += 32) {
              const int* c = a.ctr + idx + x;
              if (ld_acquire(c) >= val) continue;
              const unsigned long long t0w = globaltimer();
              while (ld_acquire(c) < val) {
                __nanosleep(64);
                if (globaltimer() - t0w > 20ull * 1000000000ull) __trap();  // schedule bug: fail loudly
              }
            }
          }
          __syncwarp();
        }
      }
      __syncthreads();
      tk = s_ticket;
      if (tk >= a.ntasks) return;
      if (a.trace && tid == 0) {
        t_grab = s_tgrab;
        t_start = globaltimer();
      }
    } else {
      if (tid == 0) {
        int nt = LU_NEXT > 0 ? s_next[NX_TK] : -1;
        if (nt < 0) nt = atomicAdd(a.ticket, 1);
        if (LU_NEXT > 0) cp_async_wait<0>();  // a prefetched record has landed
        s_ticket = nt;
        s_have = LU_NEXT > 0 && s_next[NX_REC] == nt;
        s_next[NX_TK] = -1;
      }
      __syncthreads();
      tk = s_ticket;
      if (tk >= a.ntasks) return;
      if (tid < TASK_INTS) s_task[tid] = s_have ? s_next[tid] : a.tasks[(size_t)tk * TASK_INTS + tid];
      __syncthreads();
      if (a.trace && tid == 0) t_grab = globaltimer();
      if (warp == 0) {
#pragma unroll
        for (int d = 0; d < TASK_NDEP; ++d) {
          const int code = s_task[8 + 2 * d], val = s_task[9 + 2 * d];
          const int cnt = (int)((unsigned)code >> 24), idx = code & 0xFFFFFF;
          for (int x = lane; x < cnt; x += 32) {
            const int* c = a.ctr + idx + x;
            if (ld_acquire(c) >= val) continue;
            const unsigned long long t0w = globaltimer();
            while (ld_acquire(c) < val) {
              __nanosleep(64);
              if (globaltimer() - t0w > 20ull * 1000000000ull) __trap();  // schedule bug: fail loudly
            }
          }
        }
        __syncwarp();
      }
      __syncthreads();
      if (a.trace && tid == 0) t_start = globaltimer();
    }
    const int kind = s_task[0], k = s_task[1], i = s_task[2], j = s_task[3], sl = s_task[4];
    const int out_c = s_task[5], out_v = s_task[6];  // (s_task is rewritten while thread 0 releases)
    double* Akk = a.A + ((size_t)k + (size_t)k * p) * B * B;
    // panel tasks: inner block sl (record [4]; -1: the whole tile)
    const int l0 = sl < 0 ? 0 : sl, l1 = sl < 0 ? C::NB : sl + 1;
    if (kind == LK_G) {
      getrf_task<B, S>(sm, ism, Akk, C::LT ? a.Lw + ((size_t)k + (size_t)k * p) * C::LTT : Akk, wslot_ptr(a.W, k, k, p, B, S), a.piv + ((size_t)k + (size_t)k * p) * B,
                       a.perm + ((size_t)k + (size_t)k * p) * C::NB * C::PLW, l0, l1);
    } else if (kind == LK_T) {
      double* Aik = a.A + ((size_t)i + (size_t)k * p) * B * B;
      tstrf_task<B, S>(sm, ism, Akk, Aik, C::LT ? a.Lw + ((size_t)i + (size_t)k * p) * C::LTT : Aik, wslot_ptr(a.W, i, k, p, B, S), a.piv + ((size_t)i + (size_t)k * p) * B,
                       a.perm + ((size_t)i + (size_t)k * p) * C::NB * C::PLW, l0, l1);
    } else if (kind == LK_S) {
      update_task<B, S, true>(sm, a, k, i, j, sl, s_next);
    } else {
      update_task<B, S, false>(sm, a, k, i, j, sl, s_next);
    }
    __syncthreads();
    if (LU_PF > 0 && C::LT && tid == 32) {  // overlaps thread 0's release and next ticket round trip
      // (b = 256 only: at b = 128 the panel chain bounds the run; C2 LU 8.83 -> 8.90 ms with it)
      const int nx = tk + LU_PF * (int)gridDim.x;
      if (nx < a.ntasks) lu_prefetch<B, S>(a, a.tasks + (size_t)nx * TASK_INTS);
    }
    if (tid == 0) {
      __threadfence();
      st_release(a.ctr + out_c, out_v);
      if (a.trace) {
        unsigned long long* tr = a.trace + (size_t)tk * 4;
        tr[0] = smid();
        tr[1] = t_grab;
        tr[2] = t_start;
        tr[3] = globaltimer();
      }
    }
  }
}

template <int B, int S>
static cudaError_t launch_inst(const LuArgs& a, int grid, cudaStream_t st) {
  using C = LCfg<B, S>;
  static_assert(C::SMEM <= 227 * 1024, "shared memory");
  // two instances per (b, s): LuArgs::disp picks the dispatch (one kernel holding both paths
  // cost each of them ~1%: C3 LU 166.9 -> 168.2 ms with disp, 168.9 -> 170.3 without)
  const void* fn = a.disp ? (const void*)lu_exec_kernel<B, S, true> : (const void*)lu_exec_kernel<B, S, false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (e != cudaSuccess) return e;
  void* args[] = {(void*)&a};
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(NT), args, C::SMEM, st);
}

template <int B, int S>
static int max_ctas_inst(int device) {
  using C = LCfg<B, S>;
  int nsm = 0, per = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  int per2 = 0;
  if (cudaFuncSetAttribute(lu_exec_kernel<B, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess ||
      cudaFuncSetAttribute(lu_exec_kernel<B, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess)
    return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, lu_exec_kernel<B, S, false>, NT, C::SMEM) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, lu_exec_kernel<B, S, true>, NT, C::SMEM) != cudaSuccess) return 0;
  return nsm * (per < per2 ? per : per2);
}

#define LU_INSTANCES(X) X(256, 32) X(128, 32) X(64, 16)

bool lu_supported(int b, int s) {
#define SUP(BB, SS) if (b == BB && s == SS) return true;
  LU_INSTANCES(SUP)
#undef SUP
  return false;
}
int lu_slice(int b, int s) { return lu_supported(b, s) ? (b < W ? b : W) : 0; }
bool lu_uses_ltilde(int b, int s) {
#define LT_(BB, SS) if (b == BB && s == SS) return LCfg<BB, SS>::LT;
  LU_INSTANCES(LT_)
#undef LT_
  return false;
}
int lu_ltilde_doubles(int b, int s) {
#define LTD(BB, SS) if (b == BB && s == SS) return LCfg<BB, SS>::LTT;
  LU_INSTANCES(LTD)
#undef LTD
  return 0;
}
int lu_perm_ints(int b, int s) { return (b / s) * (4 + 4 * s + 2 * (b + s)); }
int lu_max_ctas(int b, int s, int device) {
#define MC(BB, SS) if (b == BB && s == SS) return max_ctas_inst<BB, SS>(device);
  LU_INSTANCES(MC)
#undef MC
  return 0;
}
cudaError_t launch_lu_exec(int b, int s, const LuArgs& a, int grid, cudaStream_t st) {
#define LI(BB, SS) if (b == BB && s == SS) return launch_inst<BB, SS>(a, grid, st);
  LU_INSTANCES(LI)
#undef LI
  return cudaErrorInvalidValue;
}

}  // namespace lu
}  // namespace tqr
