// tqr_device.cuh -- sm_100a device building blocks of the tiled QR executor.
//
// fp64 on B200: tcgen05 has no f64 kind, so the fp64 tensor-core instruction is the
// warp-level DMMA.8x8x4 (`mma.sync.m8n8k4.f64`).  The M0 probe measured it at
// 37.14 TFLOP/s over 148 SMs (= 64 FMA/clk/SM at 1965 MHz), vs ~34 TFLOP/s for DFMA,
// sharing one pipe (profiles/r01_m0_fp64_probe.txt).  All level-3 work below is DMMA.
//
// Register-resident column groups.  Every update (LARFB, SSRFB, the trailing updates
// inside GEQRT/TSQRT, and apply-Q) is "apply a block reflector (Y_l, T_l) to a set of
// columns".  Each warp owns a group of 8 columns of the target tile and keeps the
// whole b x 8 group in DMMA accumulator registers, transposed: the group is C^T
// (8 x b), accumulator tile t covers tile rows [8t, 8t+8): fragment element h of lane j
// (j = lane&3) holds row 8t + 2j + h, which is both the accumulator's column 2j+h and, for
// the k-step h over rows {8t + 2j + h}, the A-operand index j.  So an accumulator fragment
// is ALSO a valid A-operand fragment for GEMM1 over the same rows, and W^T = C^T Y (GEMM1),
// W^T <- W^T T_l (T multiply) and C^T -= W^T Y^T (GEMM2) chain through registers with no
// shuffles and no shared memory round trip.  Shared memory only holds the reflector panel
// Y_l (b x s, swizzle swy<R>()) and T_l (s x s, swizzle swz<R>()), both bank-conflict-free.
//
// DMMA m8n8k4 fragment layouts (PTX ISA, mma.m8n8k4 .f64):
//   A 8x4 : a0 = A[lane>>2][lane&3]          B 4x8 : b0 = B[lane&3][lane>>2]
//   C 8x8 : c0,c1 = C[lane>>2][2*(lane&3) + {0,1}]
// On the reflector-column side (W, T_l) accumulator column n (0..7) of an 8-wide block maps
// to block-local index phi(n):
//   phi(2j+h) = 4h + j  -> fragment element h of lane (j = lane&3) holds index 4h+j,
// which is exactly the k index (lane&3) of a k-step over indices {4h .. 4h+3}.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace tqr {

// Per-(b, s) CTA shape.  A column group (8 columns) is held by RS warps, each owning
// RW <= 128 consecutive rows (64 accumulator registers at most); for b >= 256 the W
// partials of a group are summed through shared memory under a named barrier.  A CTA has
// 8 warps (up to 255 registers per thread: the executor contains device-function calls,
// and ptxas spilled the accumulators of the inlined update path at a 128-register cap)
// and holds GPS groups = SLICE columns.
template <int B, int S, int RWM = 128>
struct Cfg {
  static constexpr int RW = B < RWM ? B : RWM;  // rows of a column group held by one warp
  static constexpr int RS = B / RW;
  static constexpr int NWARP = 8;  // 255-register budget: no spills in the DMMA paths
  static constexpr int NT = NWARP * 32;
  static constexpr int GPS = NWARP / RS;
  static constexpr int SLICE = 8 * GPS;
  static constexpr int XW = (S / 8) * 2 * 32;  // doubles per warp for a W fragment set
  static constexpr int C1W = 8 * (S + 4);      // doubles per group for a staged C1 block
  static_assert(GPS >= 1 && (RS == 1 || GPS <= 15), "named barriers 1..15");
};

// Internal inner block of the executor for an output blocking (B, SO): the packed panel
// B x SI (double buffered in shared memory) must fit, so b = 512, s = 64 runs with SI = 16
// and assembles the 64 x 64 T_l blocks of its output afterwards (form_t_kernel).
template <int B, int SO>
struct Inner {
  static constexpr int SI = (B * SO <= 8192) ? SO : 8192 / B;
  static_assert(SO % SI == 0, "SI divides SO");
};

__device__ __forceinline__ int phi(int n) { return ((n & 1) << 2) | (n >> 1); }

// f(std::integral_constant<int, I>) for I = 0 .. N-1: register-array indices stay compile-time
// constants inside lambdas (a runtime index would move the array to local memory)
template <int N, int I = 0, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<N, I + 1>(f);
  }
}

// 8x8-block swizzled layout of an R x C operand (R, C multiples of 8): element (r, c) at
// block (r/8, c/8) (blocks column-major), inside the block column-major with the row
// index XOR-ed by (c & 6).  Conflict-free (one wavefront per half warp) for the T-multiply
// patterns (rows 4h+j, cols phi(n)) and (rows phi(n), cols 4h+j).
template <int R>
__device__ __forceinline__ int swz(int r, int c) {
  return ((((c >> 3) * (R >> 3)) + (r >> 3)) << 6) + ((c & 7) << 3) + ((r & 7) ^ (c & 6));
}

// Layout of the packed reflector panels Y (R x C): the same 8x8 blocks, inside a block
// column-major with the row index XOR-ed by xy(c) = (c bit 2) | (c bit 1) << 2.  The
// accumulators map tile row 8t + 2j + h to fragment element h of lane j (see load_cols),
// so GEMM1 reads rows {2j + h} x cols phi(n) and GEMM2 rows n x cols {4h + j}: both are
// conflict-free under xy (the c & 6 swizzle above is conflict-free for the T blocks' pattern).
__device__ __forceinline__ int xy(int c) { return ((c >> 2) & 1) | ((c & 2) << 1); }
template <int R>
__device__ __forceinline__ int swy(int r, int c) {
  return ((((c >> 3) * (R >> 3)) + (r >> 3)) << 6) + ((c & 7) << 3) + ((r & 7) ^ xy(c & 7));
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// L2 residency hints (locality): with TQR_L2HINT=1 the data an SM re-reads
// soon from L2 -- the packed reflector panels Y/T (read by every update task of one (k, i))
// and the C1 row tiles A(k, j) (read and written by the chain S(k, k+1.., j)) -- is loaded /
// stored with an evict_last policy and the C2 tile slices (touched once per step) with
// evict_first.  Measured at C3: DRAM reads 226 -> 207 GB but 0.5% slower (C4 1.1%), so the
// product build leaves it off (plain .cg accesses).
#ifndef TQR_L2HINT
#define TQR_L2HINT 0
#endif
__device__ __forceinline__ unsigned long long pol_keep() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_stream() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_cg2(const double2* p, bool keep) {
#if TQR_L2HINT
  double2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(keep ? pol_keep() : pol_stream()));
  return v;
#else
  return __ldcg(p);
#endif
}
__device__ __forceinline__ void st_cg2(double2* p, double2 v, bool keep) {
#if TQR_L2HINT
  asm volatile("st.global.cg.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
               "l"(keep ? pol_keep() : pol_stream())
               : "memory");
#else
  __stcg(p, v);
#endif
}
__device__ __forceinline__ void st_cg1(double* p, double v, bool keep) {
#if TQR_L2HINT
  asm volatile("st.global.cg.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(keep ? pol_keep() : pol_stream())
               : "memory");
#else
  __stcg(p, v);
#endif
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// cp.async of 16 bytes kept in L2 (evict_last): the C1 row tiles
__device__ __forceinline__ void cp_async16_keep(void* smem, const void* gmem) {
#if TQR_L2HINT
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol_keep())
               : "memory");
#else
  cp_async16(smem, gmem);
#endif
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ---- TMA bulk copies (cp.async.bulk -> SASS UBLKCP) completing on an mbarrier ----------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
#if TQR_L2HINT  // reflector panels: evict_last (re-read by every update task of the panel)
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol_keep())
      : "memory");
#else
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
#endif
}
// L2 prefetch of a contiguous global range (bytes % 16 == 0, 16-byte aligned); no SMEM, no
// completion tracking -- a hint that turns the next task's HBM reads into L2 hits
__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes, bool keep = false) {
  // issued in chunks of <= 64 KiB
  const char* p = static_cast<const char*>(src);
  for (unsigned off = 0; off < bytes; off += 65536u) {
    const unsigned n = bytes - off < 65536u ? bytes - off : 65536u;
#if TQR_L2HINT
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p + off), "r"(n),
                 "l"(keep ? pol_keep() : pol_stream())
                 : "memory");
#else
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + off), "r"(n) : "memory");
#endif
  }
}
// order this thread's generic-proxy accesses before subsequent async-proxy (TMA) accesses
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// system scope: counters written by peer GPUs over NVLink (multi-GPU)
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// Sums of N values (N a power of two <= 32) over the 32 lanes, every lane receiving all N sums,
// with fewer shuffles than N butterflies (5N): a reduce-scatter over lane bits 4, 3, ... (each
// level halves the values a lane carries), a butterfly over the remaining bits, and N
// broadcasts -- 2N - 1 + (5 - log2 N) shuffles (N = 4: 10 instead of 20).  The panel's
// off-critical-path column updates are shuffle-bound (they share the SM with the critical
// column's reductions).  Every sum is formed in one fixed order on every lane (deterministic).
template <int N>
__device__ __forceinline__ void warp_allreduce(double (&v)[N]) {
  static_assert(N >= 1 && N <= 32 && (N & (N - 1)) == 0, "N: power of two");
  const int lane = threadIdx.x & 31;
  constexpr int K = N == 1 ? 0 : N == 2 ? 1 : N == 4 ? 2 : N == 8 ? 3 : N == 16 ? 4 : 5;
  double r[N];
#pragma unroll
  for (int i = 0; i < N; ++i) r[i] = v[i];
#pragma unroll
  for (int lv = 0; lv < K; ++lv) {  // level lv: lane bit (4 - lv) selects the half kept
    const int o = 16 >> lv, half = N >> (lv + 1);
    const bool up = lane & o;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = up ? r[i] : r[i + half];
      const double keep = up ? r[i + half] : r[i];
      r[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (int o = 16 >> K; o > 0; o >>= 1) r[0] += __shfl_xor_sync(0xffffffffu, r[0], o);
  // lane L now holds sum c with bit (K-1-lv) of c = lane bit (4-lv)
#pragma unroll
  for (int c = 0; c < N; ++c) {
    int src = 0;
#pragma unroll
    for (int lv = 0; lv < K; ++lv) src |= ((c >> (K - 1 - lv)) & 1) << (4 - lv);
    v[c] = __shfl_sync(0xffffffffu, r[0], src);
  }
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// ---------------------------------------------------------------------------------------
// Column-group register I/O.  acc[t][h] <-> C[8t + 2(lane&3) + h][col0 + (lane>>2)] of a
// column-major tile with leading dimension B: the two elements of a lane are adjacent rows,
// so every access is one 16-byte LDG/STG (half the instructions and L1 wavefronts of the
// 4h + j row map).  DMMA k-step h of 8-row block t therefore covers rows {8t + 2j + h}.
// Global tile data is always read with .cg (L2, never L1): tiles are rewritten by other CTAs
// during the persistent launch.
// ---------------------------------------------------------------------------------------
// acc covers rows [8*t0, 8*t0 + RW) of the tile.
template <int B, int RW>
__device__ __forceinline__ void load_cols(double (&acc)[RW / 8][2], const double* tile, int col0, int t0,
                                          bool keep = false) {
  const int lane = threadIdx.x & 31;
  const double2* col = reinterpret_cast<const double2*>(tile + (size_t)(col0 + (lane >> 2)) * B + 8 * t0 + 2 * (lane & 3));
#pragma unroll
  for (int t = 0; t < RW / 8; ++t) {
    const double2 v = ld_cg2(col + 4 * t, keep);
    acc[t][0] = v.x;
    acc[t][1] = v.y;
  }
}
template <int B, int RW>
__device__ __forceinline__ void store_cols(const double (&acc)[RW / 8][2], double* tile, int col0, int t0,
                                           bool keep = false) {
  const int lane = threadIdx.x & 31;
  double2* col = reinterpret_cast<double2*>(tile + (size_t)(col0 + (lane >> 2)) * B + 8 * t0 + 2 * (lane & 3));
#pragma unroll
  for (int t = 0; t < RW / 8; ++t) st_cg2(col + 4 * t, make_double2(acc[t][0], acc[t][1]), keep);
}
// w[u][h] <-> C1[row0 + 8u + 4h + (lane&3)][col0 + (lane>>2)]  (s rows of the "top" tile)
template <int B, int S>
__device__ __forceinline__ void load_top(double (&w)[S / 8][2], const double* tile, int row0, int col0) {
  const int lane = threadIdx.x & 31;
  const double* col = tile + (size_t)(col0 + (lane >> 2)) * B + row0 + (lane & 3);
#pragma unroll
  for (int u = 0; u < S / 8; ++u) {
    w[u][0] = __ldcg(col + 8 * u);
    w[u][1] = __ldcg(col + 8 * u + 4);
  }
}
// per-warp shared-memory copy of a W-shaped fragment set (lane-interleaved: conflict-free)
// C1 block of one column group in shared memory: column n (0..7) at n*(S+4), rows
// contiguous (one 16-byte-aligned bulk copy per column); fragment (u, h) of lane reads
// element (row 8u+4h+j, column n) -> conflict-free (stride S+4 = 4 mod 16 doubles).
template <int S>
__device__ __forceinline__ int c1_idx(int u, int h, int lane) {
  return (lane >> 2) * (S + 4) + 8 * u + 4 * h + (lane & 3);
}
template <int S>
__device__ __forceinline__ void c1_put(double* c1s, const double (&w)[S / 8][2]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < S / 8; ++u) { c1s[c1_idx<S>(u, 0, lane)] = w[u][0]; c1s[c1_idx<S>(u, 1, lane)] = w[u][1]; }
}
template <int S>
__device__ __forceinline__ void frag_put(double* st, const double (&w)[S / 8][2]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < S / 8; ++u) { st[(2 * u) * 32 + lane] = w[u][0]; st[(2 * u + 1) * 32 + lane] = w[u][1]; }
}

// ---------------------------------------------------------------------------------------
// Block-reflector apply on one warp's column group (PAPER.md:395-402 DLARFB and
// PAPER.md:430-466 DSSRFB, per inner block l; readings R1, R5):
//   W   = C1 + Y_l^T C            (w holds C1, or 0, on entry; GEMM1)
//   W  <- T_l^T W  (QT)  or  T_l W (!QT)
//   C  -= Y_l W                   (GEMM2)
// Rows of Y outside the reflector block are explicit zeros in shared memory (no branches in
// the unrolled DMMA loops).  All three products are DMMA.8x8x4 chains through registers.
// ---------------------------------------------------------------------------------------
template <int B, int S, int RW>
__device__ __forceinline__ void gemm1(const double (&acc)[RW / 8][2], double (&w)[S / 8][2],
                                      const double* __restrict__ Ys, int t0) {
  const int lane = threadIdx.x & 31, j = lane & 3, pn = phi(lane >> 2);
  // W^T[8 x S] += C^T[8 x RW] * Y[RW x S]   (this warp's rows; 4 independent chains)
#pragma unroll
  for (int t = 0; t < RW / 8; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < S / 8; ++u) dmma(w[u], acc[t][h], Ys[swy<B>(8 * (t0 + t) + 2 * j + h, 8 * u + pn)]);
}

// Fused T multiply + C1 store + GEMM2, software-pipelined.  QT (W <- T_l^T W): column block
// u2 of W^T T_l needs only w[0..u2] (T_l upper triangular) and GEMM2's k-steps over u = u2
// need only that block, so blocks are finished in the order u2 = 0, 1, ... and block u2+1's
// T-multiply DMMAs are issued between GEMM2's DMMAs for u2 instead of draining the pipe
// before GEMM2 starts (per block and warp: a chain of up to 2 s/8 dependent DMMAs that both
// warps of an SMSP would otherwise wait out together).  !QT (W <- T_l W, apply Q): block u2
// needs w[u2..], so the order is u2 = NU-1, ..., 0.  Each block's T products are summed over
// (u, h) ascending; GEMM2 (C^T += (-W)^T Y^T, accumulators chained per row block t) runs its
// k-steps in the block order.
// LD: leading dimension of the C1 tile `top` (== B, the panel's rows, except for the tall
// units of DESIGN.md R30, whose 2b-row panels update b-row C1 tiles)
template <int B, int S, int RW, bool QT, int LD = B>
__device__ __forceinline__ void tmul_gemm2(double (&acc)[RW / 8][2], const double (&w)[S / 8][2],
                                           const double* __restrict__ Ys, const double* __restrict__ Ts,
                                           const double* c1s, double* top, int row0, int col0, int t0,
                                           bool store_c1) {
  const int lane = threadIdx.x & 31, j = lane & 3, pn = phi(lane >> 2), g = lane >> 2;
  constexpr int NU = S / 8, TT = RW / 8;
  double wn[NU][2];
#pragma unroll
  for (int u = 0; u < NU; ++u) { wn[u][0] = 0.0; wn[u][1] = 0.0; }
  // x-th block finished (x = 0 .. NU-1) and its T-multiply step q: (u, h)
  auto blk = [](int x) { return QT ? x : NU - 1 - x; };
  auto nsteps = [](int u2) { return QT ? 2 * (u2 + 1) : 2 * (NU - u2); };
  auto tmul_step = [&](int u2, int q) __attribute__((always_inline)) {
    const int u = (QT ? 0 : u2) + (q >> 1), h = q & 1;
    const double tv = QT ? Ts[swz<S>(8 * u + 4 * h + j, 8 * u2 + pn)] : Ts[swz<S>(8 * u2 + pn, 8 * u + 4 * h + j)];
    dmma(wn[u2], w[u][h], tv);
  };
  auto finish = [&](int u2) __attribute__((always_inline)) {  // C1 -= W (block u2), negate
    if (store_c1) {
      double* col = top + (size_t)(col0 + g) * LD + row0 + j;
      st_cg1(col + 8 * u2, c1s[c1_idx<S>(u2, 0, lane)] - wn[u2][0], true);      // C1: kept in L2
      st_cg1(col + 8 * u2 + 4, c1s[c1_idx<S>(u2, 1, lane)] - wn[u2][1], true);
    }
    wn[u2][0] = -wn[u2][0];
    wn[u2][1] = -wn[u2][1];
  };
#pragma unroll
  for (int q = 0; q < nsteps(blk(0)); ++q) tmul_step(blk(0), q);
  finish(blk(0));
#pragma unroll
  for (int x = 0; x < NU; ++x) {
    const int u = blk(x);
    const bool more = x + 1 < NU;
    const int un = more ? blk(x + 1) : 0, nn = more ? nsteps(un) : 0;
    // GEMM2 k-steps (u, h) over all row blocks t; the next block's T-multiply DMMAs are
    // spread over them (one per 4 GEMM2 DMMAs), the rest (TT/4 < nn) issued after
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        dmma(acc[t], wn[u][h], Ys[swy<B>(8 * (t0 + t) + g, 8 * u + 4 * h + j)]);
        if (more && h == 0 && (t & 3) == 3 && (t >> 2) < nn) tmul_step(un, t >> 2);
      }
    if (more) {
#pragma unroll
      for (int q = TT / 4; q < nn; ++q) tmul_step(un, q);
      finish(un);
    }
  }
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// C1 <- C1 - W with C1 held in registers (fragment layout of w)
template <int B, int S>
__device__ __forceinline__ void store_top_minus_r(const double (&c1)[S / 8][2], const double (&wn)[S / 8][2],
                                                  double* tile, int row0, int col0) {
  const int lane = threadIdx.x & 31;
  double* col = tile + (size_t)(col0 + (lane >> 2)) * B + row0 + (lane & 3);
#pragma unroll
  for (int u = 0; u < S / 8; ++u) {
    __stcg(col + 8 * u, c1[u][0] - wn[u][0]);
    __stcg(col + 8 * u + 4, c1[u][1] - wn[u][1]);
  }
}

// One column group's block-reflector apply (all RS warps of group gi call it together):
//   W = [C1] + Y^T C (row partials summed in a fixed order);  W <- T^{T|1} W;
//   [C1 -= W to global];  C -= Y W.
// c1: the group's C1 block in registers (fragment layout of w; used by rpart 0 only);
// top/row0: where C1 - W is stored.  xg: the group's RS partial buffers.  BAR2 protects
// xg when the caller reuses it before all warps of the group have read it.
template <int B, int S, int RW, int RS, bool QT, bool BAR2, int LD = B>
__device__ __forceinline__ void group_apply(double (&acc)[RW / 8][2], const double* __restrict__ Ys,
                                            const double* __restrict__ Ts, const double* c1s, double* top,
                                            int row0, int col0, int t0, int gi, int rpart, double* xg) {
  const int lane = threadIdx.x & 31;
  const bool HAS_C1 = top != nullptr;  // SSRFB / TSQRT type: C1 block staged in c1s
  constexpr int XW = (S / 8) * 2 * 32;
  double w[S / 8][2];
#pragma unroll
  for (int u = 0; u < S / 8; ++u) {
    w[u][0] = (HAS_C1 && rpart == 0) ? c1s[c1_idx<S>(u, 0, lane)] : 0.0;
    w[u][1] = (HAS_C1 && rpart == 0) ? c1s[c1_idx<S>(u, 1, lane)] : 0.0;
  }
  gemm1<B, S, RW>(acc, w, Ys, t0);
  if (RS > 1) {
    frag_put<S>(xg + rpart * XW, w);
    named_bar(1 + gi, 32 * RS);
#pragma unroll
    for (int u = 0; u < S / 8; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double x = xg[(2 * u + h) * 32 + lane];
#pragma unroll
        for (int r = 1; r < RS; ++r) x += xg[r * XW + (2 * u + h) * 32 + lane];
        w[u][h] = x;
      }
    if (BAR2) named_bar(1 + gi, 32 * RS);
  }
  tmul_gemm2<B, S, RW, QT, LD>(acc, w, Ys, Ts, c1s, top, row0, col0, t0, HAS_C1 && rpart == 0);
}

// Warp-local cp.async of one group's C1 block (rows [row0, row0+S), 8 columns from col0)
// into c1s (c1_idx layout: column n at n*(S+4)); 16-byte chunks, S/2 per column.
template <int B, int S>
__device__ __forceinline__ void c1_fetch(double* c1s, const double* tile, int row0, int col0) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = lane; q < 8 * (S / 2); q += 32) {
    const int n = q / (S / 2), r2 = 2 * (q % (S / 2));
    cp_async16_keep(c1s + n * (S + 4) + r2, tile + (size_t)(col0 + n) * B + row0 + r2);
  }
  cp_async_commit();
}

// ---------------------------------------------------------------------------------------
// Panel factorization of one inner block (s columns) in shared memory: dgeqr2-style,
// rank-1 per column (R7), warp-shuffle norms and dot products.
//
//   TS = true  (TSQRT): P rows [0, B) of the block's columns; the column's
//              "top" lives in Rb (the s x s diagonal block of R, upper triangle); the
//              reflector is [e_c; v], identity tops are mutually orthogonal.
//   TS = false (GEQRT): P holds the tile rows, block columns; column jj's
//              alpha is P[c0+jj][jj], its x is P[c0+jj+1 :][jj].
// P column c at P + c*LDP.  Column c belongs to warp c % NW and only that warp writes it.
// No block-wide barrier inside the column loop: the owner warp of column jj publishes v_jj
// (in place, P column jj is final once generated), tau_jj and beta_jj, then ARRIVES (release,
// no wait) on column jj's mbarrier pmb[jj]; every other warp waits on that mbarrier alone
// (acquire) before applying reflector jj to its own columns.  A named barrier would complete
// only when EVERY warp arrived, so each column would wait for the slowest warp's off-path
// updates of the previous column (1407 -> 1229 clk per column, tools/panel_bench.cu).  The
// owner of column jj+1 updates that column first and immediately generates the next
// reflector, so the critical path per column is one dot/update plus one Householder
// generation; the other warps' columns are updated off the critical path with their
// reductions interleaved.
// Householder generator = DESIGN.md R2-R4 (the oracle's), v = x * (1/(alpha-beta)).
// Outputs: P holds V_l (below the diagonal for GEQRT), Rb / P's upper part the new R
// entries, tau[S].
// ---------------------------------------------------------------------------------------
// pmb: S mbarriers (one arrival each), initialised once per launch (pmb_init); every call
// completes each of them exactly once, so call number g of the CTA waits on parity g & 1.
template <int B, int S, int NW, int LDP>
__device__ __forceinline__ void panel_factor(double* P, int c0, double* Rb, double* tau, const bool TS,
                                             unsigned long long* pmb, unsigned parity) {
  static_assert(S <= 64, "top block rows: two per lane at most");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NR = (B + 31) / 32;       // x-part rows per lane: row r = lane + 32 q
  constexpr int NC = (S + NW - 1) / NW;   // columns per warp: column c = warp + NW ci
  constexpr int NTR = (S + 31) / 32;      // top-block rows per lane: block row L = lane + 32 h
  // Column c of the panel = [top block (S rows); x part].  TSQRT: top = R_kk's diagonal block
  // (Rb, upper triangle), x = the B rows of A(i,k); the reflector is [e_j; v_j].  GEQRT: top =
  // tile rows [c0, c0+S), x = tile rows [c0+S, B); the reflector is [0; 1; v_j] with v_j's
  // leading part inside the top block.  Every warp keeps its columns in registers (x and
  // top), so no register row index is ever dynamic (row jj of the top block is a shuffle
  // from lane jj) and no column step touches shared memory except v_j.
  const int lox = TS ? 0 : c0 + S;  // first x-part row
  double x[NC][NR], tr[NC][NTR];
#pragma unroll
  for (int ci = 0; ci < NC; ++ci) {
    const int c = warp + NW * ci;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      x[ci][q] = (c < S && r >= lox && r < B) ? P[r + c * LDP] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < NTR; ++h) {
      const int L = lane + 32 * h;
      tr[ci][h] = (c < S && L < S && (!TS || L <= c)) ? (TS ? Rb[L + c * S] : P[c0 + L + c * LDP]) : 0.0;
    }
  }
  // block row L of column CI, broadcast to the warp
  auto getT = [&](auto CI, int L) __attribute__((always_inline)) -> double {
    constexpr int ci = decltype(CI)::value;
    const double t = (NTR == 1 || L < 32) ? tr[ci][0] : tr[ci][NTR - 1];
    return __shfl_sync(0xffffffffu, t, L & 31);
  };
  auto subT = [&](auto CI, int L, double w) __attribute__((always_inline)) {
    constexpr int ci = decltype(CI)::value;
    if (lane == (L & 31)) {
      if (NTR == 1 || L < 32) tr[ci][0] -= w; else tr[ci][NTR - 1] -= w;
    }
  };

  // Householder generation (R2-R4, R17, R20) for column jj (in CI) from alpha and
  // sigma = ||x||^2 over its rows below the pivot; stores v into P, beta, tau; publishes.
  auto house_pub = [&](auto CI, int jj, double alpha, double sigma) __attribute__((always_inline)) {
    constexpr int ci = decltype(CI)::value;
    double beta, tv, scale;
    if (sigma == 0.0) {
      beta = alpha; tv = 0.0; scale = 0.0;
    } else {
      const double nn = alpha * alpha + sigma;
      const double rn = rsqrt(nn);                // 1/nu
      const double nu = nn * rn;
      beta = (alpha >= 0.0) ? -nu : nu;
      tv = 1.0 + fabs(alpha) * rn;                 // (beta - alpha)/beta = 1 + |alpha|/nu
      scale = __drcp_rn(alpha - beta);             // correctly rounded, == 1.0 / (alpha - beta)
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      if (r >= lox && r < B) P[r + jj * LDP] = x[ci][q] * scale;
    }
    if (!TS) {
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        const int L = lane + 32 * h;
        if (L > jj && L < S) P[c0 + L + jj * LDP] = tr[ci][h] * scale;
      }
    }
    if (lane == 0) {
      if (TS) Rb[jj + jj * S] = beta; else P[c0 + jj + jj * LDP] = beta;
      tau[jj] = tv;
    }
    __syncwarp();                          // the warp's stores of v_jj, tau_jj, beta_jj ...
    if (lane == 0) mbar_arrive(pmb + jj);  // ... published (release); the owner does not wait
  };
  // ||column CI below block row j||^2: x part, plus (GEQRT) top-block rows L > j
  auto norm_below = [&](auto CI, int j) __attribute__((always_inline)) -> double {
    constexpr int ci = decltype(CI)::value;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      if (q & 1) s1 += x[ci][q] * x[ci][q]; else s0 += x[ci][q] * x[ci][q];
    }
    if (!TS) {
#pragma unroll
      for (int h = 0; h < NTR; ++h) {
        const int L = lane + 32 * h;
        if (L > j && L < S) s0 += tr[ci][h] * tr[ci][h];
      }
    }
    return warp_sum(s0 + s1);
  };

  if (warp == 0) {
    const std::integral_constant<int, 0> C0;
    const double sg = norm_below(C0, 0);
    house_pub(C0, 0, getT(C0, 0), sg);
  }
  for (int jj = 0; jj + 1 < S; ++jj) {
    if (warp != jj % NW) mbar_wait(pmb + jj, parity);  // v_jj published (acquire)
    const double tj = tau[jj];
    double vr[NR], vt[NTR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = lane + 32 * q;
      vr[q] = (r >= lox && r < B) ? P[r + jj * LDP] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < NTR; ++h) {  // v_jj inside the top block (GEQRT only; TSQRT: e_jj)
      const int L = lane + 32 * h;
      vt[h] = (!TS && L > jj && L < S) ? P[c0 + L + jj * LDP] : 0.0;
    }
    const int nxt = jj + 1;
    if (nxt % NW == warp) {
      // Critical path: update column jj+1 and generate reflector jj+1.  One interleaved
      // reduction of (x.v, x.x, v.v) over the rows below the pivot jj gives the dot product
      // AND the new norm by downdating, sigma' = x.x - 2 tw x.v + tw^2 v.v [- alpha'^2 for
      // GEQRT, whose alpha' is one of those rows]; if it may have cancelled (below 5% of the
      // magnitude of its terms) it is recomputed from the updated column (R20).
      static_for<NC>([&](auto CI) __attribute__((always_inline)) {
        constexpr int ci = decltype(CI)::value;
        if (warp + NW * ci != nxt) return;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          if (q & 1) { a1 += vr[q] * x[ci][q]; b1 += x[ci][q] * x[ci][q]; e1 += vr[q] * vr[q]; }
          else { a0 += vr[q] * x[ci][q]; b0 += x[ci][q] * x[ci][q]; e0 += vr[q] * vr[q]; }
        }
        if (!TS) {
#pragma unroll
          for (int h = 0; h < NTR; ++h) {
            const int L = lane + 32 * h;
            const double tv_ = (L > jj && L < S) ? tr[ci][h] : 0.0;
            a0 += vt[h] * tv_; b0 += tv_ * tv_; e0 += vt[h] * vt[h];
          }
        }
        double sxv = a0 + a1, sxx = b0 + b1, svv = e0 + e1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          sxv += __shfl_xor_sync(0xffffffffu, sxv, o);
          sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
          svv += __shfl_xor_sync(0xffffffffu, svv, o);
        }
        const double tw = tj * (getT(CI, jj) + sxv);
#pragma unroll
        for (int q = 0; q < NR; ++q) x[ci][q] -= tw * vr[q];
#pragma unroll
        for (int h = 0; h < NTR; ++h) tr[ci][h] -= tw * vt[h];
        subT(CI, jj, tw);
        const double alpha = getT(CI, nxt);
        const double a2 = TS ? 0.0 : alpha * alpha;
        double sigma = sxx - 2.0 * tw * sxv + tw * tw * svv - a2;
        const double mag = sxx + 2.0 * fabs(tw * sxv) + tw * tw * svv + a2;
        if (!(sigma >= 0.05 * mag)) sigma = norm_below(CI, nxt);  // possible cancellation / NaN
        house_pub(CI, nxt, alpha, sigma);
      });
    }
    // the warp's other columns c > jj+1: dots, one interleaved butterfly, register updates
#ifdef TQR_PF_SKIP_NONCRIT  // tools/panel_bench.cu timing experiment only (wrong results)
    continue;
#endif
    double dc[NC];
#pragma unroll
    for (int ci = 0; ci < NC; ++ci) {
      const int c = warp + NW * ci;
      double d0 = 0.0, d1 = 0.0;
      if (c > nxt && c < S) {
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          if (q & 1) d1 += vr[q] * x[ci][q]; else d0 += vr[q] * x[ci][q];
        }
#pragma unroll
        for (int h = 0; h < NTR; ++h) d0 += vt[h] * tr[ci][h];
      }
      dc[ci] = d0 + d1;
    }
    warp_allreduce<NC>(dc);
    static_for<NC>([&](auto CI) __attribute__((always_inline)) {
      constexpr int ci = decltype(CI)::value;
      const int c = warp + NW * ci;
      if (c > nxt && c < S) {
        const double tw = tj * (getT(CI, jj) + dc[ci]);
#pragma unroll
        for (int q = 0; q < NR; ++q) x[ci][q] -= tw * vr[q];
#pragma unroll
        for (int h = 0; h < NTR; ++h) tr[ci][h] -= tw * vt[h];
        subT(CI, jj, tw);
      }
    });
  }
  // R entries above the diagonal of the top block back to shared memory (the diagonal (beta)
  // and V were stored by house_pub)
#pragma unroll
  for (int ci = 0; ci < NC; ++ci) {
    const int c = warp + NW * ci;
#pragma unroll
    for (int h = 0; h < NTR; ++h) {
      const int L = lane + 32 * h;
      if (c < S && L < c) {
        if (TS) Rb[L + c * S] = tr[ci][h]; else P[c0 + L + c * LDP] = tr[ci][h];
      }
    }
  }
  __syncthreads();
}

// Gram matrix of the staged panel (DLARFT dot products): Z[a + b*S] = Y[:, a]^T Y[:, b]
// for the upper block triangle, by DMMA on the swizzled Ys (GEQRT: Y = U_l with its unit
// diagonal and zeros above; TSQRT: Y = V_l, identity tops orthogonal).
template <int B, int S, int NW>
__device__ void gram_upper(const double* __restrict__ Ys, double* Z) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, j = lane & 3, pn = phi(lane >> 2);
  constexpr int NU = S / 8, NTILE = NU * (NU + 1) / 2;
  for (int tile = warp; tile < NTILE; tile += NW) {
    int u1 = 0, rem = tile;
    while (rem >= NU - u1) { rem -= NU - u1; ++u1; }
    const int u2 = u1 + rem;
    // four independent accumulator chains (B/8 x 2 k-steps), summed in a fixed order
    double g[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 4
    for (int t = 0; t < B / 8; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double a = Ys[swy<B>(8 * t + 2 * j + h, 8 * u1 + pn)];
        const double bb = Ys[swy<B>(8 * t + 2 * j + h, 8 * u2 + pn)];
        dmma(g[(t & 1) * 2 + h], a, bb);
      }
    // element (m = lane>>2, n = 2j+h): Z[8u1 + phi(m)][8u2 + phi(2j+h)], phi(2j+h) = 4h+j
#pragma unroll
    for (int h = 0; h < 2; ++h)
      Z[(8 * u1 + pn) + (8 * u2 + 4 * h + j) * S] = (g[0][h] + g[1][h]) + (g[2][h] + g[3][h]);
  }
}

// T_l from tau and the Gram matrix Z (forward column-wise DLARFT; the
// oracle's larft_column recurrence):
//   T[j][j] = tau_j ;  T[t][j] = -tau_j * sum_{t'=t}^{j-1} T[t][t'] Z[t'][j]
// Row t of T only needs row t itself (and Z), so each lane computes one row in registers
// with no cross-lane dependency: lane t of warp w owns row 32w + t.  Called by warps
// 0 .. ceil(S/32)-1.  Tp: S x S plain column-major.
template <int S>
__device__ __forceinline__ void build_t(double* Tp, const double* tau, const double* Z) {
  const int t = threadIdx.x;  // row of T (threads >= S compute nothing useful)
  double row[S];
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const double tj = tau[j];
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int tp = 0; tp < j; ++tp) {  // row[tp] == 0 for tp < t
      if (tp & 1) a1 += row[tp] * Z[tp + j * S]; else a0 += row[tp] * Z[tp + j * S];
    }
    row[j] = (j == t) ? tj : (j > t ? -tj * (a0 + a1) : 0.0);
  }
  if (t < S) {
#pragma unroll
    for (int j = 0; j < S; ++j) Tp[t + j * S] = row[j];
  }
}

// T_l by 8 x 8 blocks (the same forward column-wise T as build_t; R27): the
// diagonal blocks T_bb by the row recurrence of build_t restricted to block b (warp b, one row
// per lane), then block column by block column (Schreiber / Van Loan)
//     T[0:8b, b] = -T[0:8b, 0:8b] (Z[0:8b, b] T_bb)
// as 8 x 8 x 8 DMMA tile products (two m8n8k4 k-steps each).  Called by warps 0 .. S/8 - 1
// (named barrier `bar` over them); Tp: S x S column-major (zeros below the diagonal), Z: the
// Gram matrix (upper block triangle), M: (S - 8) x 8 doubles of scratch.
// 8 x 8 tile product D (+)= X * Y, X and Y column-major in shared memory (leading dims lx, ly);
// accumulator element (lane >> 2, 2 (lane & 3) + h) in d[h].
__device__ __forceinline__ void tile_mma8(double (&d)[2], const double* X, int lx, const double* Y, int ly) {
  const int lane = threadIdx.x & 31, m = lane >> 2, k = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 8; kk += 4) dmma(d, X[m + (kk + k) * lx], Y[(kk + k) + m * ly]);
}
template <int S>
__device__ __forceinline__ void build_t_blocked(double* Tp, const double* tau, const double* Z, double* M, int bar) {
  constexpr int NB = S / 8;
  static_assert(S % 8 == 0, "8 x 8 blocks");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = lane >> 2, n0 = 2 * (lane & 3);
  // zero the strictly lower blocks, then the diagonal blocks (warp b: block b)
  for (int e = threadIdx.x; e < S * S; e += 32 * NB) {
    const int r = e % S, c = e / S;
    if (r / 8 > c / 8) Tp[e] = 0.0;
  }
  {
    const int b = warp, t = lane & 7;
    double row[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double tj = tau[8 * b + j];
      double acc = 0.0;
#pragma unroll
      for (int tp = 0; tp < j; ++tp) acc += row[tp] * Z[(8 * b + tp) + (8 * b + j) * S];
      row[j] = (j == t) ? tj : (j > t ? -tj * acc : 0.0);
    }
    if (lane < 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) Tp[(8 * b + t) + (8 * b + j) * S] = row[j];
    }
  }
  if (NB == 1) return;
  named_bar(bar, 32 * NB);
  for (int b = 1; b < NB; ++b) {
    const double* Tbb = Tp + 8 * b + 8 * b * S;
    if (warp < b) {  // M_c = Z_cb T_bb, c = warp
      double d[2] = {0.0, 0.0};
      tile_mma8(d, Z + 8 * warp + 8 * b * S, S, Tbb, S);
      M[(8 * warp + m) + n0 * (S - 8)] = d[0];
      M[(8 * warp + m) + (n0 + 1) * (S - 8)] = d[1];
    }
    named_bar(bar, 32 * NB);
    if (warp < b) {  // T_ab = -sum_{c = a}^{b-1} T_ac M_c, a = warp
      double d[2] = {0.0, 0.0};
      for (int c = warp; c < b; ++c) tile_mma8(d, Tp + 8 * warp + 8 * c * S, S, M + 8 * c, S - 8);
      Tp[(8 * warp + m) + (8 * b + n0) * S] = -d[0];
      Tp[(8 * warp + m) + (8 * b + n0 + 1) * S] = -d[1];
    }
    named_bar(bar, 32 * NB);
  }
}

}  // namespace tqr
