// tqr_exec.cu -- persistent DAG executor and layout kernels (sm_100a).
//
// The paper runs the tasks of Algorithm 1 out of order on CPU
// threads that pick ready tasks by priority.  Here one persistent
// CTA per SM (co-resident cooperative launch) takes tickets in a host-computed
// topological order (list schedule with the paper's G > T > L > S priorities) and waits
// on per-chain monotone progress counters (acquire) before running the task; on
// completion it publishes its counter (release).  Task granularity: GEQRT(k) and
// TSQRT(k,i) are whole-tile single-CTA tasks; LARFB and SSRFB are split into 64-column
// slices (one 8-column group per warp, register resident).
#include "tqr_device.cuh"
#include "tqr_internal.h"

namespace tqr {

template <int B, int S>
struct Layout {
  using C = Cfg<B, S>;
  static constexpr int YSZ = B * S;          // one Y buffer
  static constexpr int TSZ = S * S;
  static constexpr int Y0 = 0, Y1 = YSZ;     // Y[2]
  static constexpr int T0 = 2 * YSZ, T1 = 2 * YSZ + TSZ;
  static constexpr int RB = 2 * YSZ + 2 * TSZ;
  static constexpr int ZZ = RB + TSZ;
  static constexpr int TAU = ZZ + TSZ;
  static constexpr int STASH = TAU + S;                       // C1 block, one per group
  static constexpr int XBUF = STASH + C::GPS * C::XW;         // W partials, one per warp
  static constexpr int TOTAL = XBUF + (C::RS > 1 ? C::NWARP * C::XW : 0);
  static constexpr size_t BYTES = (size_t)TOTAL * sizeof(double);
  static_assert(BYTES <= 232448, "shared memory budget");
};

__device__ __forceinline__ double* tile_ptr(double* base, int i, int j, int p, int B) {
  return base + ((size_t)i + (size_t)j * p) * (size_t)B * B;
}
__device__ __forceinline__ double* tslot_ptr(double* base, int i, int k, int p, int B, int S) {
  return base + ((size_t)i + (size_t)k * p) * (size_t)S * B;
}

// One column group's block-reflector apply for the warps of group gi (rows part rpart):
//   W = [C1 +] Y^T C  (partials summed over the group);  W <- T^{T|1} W;  [C1 -= W];  C -= Y W
// HAS_TOP: SSRFB/TSQRT-type (C1 = rows [row0, row0+S) of `top`, col0.. of the group).
template <int B, int S, bool QT, bool HAS_TOP>
__device__ __forceinline__ void group_apply(double* sm, double (&acc)[Cfg<B, S>::RW / 8][2], const double* Ys,
                                            const double* Ts, double* top, int row0, int col0, int t0, int tlo,
                                            int gi, int rpart) {
  using C = Cfg<B, S>;
  using L = Layout<B, S>;
  double w[S / 8][2], wn[S / 8][2];
  double* st = sm + L::STASH + gi * C::XW;
  if (HAS_TOP && rpart == 0) {
    load_top<B, S>(w, top, row0, col0);
    frag_put<S>(st, w);
  } else {
#pragma unroll
    for (int u = 0; u < S / 8; ++u) { w[u][0] = 0.0; w[u][1] = 0.0; }
  }
  apply_cg_w<B, S, C::RW, QT>(acc, w, wn, Ys, Ts, t0, tlo);
  group_reduce<C::RS, S>(w, sm + L::XBUF + gi * C::RS * C::XW, rpart, gi);
  t_multiply<S, QT>(w, wn, Ts);
  if (HAS_TOP && rpart == 0) store_top_minus<B, S>(st, wn, top, row0, col0);
  negate<S>(wn);
  apply_cg_c<B, S, C::RW>(acc, wn, Ys, t0, tlo);
}

// ---------------------------------------------------------------------------------------
// GEQRT(k): per inner block l, panel of rows [c0,B) x cols [c0,c0+S),
// T_l, then the LARFB-type update of columns [c0+S, B) (rows >= c0).
// ---------------------------------------------------------------------------------------
template <int B, int S>
__device__ __noinline__ void task_geqrt(double* sm, double* Akk, double* Tk) {
  using C = Cfg<B, S>;
  using L = Layout<B, S>;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int gi = warp / C::RS, rpart = warp % C::RS, t0 = rpart * (C::RW / 8);
  double* P = sm + L::Y1;
  double* Ys = sm + L::Y0;
  double* Tp = sm + L::T1;
  double* Ts = sm + L::T0;
  double* Z = sm + L::ZZ;
  double* tau = sm + L::TAU;
  for (int l = 0; l < B / S; ++l) {
    const int c0 = l * S, nrows = B - c0;
    for (int e = tid; e < nrows * S; e += C::NT) {
      const int r = e % nrows, c = e / nrows;
      P[r + c * B] = __ldcg(Akk + (size_t)(c0 + c) * B + c0 + r);
    }
    __syncthreads();
    panel_factor<B, S, C::NWARP, false>(P, nrows, nullptr, tau, Z);
    if (warp == 0) build_t<S>(Tp, tau, Z);
    __syncthreads();
    for (int e = tid; e < nrows * S; e += C::NT) {
      const int r = e % nrows, c = e / nrows;
      const double v = P[r + c * B];
      __stcg(Akk + (size_t)(c0 + c) * B + c0 + r, v);
      Ys[swz<B>(c0 + r, c)] = (r == c) ? 1.0 : (r > c ? v : 0.0);
    }
    for (int e = tid; e < S * S; e += C::NT) {
      const double v = Tp[e];
      __stcg(Tk + (size_t)l * S * S + e, v);
      Ts[swz<S>(e % S, e / S)] = v;
    }
    __syncthreads();
    for (int g = (c0 + S) / 8 + gi; g < B / 8; g += C::GPS) {
      double acc[C::RW / 8][2];
      load_cols<B, C::RW>(acc, Akk, 8 * g, t0, c0 / 8);
      group_apply<B, S, true, false>(sm, acc, Ys, Ts, nullptr, 0, 8 * g, t0, c0 / 8, gi, rpart);
      store_cols<B, C::RW>(acc, Akk, 8 * g, t0, c0 / 8);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// TSQRT(k,i): per inner block l, panel of B[:, c0:c0+S] against the
// s x s diagonal block of R, T_l, then the SSRFB-type update of R[c0:c0+S, c0+S:B] and
// B[:, c0+S:B].  Only the upper triangle of A(k,k) is read or written.
// ---------------------------------------------------------------------------------------
template <int B, int S>
__device__ __noinline__ void task_tsqrt(double* sm, double* Akk, double* Aik, double* Tik) {
  using C = Cfg<B, S>;
  using L = Layout<B, S>;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int gi = warp / C::RS, rpart = warp % C::RS, t0 = rpart * (C::RW / 8);
  double* P = sm + L::Y1;
  double* Ys = sm + L::Y0;
  double* Tp = sm + L::T1;
  double* Ts = sm + L::T0;
  double* Rb = sm + L::RB;
  double* Z = sm + L::ZZ;
  double* tau = sm + L::TAU;
  for (int l = 0; l < B / S; ++l) {
    const int c0 = l * S;
    const double* src = Aik + (size_t)c0 * B;
    for (int e = tid; e < B * S; e += C::NT) P[e] = __ldcg(src + e);
    for (int e = tid; e < S * S; e += C::NT) {
      const int r = e % S, c = e / S;
      Rb[e] = (r <= c) ? __ldcg(Akk + (size_t)(c0 + c) * B + c0 + r) : 0.0;
    }
    __syncthreads();
    panel_factor<B, S, C::NWARP, true>(P, B, Rb, tau, Z);
    if (warp == 0) build_t<S>(Tp, tau, Z);
    __syncthreads();
    double* dst = Aik + (size_t)c0 * B;
    for (int e = tid; e < B * S; e += C::NT) {
      const double v = P[e];
      __stcg(dst + e, v);
      Ys[swz<B>(e % B, e / B)] = v;
    }
    for (int e = tid; e < S * S; e += C::NT) {
      const int r = e % S, c = e / S;
      if (r <= c) __stcg(Akk + (size_t)(c0 + c) * B + c0 + r, Rb[e]);
      const double v = Tp[e];
      __stcg(Tik + (size_t)l * S * S + e, v);
      Ts[swz<S>(r, c)] = v;
    }
    __syncthreads();
    for (int g = (c0 + S) / 8 + gi; g < B / 8; g += C::GPS) {
      double acc[C::RW / 8][2];
      load_cols<B, C::RW>(acc, Aik, 8 * g, t0, 0);
      group_apply<B, S, true, true>(sm, acc, Ys, Ts, Akk, c0, 8 * g, t0, 0, gi, rpart);
      store_cols<B, C::RW>(acc, Aik, 8 * g, t0, 0);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// Update task on one column slice (PAPER.md:395-402 DLARFB, PAPER.md:430-466 DSSRFB):
//   SS = false: C <- (I - U_l T_l^{T or 1} U_l^T) C for each l (U_l unit lower of V)
//   SS = true : [C1; C] <- (I - [E_l; V_l] T_l^{T or 1} [E_l; V_l]^T) [C1; C]
// QT = true: Q^T direction (l ascending, T_l^T); false: Q direction (l descending, T_l).
// Y_l / T_l are double-buffered in shared memory by cp.async; the slice stays in
// registers for the whole task.
// ---------------------------------------------------------------------------------------
template <int B, int S, bool SS>
__device__ __forceinline__ void issue_panel(double* Ys, double* Ts, const double* V, const double* Tsl, int l) {
  using C = Cfg<B, S>;
  const int tid = threadIdx.x;
  const int c0 = l * S;
  if (SS) {
    for (int qd = tid; qd < B * S / 2; qd += C::NT) {
      const int c = qd / (B / 2), r = 2 * (qd % (B / 2));
      cp_async16(Ys + swz<B>(r, c), V + (size_t)(c0 + c) * B + r);
    }
  } else {
    const int nr = B - c0 - S;  // rows below the s x s top block
    for (int qd = tid; qd < nr * S / 2; qd += C::NT) {
      const int c = qd / (nr / 2), r = c0 + S + 2 * (qd % (nr / 2));
      cp_async16(Ys + swz<B>(r, c), V + (size_t)(c0 + c) * B + r);
    }
    // unit-lower top block: 1 on the diagonal, V_kk strictly below, 0 above (R is not read)
    for (int e = tid; e < S * S; e += C::NT) {
      const int r = e % S, c = e / S;
      Ys[swz<B>(c0 + r, c)] = (r == c) ? 1.0 : (r > c ? __ldcg(V + (size_t)(c0 + c) * B + c0 + r) : 0.0);
    }
  }
  for (int qd = tid; qd < S * S / 2; qd += C::NT) {
    const int c = qd / (S / 2), r = 2 * (qd % (S / 2));
    cp_async16(Ts + swz<S>(r, c), Tsl + (size_t)l * S * S + (size_t)c * S + r);
  }
  cp_async_commit();
}

template <int B, int S, bool SS, bool QT>
__device__ __noinline__ void task_update(double* sm, const double* V, const double* Tsl, double* C1, double* Ct,
                                         int slice) {
  using C = Cfg<B, S>;
  using L = Layout<B, S>;
  constexpr int NL = B / S;
  const int warp = threadIdx.x >> 5;
  const int gi = warp / C::RS, rpart = warp % C::RS, t0 = rpart * (C::RW / 8);
  const int cg0 = slice * C::SLICE + gi * 8;
  const bool active = cg0 < B;
  double acc[C::RW / 8][2];
  if (active) load_cols<B, C::RW>(acc, Ct, cg0, t0, 0);
  issue_panel<B, S, SS>(sm + L::Y0, sm + L::T0, V, Tsl, QT ? 0 : NL - 1);
  for (int li = 0; li < NL; ++li) {
    const int l = QT ? li : NL - 1 - li;
    const int buf = li & 1;
    if (li + 1 < NL) {
      const int ln = QT ? li + 1 : NL - 2 - li;
      issue_panel<B, S, SS>(sm + (buf ? L::Y0 : L::Y1), sm + (buf ? L::T0 : L::T1), V, Tsl, ln);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (active) {
      const double* Yb = sm + (buf ? L::Y1 : L::Y0);
      const double* Tb = sm + (buf ? L::T1 : L::T0);
      group_apply<B, S, QT, SS>(sm, acc, Yb, Tb, C1, l * S, cg0, t0, SS ? 0 : (l * S) / 8, gi, rpart);
    }
    __syncthreads();
  }
  if (active) store_cols<B, C::RW>(acc, Ct, cg0, t0, 0);
}

// ---------------------------------------------------------------------------------------
// Persistent executor.
// ---------------------------------------------------------------------------------------
template <int B, int S>
__global__ void __launch_bounds__(Cfg<B, S>::NT, 1) exec_kernel(ExecArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_task[TASK_INTS];
  __shared__ int s_ticket;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (;;) {
    if (tid == 0) s_ticket = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int tk = s_ticket;
    if (tk >= a.ntasks) return;
    if (tid < TASK_INTS) s_task[tid] = a.tasks[(size_t)tk * TASK_INTS + tid];
    __syncthreads();
    unsigned long long t_grab = 0, t_start = 0;
    if (a.trace && tid == 0) t_grab = globaltimer();
    if (warp == 0) {
#pragma unroll
      for (int d = 0; d < TASK_NDEP; ++d) {
        const int code = s_task[8 + 2 * d], val = s_task[9 + 2 * d];
        const int cnt = (int)((unsigned)code >> 24), idx = code & 0xFFFFFF;
        for (int x = lane; x < cnt; x += 32) {
          if (ld_acquire(a.ctr + idx + x) >= val) continue;
          const unsigned long long t0w = globaltimer();
          while (ld_acquire(a.ctr + idx + x) < val) {
            __nanosleep(200);
            // watchdog: a dependency that never resolves is a schedule bug; fail loudly
            if (globaltimer() - t0w > 20ull * 1000000000ull) __trap();
          }
        }
      }
      __syncwarp();
    }
    __syncthreads();
    if (a.trace && tid == 0) t_start = globaltimer();
    const int kind = s_task[0], k = s_task[1], i = s_task[2], j = s_task[3], sl = s_task[4];
    const int p = a.p;
    switch (kind) {
      case K_G:
        task_geqrt<B, S>(sm, tile_ptr(a.A, k, k, p, B), tslot_ptr(a.T, k, k, p, B, S));
        break;
      case K_T:
        task_tsqrt<B, S>(sm, tile_ptr(a.A, k, k, p, B), tile_ptr(a.A, i, k, p, B), tslot_ptr(a.T, i, k, p, B, S));
        break;
      case K_L:
        task_update<B, S, false, true>(sm, tile_ptr(a.A, k, k, p, B), tslot_ptr(a.T, k, k, p, B, S), nullptr,
                                       tile_ptr(a.A, k, j, p, B), sl);
        break;
      case K_S:
        task_update<B, S, true, true>(sm, tile_ptr(a.A, i, k, p, B), tslot_ptr(a.T, i, k, p, B, S),
                                      tile_ptr(a.A, k, j, p, B), tile_ptr(a.A, i, j, p, B), sl);
        break;
      case K_LQT:
        task_update<B, S, false, true>(sm, tile_ptr(a.A, k, k, p, B), tslot_ptr(a.T, k, k, p, B, S), nullptr,
                                       tile_ptr(a.Bt, k, j, p, B), sl);
        break;
      case K_SQT:
        task_update<B, S, true, true>(sm, tile_ptr(a.A, i, k, p, B), tslot_ptr(a.T, i, k, p, B, S),
                                      tile_ptr(a.Bt, k, j, p, B), tile_ptr(a.Bt, i, j, p, B), sl);
        break;
      case K_LQ:
        task_update<B, S, false, false>(sm, tile_ptr(a.A, k, k, p, B), tslot_ptr(a.T, k, k, p, B, S), nullptr,
                                        tile_ptr(a.Bt, k, j, p, B), sl);
        break;
      case K_SQ:
        task_update<B, S, true, false>(sm, tile_ptr(a.A, i, k, p, B), tslot_ptr(a.T, i, k, p, B, S),
                                       tile_ptr(a.Bt, k, j, p, B), tile_ptr(a.Bt, i, j, p, B), sl);
        break;
      default:
        break;
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(a.ctr + s_task[5], s_task[6]);
      if (a.trace) {
        unsigned long long* tr = a.trace + (size_t)tk * 4;
        tr[0] = ((unsigned long long)smid() << 32) | (unsigned)tk;
        tr[1] = t_grab;
        tr[2] = t_start;
        tr[3] = globaltimer();
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// Instances and dispatch.  (b, s) pairs built: the BASELINE.json configs (64,16),
// (128,32), (256,32) plus small/test shapes and s == b (the paper's unblocked kernels).
// ---------------------------------------------------------------------------------------
#define TQR_INSTANCES(X) \
  X(16, 8) X(16, 16) X(32, 8) X(32, 32) X(64, 16) X(64, 64) X(128, 32) X(256, 32)

template <int B, int S>
static cudaError_t launch_one(const ExecArgs& a, int grid, cudaStream_t st) {
  using L = Layout<B, S>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(exec_kernel<B, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  ExecArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((const void*)exec_kernel<B, S>, dim3(grid), dim3(Cfg<B, S>::NT), params, L::BYTES,
                                     st);
}

template <int B, int S>
static int max_ctas_one(int device) {
  using L = Layout<B, S>;
  cudaFuncSetAttribute(exec_kernel<B, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
  int per_sm = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, exec_kernel<B, S>, Cfg<B, S>::NT, L::BYTES) != cudaSuccess)
    return 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return per_sm * sms;
}

bool exec_supported(int b, int s) {
#define X(BB, SS) if (b == BB && s == SS) return true;
  TQR_INSTANCES(X)
#undef X
  return false;
}

cudaError_t launch_exec(int b, int s, const ExecArgs& a, int grid, cudaStream_t st) {
#define X(BB, SS) if (b == BB && s == SS) return launch_one<BB, SS>(a, grid, st);
  TQR_INSTANCES(X)
#undef X
  return cudaErrorInvalidValue;
}

int exec_slice(int b, int s) {
#define X(BB, SS) if (b == BB && s == SS) return Cfg<BB, SS>::SLICE;
  TQR_INSTANCES(X)
#undef X
  return 0;
}

int exec_max_ctas(int b, int s, int device) {
#define X(BB, SS) if (b == BB && s == SS) return max_ctas_one<BB, SS>(device);
  TQR_INSTANCES(X)
#undef X
  return 0;
}

// ---------------------------------------------------------------------------------------
// Layout kernels (Block Data Layout).  HBM-bound copies: one thread per
// element, tile-row index fastest so both the column-major and the tile-major side are
// contiguous runs of b doubles.
// ---------------------------------------------------------------------------------------
__global__ void pack_kernel(const double* __restrict__ A, int64_t lda, double* __restrict__ At, int64_t m, int64_t n,
                            int b, int64_t p, int64_t total) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bb = (int64_t)b * b;
    const int64_t tile = e / bb, in = e % bb;
    const int64_t i = tile % p, jt = tile / p;
    const int64_t r = i * b + in % b, c = jt * b + in / b;
    At[e] = (r < m && c < n) ? A[r + c * lda] : 0.0;
  }
}
__global__ void unpack_kernel(const double* __restrict__ At, double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                              int b, int64_t p) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % m, c = e / m;
    const int64_t i = r / b, jt = c / b;
    A[r + c * lda] = At[((i + jt * p) * b + (c % b)) * b + (r % b)];
  }
}
__global__ void get_r_kernel(const double* __restrict__ At, double* __restrict__ R, int64_t ldr, int64_t m, int64_t n,
                             int b, int64_t p) {
  const int64_t k = m < n ? m : n;
  const int64_t total = k * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % k, c = e / k;
    const int64_t i = r / b, jt = c / b;
    R[r + c * ldr] = (r <= c) ? At[((i + jt * p) * b + (c % b)) * b + (r % b)] : 0.0;
  }
}
__global__ void eye_tiles_kernel(double* __restrict__ Qt, int64_t m, int64_t k, int b, int64_t p, int64_t total) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bb = (int64_t)b * b;
    const int64_t tile = e / bb, in = e % bb;
    const int64_t i = tile % p, jt = tile / p;
    const int64_t r = i * b + in % b, c = jt * b + in / b;
    Qt[e] = (r == c && c < k && r < m) ? 1.0 : 0.0;
  }
}

static int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (int)g;
}

cudaError_t launch_pack(const double* A, int64_t lda, double* At, int64_t m, int64_t n, int b, int64_t p, int64_t q,
                        cudaStream_t st) {
  const int64_t total = p * q * (int64_t)b * b;
  pack_kernel<<<grid_for(total), 256, 0, st>>>(A, lda, At, m, n, b, p, total);
  return cudaGetLastError();
}
cudaError_t launch_unpack(const double* At, double* A, int64_t lda, int64_t m, int64_t n, int b, int64_t p,
                          cudaStream_t st) {
  unpack_kernel<<<grid_for(m * n), 256, 0, st>>>(At, A, lda, m, n, b, p);
  return cudaGetLastError();
}
cudaError_t launch_get_r(const double* At, double* R, int64_t ldr, int64_t m, int64_t n, int b, int64_t p,
                         cudaStream_t st) {
  const int64_t k = m < n ? m : n;
  get_r_kernel<<<grid_for(k * n), 256, 0, st>>>(At, R, ldr, m, n, b, p);
  return cudaGetLastError();
}
cudaError_t launch_eye_tiles(double* Qt, int64_t m, int64_t k, int b, int64_t p, int64_t qb, cudaStream_t st) {
  const int64_t total = p * qb * (int64_t)b * b;
  eye_tiles_kernel<<<grid_for(total), 256, 0, st>>>(Qt, m, k, b, p, total);
  return cudaGetLastError();
}

}  // namespace tqr
