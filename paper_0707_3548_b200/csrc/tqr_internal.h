// tqr_internal.h -- declarations shared by the host runtime (tqr_host.cpp) and the
// CUDA translation unit (tqr_exec.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tqr {

// Task kinds (priority classes of PAPER.md:612-615 are G < T < L < S).
enum Kind : int {
  K_G = 0,      // GEQRT(k)              on A(k,k), T(k,k)
  K_T = 1,      // TSQRT(k,i)            on A(k,k) upper, A(i,k), T(i,k)
  K_L = 2,      // LARFB(k,j), slice sl  on A(k,j)
  K_S = 3,      // SSRFB(k,i,j), slice   on A(k,j), A(i,j)
  K_LQT = 4,    // apply-Q^T: LARFB-type on Bt(k,j)
  K_SQT = 5,    // apply-Q^T: SSRFB-type on Bt(k,j), Bt(i,j)
  K_LQ = 6,     // apply-Q:   LARFB-type, T_l untransposed, l descending
  K_SQ = 7,     // apply-Q:   SSRFB-type
};

// One task record = 16 int32:
//   [0] kind [1] k [2] i [3] j [4] slice [5] out counter index [6] out value [7] unused
//   [8 + 2d], [9 + 2d], d = 0..2: dependency d = (index | count << 24, value):
//   wait until ctr[index + x] >= value for x in [0, count); count == 0 means no dependency.
constexpr int TASK_INTS = 16;
constexpr int TASK_NDEP = 3;

struct ExecArgs {
  double* A;          // tile-major factors (p x q tiles)
  double* T;          // T slots (p x q slots of s*b)
  double* Bt;         // apply-Q target, tile-major with p row tiles
  double* Yp;         // workspace: packed reflector panels (p x q tiles of b*b)
  double* Tp;         // workspace: packed T blocks (p x q slots of s*b)
  const int* tasks;   // TASK_INTS per task, dispatch order
  int ntasks;
  int p;              // row tiles (same for A and Bt)
  int* ticket;        // next ticket (reset to 0 before the launch)
  int* ctr;           // monotone progress counters (reset to 0)
  unsigned long long* trace;  // 4 per task or nullptr
  long long* phases;          // TQR_PROFILE_PHASES builds: 8 phase-cycle totals, or nullptr
};

// Launch the persistent executor for tile size b, inner block s.  Returns cudaSuccess or
// the launch error; *grid_out receives the co-resident grid used.
// mode: 0 factorization, 1 apply Q^T, 2 apply Q.
cudaError_t launch_exec(int b, int s, int mode, const ExecArgs& a, int grid, cudaStream_t st);
// Max co-resident CTAs for (b, s) on this device (0 if no instance).
int exec_max_ctas(int b, int s, int device);
bool exec_supported(int b, int s);
// Columns per LARFB/SSRFB slice task for (b, s) (0 if no instance).
int exec_slice(int b, int s);

cudaError_t launch_pack(const double* A, int64_t lda, double* At, int64_t m, int64_t n, int b, int64_t p, int64_t q,
                        cudaStream_t st);
cudaError_t launch_unpack(const double* At, double* A, int64_t lda, int64_t m, int64_t n, int b, int64_t p,
                          cudaStream_t st);
cudaError_t launch_get_r(const double* At, double* R, int64_t ldr, int64_t m, int64_t n, int b, int64_t p,
                         cudaStream_t st);
cudaError_t launch_pack_factors(const double* A, const double* T, double* Yp, double* Tp, int b, int s, int64_t p,
                                int64_t K, cudaStream_t st);
cudaError_t launch_eye_tiles(double* Qt, int64_t m, int64_t k, int b, int64_t p, int64_t qb, cudaStream_t st);

}  // namespace tqr
