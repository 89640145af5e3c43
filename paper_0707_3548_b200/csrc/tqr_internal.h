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
//   [0] kind [1] k (global step; indexes the reflector workspace) [2] i
//   [3] j: STORAGE tile column of the updated tile (L/S/apply-Q kinds)
//   [4] slice [5] out counter index [6] out value
//   [7] kc: STORAGE tile column of tile column k (A(k,k), A(i,k), T(., k))
//   [8 + 2d], [9 + 2d], d = 0..2: dependency d = (index | count << 24, value):
//       wait until ctr[index + x] >= base + value for x in [0, count); count 0 = none
//   [14] flags: bit 0 = publish the out counter on every rank (panel progress, multi-GPU),
//        bit 1 / bit 2 = panel apply / factor part, bits 3..5 = dependency 0..2 is a counter a
//        peer GPU publishes (system-scope acquire on a real multi-GPU job; gpu scope otherwise),
//        bit 6 = pipelined panel dependency (update tasks: dependency 0 names PF(k, last block);
//        the task starts on PF(k, 0) and waits for block l just before staging it);
//        bits 8..31 = 1 + an early-release
//        counter that a panel factor part sets to [6] once R_kk's rows of its block are final
//   [15] update tasks: np | ocnt << 8 -- register passes [slice, slice + np) (slice = [4], in
//        units of SLICE columns), and ocnt consecutive out counters [5] .. [5] + ocnt - 1 set
//        to [6] on completion (0 / panel tasks: one)
// Counter values of one factorization are base + v with v in [1, p + 1]; the base grows by
// (p + 2) per call, so counters are never reset (no cross-rank reset race).
constexpr int TASK_INTS = 16;
constexpr int TASK_NDEP = 3;
constexpr int MAX_RANKS = 8;

// One rank's task stream and its tile storage.  In the single-launch multi-rank
// emulation every rank of the job is a RankLocal of the same launch; on a real multi-GPU
// job each process runs exactly one.
struct RankLocal {
  const int* tasks;   // TASK_INTS per task, dispatch order
  int ntasks;
  int rank;           // job rank id (index into ExecArgs::Yp/Tp/ctr)
  int* ticket;        // next ticket (reset to 0 before the launch)
  int* ctr;           // this rank's progress counters
  double* A;          // tile-major factors (p row tiles, storage columns)
  double* T;          // T slots (p x storage columns, s*b each)
  double* Bt;         // apply-Q target, tile-major with p row tiles (single rank only)
  unsigned long long* trace;  // 4 per task or nullptr
};

struct ExecArgs {
  RankLocal loc[MAX_RANKS];
  int nloc;                 // ranks run by this launch (CTA c serves loc[c % nloc])
  int nranks;               // ranks of the job
  double* Yp[MAX_RANKS];    // every rank's workspace: packed reflector panels (p x K tiles of b*b)
  double* Tp[MAX_RANKS];    //   and packed T blocks (p x K slots of s*b)
  int* ctr[MAX_RANKS];      // every rank's counters (panel progress is published to all)
  int p;                    // row tiles (same for A and Bt)
  int base;                 // counter generation base of this call
  int sys;                  // 1: peers on other GPUs (system-scope acquire/release)
  int nctr;                 // counters per rank (TQR_CHECKS builds: bounds of every counter access)
  int qcols;                // storage tile columns of A (and of Bt in apply-Q) (TQR_CHECKS)
  int nsl;                  // update tasks per tile (TQR_CHECKS)
  long long* phases;        // TQR_PROFILE_PHASES builds: 16 phase-cycle totals, or nullptr
};

// Launch the persistent executor for tile size b, inner block s (cooperative launch).
// mode: 0 factorization, 1 apply Q^T, 2 apply Q.
// rwm: rows-per-warp variant (128 or 256; b >= 256 only, otherwise ignored).
cudaError_t launch_exec(int b, int s, int mode, int rwm, const ExecArgs& a, int grid, cudaStream_t st);
// Max co-resident CTAs for (b, s, rwm) on this device (0 if no instance).
int exec_max_ctas(int b, int s, int rwm, int device);
bool exec_supported(int b, int s);
// Columns of one register-resident pass of a LARFB/SSRFB task for (b, s) (0 if no instance);
// a task covers np consecutive passes (host policy, task record [15]).
int exec_slice(int b, int s, int rwm);
// Internal inner block SI of the executor for (b, s) (== s except b = 512).
int exec_inner(int b, int s);
// Off-diagonal blocks of the output T_L when SI < s (no-op otherwise).
cudaError_t launch_form_t(const double* A, double* T, int b, int s, int64_t p, int64_t qloc, int cstride, int coff,
                          cudaStream_t st);

// Tall-unit executor (R30: the tile rows below the diagonal in units of two b x b
// tiles; b = 256, s = 32 only, one rank, factorization only).  Records as for the square
// executor with [2] = the unit's first tile row, [14] bit 7 = a second tile and, for the split
// apply parts, [4] = l | (lp + 1) << 8 (apply output block lp to block l's columns); the workspace
// holds 2 b^2 doubles of packed panels per (tile row, step).
cudaError_t launch_exec_tall(const ExecArgs& a, int grid, cudaStream_t st);
int exec_max_ctas_tall(int device);
int exec_slice_tall();  // columns per register pass of its update tasks
// off-diagonal blocks of the output T_L of the units listed in d_units (3 ints each: i0, k, nt)
cudaError_t launch_form_t_tall(const double* A, double* T, const int* d_units, int nunits, int p, cudaStream_t st);

// Layout kernels.  Tile-major arrays hold the tile columns j = coff + jl*cstride of the
// global p x q grid at storage column jl (single GPU / emulation: cstride 1, coff 0).
cudaError_t launch_pack(const double* A, int64_t lda, double* At, int64_t m, int64_t n, int b, int64_t p,
                        int64_t qloc, int cstride, int coff, cudaStream_t st);
cudaError_t launch_unpack(const double* At, double* A, int64_t lda, int64_t m, int64_t n, int b, int64_t p,
                          int64_t qloc, int cstride, int coff, cudaStream_t st);
cudaError_t launch_get_r(const double* At, double* R, int64_t ldr, int64_t m, int64_t n, int b, int64_t p,
                         int64_t qloc, int cstride, int coff, cudaStream_t st);
// Packed reflector panels of the factors (A, T) -- storage columns kc of global tile column
// coff + kc*cstride, qloc of them -- into nd workspaces (Yp[d], Tp[d], indexed by the global
// step k); sys_fence: the stores go to peer GPUs (system-scope fence at the end).
cudaError_t launch_pack_factors(const double* A, const double* T, double* const* Yp, double* const* Tp, int nd, int b,
                                int s, int64_t p, int64_t K, int64_t qloc, int cstride, int coff, bool sys_fence,
                                cudaStream_t st);
// Tile-major [I_k; 0] (m x k) in the storage columns jl of global tile column coff + jl*cstride.
cudaError_t launch_eye_tiles(double* Qt, int64_t m, int64_t k, int b, int64_t p, int64_t qloc, int cstride, int coff,
                             cudaStream_t st);
// Cross-rank entry barrier of one call (real multi-GPU): publish `gen` into every rank's
// arrive[me] (system scope), wait until arrive[g] >= gen for all g on this rank.
cudaError_t launch_rank_barrier(int* const* arrive_all, int nranks, int me, int gen, cudaStream_t st);
// Store magic + me into slot me of every rank's ping array (tqr_comm_ping).
cudaError_t launch_ping(int* const* ping_all, int nranks, int me, int magic, cudaStream_t st);

// Sets the thread's tqr_last_error() message and tqr_last_bad_arg() index (tqr_host.cpp).
void set_last_error(const char* what, int bad_arg_idx);

}  // namespace tqr
