// tlu_internal.h -- declarations shared by the tiled-LU host runtime (tlu_host.cpp) and its
// CUDA translation unit (tlu_exec.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tqr {
namespace lu {

// Task kinds (LU1-LU7; the analogues of GEQRT, TSQRT, LARFB, SSRFB)
enum Kind : int { LK_G = 0, LK_T = 1, LK_L = 2, LK_S = 3 };

// Task records: the tiled-QR record format (tqr_internal.h TASK_INTS) -- [0] kind, [1] k,
// [2] i, [3] j, [4] slice (update tasks; -1 for panels), [5] out counter, [6] out value,
// [8 + 2d], [9 + 2d] dependency d = (index | count << 24, value), [14] 0, [15] 1.
struct LuArgs {
  const int* tasks;
  int ntasks;
  int* ticket;  // reset to 0 before the launch
  int* ctr;     // progress counters (reset to 0 before the launch)
  double* A;    // tiles, Block Data Layout (p x q tiles of b x b, column-major inside)
  double* W;    // p x K slots of s x b: block l's W_l = (I + Ltilde_l)^{-1} / L11_l^{-1}, column-major
  int* piv;     // p x K slots of b ints (oracle_lu.h semantics)
  int* perm;    // workspace: p x K slots of (b / s) x (2 + 4 s) ints -- each block's net interchange
                //   as (count, -, dst0, src0, dst1, src1, ...; 4 + 4s ints per block) over rows [0, b) of the updated tile
                //   and [b, b + s) of the s pivot-block rows (the GESSM / SSSSM "X" rows)
  double* Lw;   // workspace: p x K tiles of b x (b + 4) -- each block's Ltilde_l = L_l W_l (LU12),
                //   written by the panels, read by the update tasks instead of L_l (b = 256 only)
  int p, q;
  int nctr;
  int disp;  // 1: the next task is dispatched by warp 2 during the previous task's release (throughput-bound grids)
  unsigned long long* trace;  // 4 per task or nullptr
};

bool lu_supported(int b, int s);
int lu_slice(int b, int s);          // columns per update task slice
int lu_perm_ints(int b, int s);      // perm ints per slot
bool lu_uses_ltilde(int b, int s);   // the instance's update reads Ltilde tiles from the workspace (LU12)
int lu_ltilde_doubles(int b, int s); // doubles per workspace Ltilde tile (b (b + 4): the shared layout)
int lu_max_ctas(int b, int s, int device);
cudaError_t launch_lu_exec(int b, int s, const LuArgs& a, int grid, cudaStream_t st);

}  // namespace lu
}  // namespace tqr
