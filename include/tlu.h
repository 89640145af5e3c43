/*
 * tlu.h -- C ABI of the B200 tiled LU factorization (the paper's first named extension,
 * "The LU factorization can be performed with an algorithm that is analogous
 * to the QR one described in Section [tiled] ... the only difference between the block
 * algorithms for the LU and QR factorizations is in the elementary operations"; SURVEY 8(f)
 * NEXT-4).  The elementary operations are DESIGN.md readings LU1-LU9 (pairwise / incremental
 * pivoting of the out-of-core LU the paper cites):
 *   GETRF(k)      LU with partial pivoting of the diagonal tile A_kk (inner blocking s)
 *   GESSM(k,j)    A_kj <- GETRF(k)'s interchanges and eliminations applied to A_kj
 *   TSTRF(k,i)    LU with partial pivoting of the stacked [U_kk; A_ik] (candidates: U_kk's
 *                 diagonal row and every row of A_ik)
 *   SSSSM(k,i,j)  [A_kj; A_ij] <- TSTRF(k,i)'s interchanges and eliminations
 * run in the DAG order of the tiled QR (the same edges with the kernels renamed) by one
 * persistent launch per call, like tqr_geqrf.
 *
 * Conventions (as include/tqr.h): fp64; every data pointer is device memory owned by the
 * caller, 16-byte aligned; calls are asynchronous on the plan's stream; errors are return
 * codes (tqr_status), never aborts; tqr_last_error() / tqr_last_bad_arg() describe the last one.
 *
 * Storage (oracle/oracle_lu.h semantics, Block Data Layout of PAPER.md:656-663):
 *   At   p*q tiles of b*b doubles (tqr_pack layout); after tlu_getrf: U = the upper trapezoid,
 *        GETRF's multipliers in the strict lower part of A_kk, TSTRF's in all of A_ik;
 *   W    p*K slots of s*b doubles, slot (i,k) at (i + k p) s b: block l's s x s unit-lower
 *        W_l in columns [l s, l s + s), column-major -- the INVERSE of the block's unit-lower
 *        factor (slot (k,k): of L11_l, the unit-lower diagonal block of GETRF's block l; slot
 *        (i,k), i > k: of I + Ltilde_l, TSTRF's block l; LU8);
 *   piv  p*K slots of b int32, slot (i,k) at (i + k p) b: GETRF: the tile row interchanged with
 *        row c; TSTRF: -1 if U_kk's row c stayed, else the row of A_ik interchanged with it.
 * Supported (b, s): (256, 32), (128, 32), (64, 16) (tlu_supported).
 */
#ifndef TLU_H
#define TLU_H
#include "tqr.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tlu_plan tlu_plan;

typedef struct {
  int64_t m, n;    /* matrix size, >= 1 (bad-arg indices: m=1, n=2) */
  int32_t b, s;    /* tile size and inner blocking, s | b (b=3, s=4) */
  int32_t device;  /* CUDA device ordinal (5) */
  void* stream;    /* cudaStream_t, NULL = legacy default stream */
  uint32_t flags;  /* TQR_FLAG_TRACE */
} tlu_params;

/* Validates, builds the DAG task table (list-schedule order by bottom level), allocates the
 * device task table and counters.  TQR_ERR_UNSUPPORTED if (b, s) has no kernel instance. */
tqr_status tlu_plan_create(tlu_plan** out, const tlu_params* p);
tqr_status tlu_plan_destroy(tlu_plan* plan);
/* Element counts of At (doubles), W (doubles), piv (int32). */
tqr_status tlu_sizes(const tlu_plan* plan, size_t* a_doubles, size_t* w_doubles, size_t* piv_ints);
/* Bytes of the caller-allocated workspace of tlu_getrf: each block's net interchange lists, then
 * (b = 256) p x min(p, q) tiles of b x (b + 4) doubles holding each block's L_l W_l (the multipliers
 * times W_l, LU12; scratch, not an output).  Device memory, 16-byte aligned. */
tqr_status tlu_workspace_size(const tlu_plan* plan, size_t* bytes);
/* Column-major A (m x n, lda >= m) -> tiles (zero padding); tiles -> column-major. */
tqr_status tlu_pack(tlu_plan* plan, const double* A, int64_t lda, double* At);
tqr_status tlu_unpack(tlu_plan* plan, const double* At, double* A, int64_t lda);
/* The tiled LU factorization: At in (the packed A), out (U + multipliers); W, piv out. */
tqr_status tlu_getrf(tlu_plan* plan, double* At, double* W, int32_t* piv, void* work);
/* U = the upper trapezoid, min(m,n) x n column-major (ldu >= min(m,n)), zeros below. */
tqr_status tlu_get_u(tlu_plan* plan, const double* At, double* U, int64_t ldu);
tqr_status tlu_sync(tlu_plan* plan);
/* The dispatch records this plan executes (16 int32 each, include/tqr.h record format with
 * kinds 0 GETRF, 1 TSTRF, 2 GESSM, 3 SSSSM): rec may be NULL to query *n. */
tqr_status tlu_plan_records(tlu_plan* plan, int32_t* rec, int64_t cap, int64_t* n);
/* The records a plan for (m, n, b, s) would execute with `workers` CTAs (pure host, no device;
 * the CPU tests replay them): rec may be NULL to query *ntask; *nctr = counters used. */
tqr_status tlu_schedule_records(int64_t m, int64_t n, int32_t b, int32_t s, int32_t workers, int32_t* rec, int64_t cap,
                                int64_t* ntask, int32_t* nctr);
/* Trace of the last tlu_getrf (TQR_FLAG_TRACE): 8 int64 per task in dispatch order --
 * kind, k, i, j, SM id, ticket-grab / start / end %globaltimer stamps (ns). */
tqr_status tlu_trace_fetch(tlu_plan* plan, int64_t* rec, int64_t cap, int64_t* n);
int32_t tlu_supported(int32_t b, int32_t s);
/* Flop counts: standard mn^2 - n^3/3 (m >= n; LAPACK dgetrf), and the tiled algorithm's
 * executed count (LU9). */
double tlu_flops_standard(int64_t m, int64_t n);
double tlu_flops_tiled(int64_t m, int64_t n, int32_t b, int32_t s);

#ifdef __cplusplus
}
#endif
#endif
