/*
 * tqr.h -- C ABI of the B200-native (sm_100a) fp64 tiled QR library.
 *
 * Method: the tiled QR factorization of arXiv 0707.3548 (PAPER.md, "Tiled
 * algorithms" / "A Fine-Grain Algorithm for QR Factorization"),
 * executed out of order under its DAG by a persistent
 * device-side executor.  Storage is the paper's Block Data Layout
 * (PAPER.md:642-666): b x b tiles, column-major inside a tile, tiles
 * column-major in the p x q grid; tile (i,j) starts at (i + j*p)*b*b.
 *
 * Conventions shared by every call
 *   - All data pointers are DEVICE pointers owned by the caller (e.g. torch
 *     tensors); the library never frees or reallocates caller memory.  They must
 *     be 16-byte aligned.  The library allocates only inside tqr_plan_create and
 *     frees that in tqr_plan_destroy.
 *   - Every call is asynchronous on the plan's CUDA stream (tqr_params.stream);
 *     it returns after enqueueing.  Device faults surface at tqr_sync or at the
 *     next call.
 *   - Errors are return codes; nothing throws or aborts across the ABI.  After
 *     TQR_ERR_INVALID_ARG, tqr_last_bad_arg() gives the LAPACK-style 1-based
 *     index of the offending argument of the failing call.
 *   - T factors: slot (i,k) (i >= k) holds s x b doubles at (i + k*p)*s*b of the
 *     T array; inside a slot, T_l (s x s upper triangular, zeros below) occupies
 *     columns [l*s, l*s+s).  Slot (k,k) comes from GEQRT(k), slot (i,k), i>k,
 *     from TSQRT(k,i).  (Inner blocking s is DESIGN.md reading R5; s == b is the
 *     paper's kernel.)
 *   - Q^T = H_N ... H_1 is applied as I - V T^T V^T per inner block (DESIGN.md
 *     reading R1: the paper prints (I - V T V^T), which is
 *     the forward product H_1 ... H_b; the factorization applies its transpose).
 */
#ifndef TQR_H
#define TQR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TQR_OK = 0,
  TQR_ERR_INVALID_ARG = 1, /* see tqr_last_bad_arg() */
  TQR_ERR_CUDA = 2,        /* a CUDA runtime call failed (message: tqr_last_error()) */
  TQR_ERR_NCCL = 3,        /* multi-GPU transport failure */
  TQR_ERR_OOM = 4,         /* device allocation inside tqr_plan_create failed */
  TQR_ERR_UNSUPPORTED = 5  /* valid but not built (e.g. (b,s) without a kernel instance) */
} tqr_status;

typedef struct tqr_plan tqr_plan;

typedef struct {
  int64_t m;       /* rows of A, >= 1 */
  int64_t n;       /* columns of A, >= 1 */
  int32_t b;       /* tile size, >= 1 (built instances: see tqr_supported) */
  int32_t s;       /* inner block size: 1 <= s <= b, s divides b */
  int32_t device;  /* CUDA device ordinal */
  void* stream;    /* cudaStream_t to enqueue on; NULL = legacy default stream */
  int32_t nranks;  /* ranks of the job, 1..8: tile columns are 1D block-cyclic, rank r owns
                      columns j == r (mod nranks) (multi-GPU section below) */
  int32_t rank;    /* 0 <= rank < nranks (0 with TQR_FLAG_EMULATE_RANKS) */
  uint32_t flags;  /* TQR_FLAG_* */
} tqr_params;

#define TQR_FLAG_TRACE 1u          /* record per-task (sm, start, end) %globaltimer stamps */
#define TQR_FLAG_EMULATE_RANKS 2u  /* nranks > 1 on ONE device in ONE launch: every rank's task
                                      stream, counters and workspace, the same peer-store protocol
                                      (test mode for the multi-GPU path on a single GPU) */
#define TQR_FLAG_TALL_TILES 4u     /* the paper's non-square 2b x b tiles (PAPER.md:582-583,
                                      DESIGN.md R30): the tile rows below the diagonal in units of
                                      two tiles (units start right below the diagonal tile; the last
                                      may be one tile); TSQRT / SSRFB work on a unit's 2b x b stack,
                                      its T factors in the T slot of its first tile row (the other
                                      slots 0).  A different reflector sequence than square tiles:
                                      R differs in row signs / rounding.  Built for b = 256, s = 32,
                                      one rank, factorization (tqr_geqrf, tqr_get_r) only;
                                      TQR_ERR_UNSUPPORTED otherwise. */
#define TQR_FLAG_LOCALITY 8u       /* locality-aware dispatch ("Enforcing data
                                      locality"; R22): the update tasks that apply one
                                      reflector panel (k, i) share one priority so they run together
                                      and read the panel from L2 (about half the DRAM reads at C3),
                                      except in the last quarter of the steps, where the critical
                                      path decides.  Same results bit for bit (dispatch order only);
                                      square tiles, factorization schedule. */

/* ---- plan -------------------------------------------------------------------------- */
/* Validates p (argument 2's fields: m=1, n=2, b=3, s=4, device=5, nranks=7, rank=8 are
 * reported as bad-arg indices), builds the DAG task tables and
 * allocates device-side task tables and progress counters. */
tqr_status tqr_plan_create(tqr_plan** out, const tqr_params* p);
tqr_status tqr_plan_destroy(tqr_plan* plan);

/* Sizes of the caller-owned tile arrays, in doubles: At = p*ql*b*b, T = p*ql*s*b
 * (m rounded up to p = ceil(m/b) tiles, n to q = ceil(n/b)); ql = q, except on a real
 * multi-rank plan, where ql = number of tile columns this rank owns (its storage column jl
 * holds global tile column rank + jl*nranks). */
tqr_status tqr_tiles_size(const tqr_plan* plan, size_t* a_doubles, size_t* t_doubles);
/* Device workspace the caller must pass as `work` to geqrf/ormqr/orgqr (bytes):
 * (p*q*b*b + p*q*s*b) doubles holding packed (shared-memory-layout) copies of every
 * reflector panel and T block, written once by the panel tasks and streamed by TMA bulk
 * copies into every update task.  Not needed after the call returns.  Multi-rank plans
 * (nranks > 1) own a peer-visible workspace per rank instead: 0 bytes, `work` may be NULL. */
tqr_status tqr_workspace_size(const tqr_plan* plan, size_t* bytes);

/* ---- layout ------------------------------------------------------ */
/* Column-major m x n A (lda >= m) -> tile-major At, zero padding beyond m, n.  On a real
 * multi-rank plan A is the whole matrix and only this rank's tile columns are packed. */
tqr_status tqr_pack(tqr_plan* plan, const double* A, int64_t lda, double* At);
/* Tile-major At -> column-major m x n A (lda >= m); padding is dropped (multi-rank: only
 * this rank's columns of A are written). */
tqr_status tqr_unpack(tqr_plan* plan, const double* At, double* A, int64_t ldr);

/* ---- factorization (Algorithm 1) ---------------------------------- */
/* In: At = packed A.  Out: At holds R in its upper trapezoid and the Householder
 * vectors V below it (V_kk strictly lower in diagonal tiles, V_ik full in tiles
 * below the diagonal); T receives every T slot.
 * GEQRT, TSQRT, LARFB and SSRFB tasks run out of order on the device in a
 * topological order of the DAG, prioritised by critical-path length (the criterion behind
 * the paper's G > T > L > S priorities; R10).  The order never
 * changes the result: R, V and T are bitwise reproducible run to run. */
tqr_status tqr_geqrf(tqr_plan* plan, double* At, double* T, void* work);  /* work: see tqr_workspace_size */

/* R = upper trapezoid of the factored tiles, min(m,n) x n column-major (ldr >= min(m,n)),
 * zeros below the diagonal (multi-rank: only this rank's columns of R are written). */
tqr_status tqr_get_r(tqr_plan* plan, const double* At, double* R, int64_t ldr);

/* Apply Q^T (trans = 'T') or Q (trans = 'N') from the factors (At, T) to a tile-major
 * m x nrhs matrix Bt laid out like At (p row tiles, ceil(nrhs/b) tile columns),
 * in place.  (DORMQR analogue; reading R8.)
 * Multi-rank plans: COLLECTIVE (every rank calls it with the same trans, nrhs).  Bt is 1D
 * block-cyclic like At (a real rank holds B's tile columns jb == rank mod nranks, storage
 * column jb / nranks; emulated plans the global grid); each rank packs the reflector panels
 * of its own columns of (At, T) into every rank's workspace over peer memory between two
 * device-side rank barriers, then applies Q to its own columns of B with no further
 * exchange.  `work` may be NULL (the plan owns the workspaces). */
tqr_status tqr_ormqr(tqr_plan* plan, char trans, const double* At, const double* T,
                     double* Bt, int64_t nrhs, void* work);

/* Form the first k columns of Q explicitly (Q [I_k; 0]) into tile-major Qt
 * (p row tiles, ceil(k/b) tile columns); 1 <= k <= m.  (DORGQR analogue.)
 * Multi-rank plans: collective, Qt block-cyclic as Bt of tqr_ormqr. */
tqr_status tqr_orgqr(tqr_plan* plan, const double* At, const double* T, int64_t k,
                     double* Qt, void* work);

/* ---- multi-GPU ---------------------------------------
 * One process per GPU, tile columns 1D block-cyclic.  The panel tasks of step k (GEQRT(k),
 * TSQRT(k,i)) run on owner(k) = k mod nranks and store their packed V/T tiles directly into
 * every rank's workspace over NVLink peer memory, then release-store that rank's panel-k
 * progress counter at system scope: the per-tile V/T broadcast is fused into the panel task
 * (no separate collective).  LARFB/SSRFB run on the owner of the updated column.  R, V and T
 * are bitwise identical to the single-GPU factorization.
 *
 * Connection, once per plan, after every rank created its plan with the same (m, n, b, s,
 * nranks): tqr_comm_export writes this rank's TQR_IPC_BLOB_BYTES-byte CUDA IPC blob;
 * the caller all-gathers the blobs (any transport, e.g. torch.distributed) in rank order
 * and passes the concatenation to tqr_comm_connect.  Errors: TQR_ERR_UNSUPPORTED on
 * single-rank or emulated plans; TQR_ERR_INVALID_ARG(2) if a blob does not match the plan;
 * TQR_ERR_CUDA if the IPC mapping fails.  Every tqr_geqrf of a connected plan starts with a
 * device-side entry barrier across ranks (a rank that never arrives traps after 60 s). */
#define TQR_IPC_BLOB_BYTES 256
tqr_status tqr_comm_export(tqr_plan* plan, void* blob /* TQR_IPC_BLOB_BYTES, host */);
tqr_status tqr_comm_connect(tqr_plan* plan, const void* blobs /* nranks * TQR_IPC_BLOB_BYTES, host */);
/* Connectivity check of a connected plan, no waiting on peers: tqr_comm_ping stores
 * magic + rank into slot `rank` of every rank's ping array through the peer mappings
 * (system-scope release stores; synchronous); after a host-side barrier, tqr_comm_flags
 * copies this rank's nranks ping slots to host memory `out` (slot g == magic + g when rank g's
 * stores arrived).  TQR_ERR_UNSUPPORTED on plans that are not real multi-rank. */
tqr_status tqr_comm_ping(tqr_plan* plan, int32_t magic);
tqr_status tqr_comm_flags(tqr_plan* plan, int32_t* out /* nranks, host */);

/* ---- flop models -------------------------------------------------------------------- */
/* Standard count 2n^2(m - n/3) for m >= n, 2m^2(n - m/3) otherwise. */
double tqr_flops_standard(int64_t m, int64_t n);
/* Executed count of the tiled algorithm with inner blocking s:
 * per task GEQRT 4/3 b^3 + 2/3 s b^2, LARFB 2b^3 + s b^2, TSQRT 2b^3 + 4/3 s b^2,
 * SSRFB 4b^3 + s b^2 -- at s == b the paper's 2, 3, 10/3, 5 b^3. */
double tqr_flops_tiled(int64_t m, int64_t n, int32_t b, int32_t s);

/* ---- misc --------------------------------------------------------------------------- */
tqr_status tqr_sync(tqr_plan* plan);              /* cudaStreamSynchronize + error check */
const char* tqr_status_string(tqr_status st);
const char* tqr_last_error(void);                 /* thread-local detail of the last failure */
int32_t tqr_last_bad_arg(void);                   /* thread-local; 0 if none */
int32_t tqr_supported(int32_t b, int32_t s);      /* 1 if a kernel instance exists for (b, s) */

/* Introspection of the host-built schedule (pure host, usable without a GPU):
 * number of tasks of each kind {G, T, L, S} in the plan-independent DAG for a
 * p x q tile grid with `nslice` column slices per tile, and a topological check of
 * the dispatch order the library would use with `workers` concurrent CTAs.
 * Returns TQR_OK when the order is a valid topological order of the DAG. */
tqr_status tqr_schedule_inspect(int64_t p, int64_t q, int32_t nslice, int32_t workers,
                                int64_t counts[4], int64_t* n_edges);

/* The per-rank dispatch records (16 int32 per task, layout of csrc/tqr_internal.h) of the
 * factorization schedule for a p x q grid with `nslice` slices, `workers` CTAs per rank and
 * `nranks` ranks (real multi-rank storage columns for nranks > 1); *n = task count of
 * `rank`, *nctr = its counter count; up to `cap` records copied to rec (host).  Pure host:
 * lets CPU tests replay the distributed protocol. */
tqr_status tqr_schedule_records(int64_t p, int64_t q, int32_t nslice, int32_t workers, int32_t nranks, int32_t rank,
                                int32_t* rec, int64_t cap, int64_t* n, int32_t* nctr);
/* The same with the tile rows below the diagonal in units of h (1..4; TQR_FLAG_TALL_TILES
 * uses h = 2): record [2] = a unit's first tile row, [14] bit 7 = a multi-tile unit. */
tqr_status tqr_schedule_records_h(int64_t p, int64_t q, int32_t nslice, int32_t workers, int32_t nranks,
                                  int32_t rank, int32_t h, int32_t* rec, int64_t cap, int64_t* n, int32_t* nctr);
/* The factorization records a plan for (m, n, b, s, nranks, flags) would execute on `rank`
 * with `workers` CTAs per rank (the plan policy -- tile columns 1D block-cyclic for nranks > 1,
 * TQR_FLAG_TALL_TILES selects the tall-unit executor's schedule; pure host, no device): for
 * footprint / race checks of the production schedules (tests/test_race_model.py).  *ntask =
 * task count, up to `cap` records copied to host `rec` (may be NULL); *nctr = the rank's
 * counter count; info (may be NULL) = {panel blocks per tile b/s, columns per register pass,
 * register passes per tile, tile rows per unit}.  TQR_ERR_INVALID_ARG: 1 m, 2 n, 3 (b, s)
 * without a kernel instance, 5 nranks, 6 rank, 7 workers, 8 tall flag off its (256, 32, 1 rank)
 * instance, 11 ntask NULL. */
tqr_status tqr_schedule_records_policy(int64_t m, int64_t n, int32_t b, int32_t s, int32_t nranks, int32_t rank,
                                       int32_t workers, uint32_t flags, int32_t* rec, int64_t cap, int64_t* ntask,
                                       int32_t* nctr, int32_t info[4]);

/* Scaling MODEL (not a measurement; pure host): the list-schedule simulation the dispatch order
 * comes from, run for an m x n factorization with the plan policy for (b, s) on `nranks`
 * ranks of `workers` CTAs each (1D block-cyclic columns), task durations from the B200-fitted
 * duration model, plus `remote_ns` on every dependency whose producer runs on another rank.
 * *makespan_ns = modelled factorization time; *busy (may be NULL) = modelled utilisation. */
tqr_status tqr_schedule_model(int64_t m, int64_t n, int32_t b, int32_t s, int32_t nranks, int32_t workers,
                              double remote_ns, double* makespan_ns, double* busy);

/* The factorization dispatch records THIS plan executes (same 16-int32 layout), for its
 * local rank index `local` (0 .. ranks run by this process - 1; emulated plans run every
 * rank): *n = task count, up to `cap` records copied to host `rec` (synchronous device copy).
 * Lets tests check which task granularities (register passes per update task, record [15])
 * a parity case actually exercises.  TQR_ERR_INVALID_ARG(2) for a bad local index. */
tqr_status tqr_plan_records(tqr_plan* plan, int32_t local, int32_t* rec, int64_t cap, int64_t* n);
/* Policy the plan chose (host): info[0] rows-per-warp variant (128 / 256), [1] register passes
 * per default update task, [2] register passes (column slices) per tile, [3] panel A/F split,
 * [4] early R_kk release, [5] executor CTAs, [6] priority (0 classes, 1 bottom level),
 * [7] fine-granularity rule (R23), [8] internal inner block SI of the executor (== s
 * except b*s > 8192, R16), [9] ranks of the job, [10] ranks run by this process,
 * [11] columns per register pass, [12] tile rows per TSQRT / SSRFB unit (1, or 2 with
 * TQR_FLAG_TALL_TILES), [13..15] 0. */
tqr_status tqr_plan_info(const tqr_plan* plan, int32_t info[16]);

/* Trace of the last tqr_geqrf with TQR_FLAG_TRACE: up to `cap` records of
 * {kind, k, i, j, slice | flags << 16, sm, start_ns, end_ns} as 8 int64 each (host memory;
 * flags = the low byte of task record [14]: 2 panel apply part, 4 panel factor part);
 * returns the number of records written in *n. */
tqr_status tqr_trace_fetch(tqr_plan* plan, int64_t* rec, int64_t cap, int64_t* n);

/* Profiling aid: run `count` mutually independent tasks of one kind (0 = GEQRT, 1 = TSQRT
 * (whole tiles), 2 = LARFB slice, 3 = SSRFB slice, 4..7 the apply-Q kinds, 8 / 9 = the factor
 * part alone of one inner block of a GEQRT / TSQRT, R21) through the same persistent executor on the plan's
 * tiles, with no DAG dependencies.  Results in At/T are meaningless afterwards (tasks race
 * on shared tiles); only the timing is.  Used to profile one kernel body in isolation with
 * ncu.  Requires p >= 2 and q >= 2. */
tqr_status tqr_profile_tasks(tqr_plan* plan, int32_t kind, int64_t count, double* At, double* T, void* work);

/* Profiling builds only (libtqr_phases.so, compiled with -DTQR_PROFILE_PHASES): attach a
 * caller-owned device array of 16 int64 per-phase clock64 totals (thread 0 of every CTA adds
 * its cycles in: 0 update prologue up to the first staged block, 1 ticket + task record,
 * 2 end-of-task barrier, 3 release, 4 update phase of an update task, 5 its epilogue,
 * 6 dependency wait, 7 update phase of a panel task, 8 panel staging, 9 panel factorization,
 * 10 V/R out, 11 Gram + packed Y out, 12 T build, 13 T out).  NULL detaches.  No-op in
 * product builds. */
tqr_status tqr_phase_counters(tqr_plan* plan, long long* d_counters);

#ifdef __cplusplus
}
#endif
#endif /* TQR_H */
