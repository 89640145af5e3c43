/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the tiled QR
 * factorization of arXiv 0707.3548 (PAPER.md, "Tiled algorithms" section).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_0707_3548_b200/) never links, imports or calls it.
 * It shares no code, header, table or helper with the CUDA path.
 *
 * Conventions (all fp64, IEEE round-to-nearest, compiled -O2 -ffp-contract=off):
 *   - A tile is b x b, column-major: element (r,c) at r + c*b.
 *   - Block Data Layout: tile (i,j) of the p x q grid is at
 *     offset (i + j*p)*b*b ("blocks are stored in Column Major Format with
 *     respect to each other").
 *   - T factors: slot (i,k) holds s x b doubles at offset (i + k*p)*s*b; inside a
 *     slot, T_l (s x s, upper triangular) occupies columns [l*s, l*s+s):
 *     T_l[r][c] at (l*s + c)*s + r.  Slot (k,k) is GEQRT's T_kk, slot (i,k),
 *     i>k, is TSQRT's T_ik.  Inner blocking s is DESIGN.md reading R5
 *     (the paper's kernels are the s == b case).
 *   - Updates apply Q^T = I - V T^T V^T  (reading R1; the paper's
 *     printed "(I - V T V^T)" at PAPER.md:401,436-466 is the forward-T
 *     product H_1...H_b, whose transpose is what the factorization applies).
 *
 * Return codes: 0 ok, -k invalid argument number k.
 */
#ifndef TQR_ORACLE_H
#define TQR_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Householder generator, readings R2/R3/R4 (paper silent). */
void oracle_house(double alpha, const double* x, int64_t L, double* beta, double* tau, double* v);

/* Tile kernels ("A Fine-Grain Algorithm for QR Factorization"). */
int oracle_geqrt(int b, int s, double* A, double* T);                      /* DGEQT2 */
int oracle_tsqrt(int b, int s, double* R, double* B, double* T);           /* DTSQT2 */
int oracle_larfb(int b, int s, const double* V, const double* T, double* C, int trans); /* DLARFB */
int oracle_ssrfb(int b, int s, const double* V, const double* T, double* C1, double* C2, int trans); /* DSSRFB */
/* trans = 1 applies Q^T (factorization, l ascending, T_l^T);
 * trans = 0 applies Q (l descending, T_l), used by apply-Q / form-Q. */

/* TSQRT / SSRFB with `rows` rows in the lower block (ld = rows; rows = b: the functions above;
 * rows = h b: the non-square 2b x b tiles of P:582-583, reading R30). */
int oracle_tsqrt_rows(int b, int s, int rows, double* R, double* B, double* T);
int oracle_ssrfb_rows(int b, int s, int rows, const double* V, const double* T, double* C1, double* C2, int trans);

/* Block Data Layout pack/unpack, zero padding (R9). */
int oracle_pack(int64_t m, int64_t n, int b, const double* A, int64_t lda, double* At);
int oracle_unpack(int64_t m, int64_t n, int b, const double* At, double* A, int64_t lda);

/* Algorithm 1 on a tile-major matrix.  nthreads == 1 runs the
 * loop nest literally; nthreads > 1 runs the same tasks as a DAG with the
 * paper's 4-level priorities on POSIX threads.  Results are
 * bitwise identical either way (each tile's operation sequence is fixed by the
 * DAG edges). */
int oracle_geqrf_tiles(int64_t m, int64_t n, int b, int s, double* At, double* T, int nthreads);

/* Algorithm 1 with the tile rows below the diagonal grouped in units of h (R30:
 * units k+1.., k+1+h.., ...; the last may be shorter): TSQRT / SSRFB work on the (nt b) x b
 * stack of a unit's tiles; its T factors are in the T slot of its first tile row (the other
 * slots stay 0).  h = 1 is oracle_geqrf_tiles. */
int oracle_geqrf_tiles_h(int64_t m, int64_t n, int b, int s, int h, double* At, double* T, int nthreads);
int oracle_ormqr_tiles_h(int64_t m, int64_t n, int b, int s, int h, const double* At, const double* T,
                         int trans, int64_t nrhs, double* Bt, int nthreads);
int64_t oracle_dag_edges_h(int64_t p, int64_t q, int h, int64_t* out, int64_t cap);
double oracle_flops_eq4_h(int64_t p, int64_t q, double b, int h);

/* Apply Q^T (trans=1) or Q (trans=0) to a tile-major m x nrhs matrix Bt
 * (same row tiling p = ceil(m/b); ceil(nrhs/b) tile columns).
 * ("DORMQR"-style future use; R8.) */
int oracle_ormqr_tiles(int64_t m, int64_t n, int b, int s, const double* At, const double* T,
                       int trans, int64_t nrhs, double* Bt, int nthreads);

/* R = upper trapezoid, min(m,n) x n column-major, zeros below the diagonal. */
int oracle_get_r(int64_t m, int64_t n, int b, const double* At, double* R, int64_t ldr);

/* Flop models.  Standard LAPACK count 2n^2(m - n/3).
 * Paper per-kernel model 2b^3, 3b^3, 10/3 b^3, 5b^3,
 * kind: 0=GEQT2 1=LARFB 2=TSQT2 3=SSRFB.  Eq. (4) exact sum. */
double oracle_flops_standard(int64_t m, int64_t n);
double oracle_kernel_flops(int kind, double b);
double oracle_flops_eq4(int64_t p, int64_t q, double b);

/* Test hook: the DAG edges of Algorithm 1 for a p x q grid (SPEC dag module rules), as 8 int64
 * per edge {kind, k, i, j} of predecessor and successor (kind 0 G, 1 T, 2 L, 3 S).  Returns
 * the edge count (-1 on bad p, q); writes at most cap edges. */
int64_t oracle_dag_edges(int64_t p, int64_t q, int64_t* out, int64_t cap);

/* Test hook: count of tasks executed by the last oracle_geqrf_tiles call, per kind. */
void oracle_last_task_counts(int64_t counts[4]);

#ifdef __cplusplus
}
#endif
#endif
