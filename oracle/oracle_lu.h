/*
 * oracle_lu.h -- plain, slow, obviously-correct CPU oracle for the tiled LU factorization
 * the paper names as its first extension ("Implement other linear algebra
 * operations": "The LU factorization can be performed with an algorithm that is analogous to
 * the QR one described in Section [tiled] ... the only difference between the block
 * algorithms for the LU and QR factorizations is in the elementary operations").
 *
 * TEST INFRASTRUCTURE ONLY (same rules as oracle.h): only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs load it; it shares no code, header or
 * helper with the CUDA path.
 *
 * The paper does not spell the LU elementary operations out; readings LU1-LU7 fix
 * them (pairwise / incremental pivoting, the out-of-core LU the paper cites):
 *   GETRF(k)      A_kk = its own in-tile LU with partial pivoting, inner blocking s
 *                 (the analogue of GEQRT);
 *   GESSM(k,j)    A_kj <- (GETRF(k)'s row interchanges and unit-lower eliminations) A_kj
 *                 (the analogue of LARFB);
 *   TSTRF(k,i)    LU with partial pivoting of the stacked [U_kk; A_ik] (the analogue of TSQRT,
 *                 PAPER.md:404-428; pivot candidates: the diagonal row of U_kk and every row of
 *                 A_ik);
 *   SSSSM(k,i,j)  [A_kj; A_ij] <- (TSTRF(k,i)'s interchanges and eliminations) [A_kj; A_ij]
 *                 (the analogue of SSRFB).
 *
 * Storage (same Block Data Layout as the QR oracle):
 *   tiles  At: tile (i,j) at (i + j p) b^2, column-major inside; after the factorization U is
 *          the upper trapezoid, the multipliers of GETRF (strict lower part of A_kk) and of
 *          TSTRF (all of A_ik) are stored in place;
 *   Lt     p*K slots of s x b doubles (like T), slot (i,k) at (i + k p) s b: for i > k block l's
 *          s x s unit-lower Ltilde_l (strict lower part; its diagonal and upper part are 0) in
 *          columns [l s, l s + s): Ltilde_l[r][c] at (l s + c) s + r;  slot (k,k) unused (0);
 *   piv    p*K slots of b int32, slot (i,k) at (i + k p) b:
 *          GETRF: piv[c] = the tile row (in [c, b)) interchanged with row c;
 *          TSTRF: piv[c] = -1 if U_kk's row c stayed the pivot row, else the row r in [0, b) of
 *          A_ik interchanged with it.
 * Return codes: 0 ok, -k invalid argument number k.
 */
#ifndef TQR_ORACLE_LU_H
#define TQR_ORACLE_LU_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Tile kernels (tiles b x b column-major, inner blocking s | b). */
int oracle_lu_getrf(int b, int s, double* A, int32_t* piv);
int oracle_lu_gessm(int b, int s, const double* L, const int32_t* piv, double* C);
int oracle_lu_tstrf(int b, int s, double* U, double* A, double* Lt, int32_t* piv);
int oracle_lu_ssssm(int b, int s, const double* V, const double* Lt, const int32_t* piv, double* C1, double* C2);

/* The tiled factorization of an m x n matrix in tile layout (zero-padded, like the QR oracle's
 * pack): step k = GETRF(k); GESSM(k, j > k); TSTRF(k, i > k) in i order; SSSSM(k, i, j > k).
 * nthreads > 1 runs the updates of different tile columns in parallel (every tile's sequence
 * of operations is the same, so the result is bitwise identical to nthreads = 1). */
int oracle_lu_getrf_tiles(int64_t m, int64_t n, int b, int s, double* At, double* Lt, int32_t* piv, int nthreads);

/* The same factorization with every pivot FORCED to forced[] (same layout as piv; DESIGN.md
 * LU10: where rounding decides a pivot, several pivot sequences are correct).  *nearties =
 * decisions where the forced pivot differs from the search's but its |candidate| is within
 * `rel` (relative) of the largest; *invalid = decisions where it is not (a wrong pivot).
 * Not thread-safe across concurrent calls (one forced sequence at a time). */
int oracle_lu_getrf_tiles_forced(int64_t m, int64_t n, int b, int s, double* At, double* Lt, int32_t* piv,
                                  const int32_t* forced, double rel, int64_t* nearties, int64_t* invalid,
                                  int nthreads);

/* Forward application of the factorization's transformation M (= every interchange and
 * elimination of the factorization, in its order) to a tile-major B with p tile rows and
 * qb tile columns (same b): B <- M B.  With M A = U: the forward half of a solve. */
int oracle_lu_apply(int64_t m, int64_t n, int b, int s, const double* At, const double* Lt, const int32_t* piv,
                    int64_t qb, double* Bt, int nthreads);

/* Solve A X = B for square A (m = n) with the tiled factors: B <- U^{-1} M B, tile-major B. */
int oracle_lu_solve(int64_t n, int b, int s, const double* At, const double* Lt, const int32_t* piv,
                    int64_t qb, double* Bt, int nthreads);

/* Leading-order flop counts: standard LU  mn^2 - n^3/3 (m >= n; LAPACK dgetrf's count), and
 * the tiled algorithm's executed count (every kernel's multiply-adds x 2, s-blocked). */
double oracle_lu_flops_standard(int64_t m, int64_t n);
double oracle_lu_flops_tiled(int64_t m, int64_t n, int b, int s);

#ifdef __cplusplus
}
#endif
#endif
