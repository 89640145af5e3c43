/*
 * oracle_lu.c -- plain CPU oracle for the tiled LU factorization.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle_lu.h): loaded by tests/, smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, never by the product path.
 *
 * Every routine is a literal, loop-by-loop transcription of the step it cites and of the
 * DESIGN.md reading (LU1-LU7) that fixes what the paper leaves open; no blocking, fusion
 * or reordering beyond that.  Compiled with -O2 -ffp-contract=off (no FMA contraction).
 */
#include "oracle_lu.h"
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define TILE(At, i, j, p, b) ((At) + ((int64_t)(i) + (int64_t)(j) * (p)) * (int64_t)(b) * (b))
#define LSLOT(L, i, k, p, s, b) ((L) + ((int64_t)(i) + (int64_t)(k) * (p)) * (int64_t)(s) * (b))
#define PSLOT(P, i, k, p, b) ((P) + ((int64_t)(i) + (int64_t)(k) * (p)) * (int64_t)(b))
#define E(X, r, c, b) (X)[(int64_t)(r) + (int64_t)(c) * (b)]

static int check_bs(int b, int s) {
  if (b < 1) return -1;
  if (s < 1 || s > b || b % s != 0) return -2;
  return 0;
}

static void swap_rows(double* X, int ldx, int r1, double* Y, int ldy, int r2, int c_lo, int c_hi) {
  for (int c = c_lo; c < c_hi; ++c) {
    double t = X[r1 + (int64_t)c * ldx];
    X[r1 + (int64_t)c * ldx] = Y[r2 + (int64_t)c * ldy];
    Y[r2 + (int64_t)c * ldy] = t;
  }
}

/* One inner block l of GESSM (LU2, PAPER.md:395-402 analogue) on columns
 * [c_lo, c_hi) of C (ld b): the block's interchanges (rows c <-> piv[c], c ascending), the
 * unit-lower triangular solve of rows [c0, c0+s) with L11 (forward substitution, row order),
 * then rows [c0+s, b) -= L21 * rows [c0, c0+s). */
static void gessm_block(int b, int s, int l, const double* L, const int32_t* piv, double* C, int c_lo, int c_hi) {
  const int c0 = l * s;
  for (int c = c0; c < c0 + s; ++c)
    if (piv[c] != c) swap_rows(C, b, c, C, b, piv[c], c_lo, c_hi);
  for (int t = c_lo; t < c_hi; ++t)
    for (int c = c0; c < c0 + s; ++c)
      for (int c2 = c0; c2 < c; ++c2) E(C, c, t, b) -= E(L, c, c2, b) * E(C, c2, t, b);
  for (int t = c_lo; t < c_hi; ++t)
    for (int r = c0 + s; r < b; ++r) {
      double acc = 0.0;
      for (int c = c0; c < c0 + s; ++c) acc += E(L, r, c, b) * E(C, c, t, b);
      E(C, r, t, b) -= acc;
    }
}

/* One inner block l of SSSSM (LU4, PAPER.md:430-466 analogue) on columns
 * [c_lo, c_hi) of the stacked [C1; C2] (both ld b): interchanges C1 row c <-> C2 row piv[c]
 * (piv[c] >= 0; c ascending), C1 rows [c0, c0+s) <- (I + Ltilde_l)^{-1} C1 rows [c0, c0+s)
 * (forward substitution), then C2 -= V[:, c0:c0+s] * C1 rows [c0, c0+s). */
static void ssssm_block(int b, int s, int l, const double* V, const double* Lt, const int32_t* piv, double* C1,
                        double* C2, int c_lo, int c_hi) {
  const int c0 = l * s;
  for (int c = c0; c < c0 + s; ++c)
    if (piv[c] >= 0) swap_rows(C1, b, c, C2, b, piv[c], c_lo, c_hi);
  for (int t = c_lo; t < c_hi; ++t)
    for (int jj = 0; jj < s; ++jj)
      for (int j2 = 0; j2 < jj; ++j2)
        E(C1, c0 + jj, t, b) -= Lt[(int64_t)(c0 + j2) * s + jj] * E(C1, c0 + j2, t, b);
  for (int t = c_lo; t < c_hi; ++t)
    for (int r = 0; r < b; ++r) {
      double acc = 0.0;
      for (int c = c0; c < c0 + s; ++c) acc += E(V, r, c, b) * E(C1, c, t, b);
      E(C2, r, t, b) -= acc;
    }
}

/* GETRF(k) (LU1): in-tile LU with partial pivoting, inner blocking s.  For each
 * block l and column c in it: the pivot is the first row of largest |A[r][c]|, r in [c, b)
 * (LAPACK idamax); rows c and piv[c] are interchanged in the block's columns only (the
 * earlier blocks' multipliers stay where they were computed: LU3); the multipliers
 * A[r][c] /= A[c][c] (r > c; skipped if the pivot is 0 -- then the whole column is 0); the
 * rank-1 update of the block's later columns; after the block, the trailing columns get the
 * block's interchanges and eliminations (gessm_block). */
/* Forced-pivot mode (LU10; test infrastructure for pivots decided by rounding):
 * when g_forced is set, the pivot of every column is taken from it instead of the search;
 * a forced pivot that differs from the search's counts as a near-tie if its |candidate| is
 * within g_rel (relative) of the largest, as invalid otherwise. */
static const int32_t* g_forced = NULL;
static double g_rel = 0.0;
static int64_t g_nearties = 0, g_invalid = 0;

static int take_forced(int pr, int fp, double best, double fv) {
  if (fp != pr) {
    if (fv >= best * (1.0 - g_rel)) g_nearties++;
    else g_invalid++;
  }
  return fp;
}

int oracle_lu_getrf(int b, int s, double* A, int32_t* piv) {
  int rc = check_bs(b, s);
  if (rc) return rc;
  const int32_t* forced = g_forced;
  for (int l = 0; l < b / s; ++l) {
    const int c0 = l * s;
    for (int c = c0; c < c0 + s; ++c) {
      int pr = c;
      double best = fabs(E(A, c, c, b));
      for (int r = c + 1; r < b; ++r)
        if (fabs(E(A, r, c, b)) > best) { best = fabs(E(A, r, c, b)); pr = r; }
      if (forced) pr = take_forced(pr, forced[c], best, fabs(E(A, forced[c], c, b)));
      piv[c] = pr;
      if (pr != c) swap_rows(A, b, c, A, b, pr, c0, c0 + s);
      const double d = E(A, c, c, b);
      if (d != 0.0)
        for (int r = c + 1; r < b; ++r) E(A, r, c, b) /= d;
      for (int c2 = c + 1; c2 < c0 + s; ++c2)
        for (int r = c + 1; r < b; ++r) E(A, r, c2, b) -= E(A, r, c, b) * E(A, c, c2, b);
    }
    gessm_block(b, s, l, A, piv, A, c0 + s, b);
  }
  return 0;
}

/* GESSM(k,j): every block of GETRF(k) applied to C = A_kj, l ascending. */
int oracle_lu_gessm(int b, int s, const double* L, const int32_t* piv, double* C) {
  int rc = check_bs(b, s);
  if (rc) return rc;
  for (int l = 0; l < b / s; ++l) gessm_block(b, s, l, L, piv, C, 0, b);
  return 0;
}

/* TSTRF(k,i) (LU3): LU with partial pivoting of the stacked [U; A] (U = the upper
 * triangle of A_kk incl. its diagonal, A = A_ik), inner blocking s.  Column c of block l:
 * candidates are U's row c (its entry U[c][c]) and every row of A; the first largest |.| wins,
 * U's row first (LU5).  If A's row r wins, U's row c and A's row r are interchanged in the
 * block's columns: the multipliers A[r][c0..c) move into Ltilde_l's row c - c0 and A's row r
 * takes U's row c (zeros left of the diagonal, LU3).  Multipliers A[r][c] /= U[c][c] (all r;
 * skipped if 0), rank-1 update of the block's later columns of A (U's rows below c are 0 in
 * column c), then the trailing columns [c0+s, b) get the block's interchanges and
 * eliminations (ssssm_block).  U's strict lower part (GETRF's multipliers) is never touched. */
int oracle_lu_tstrf(int b, int s, double* U, double* A, double* Lt, int32_t* piv) {
  int rc = check_bs(b, s);
  if (rc) return rc;
  const int32_t* forced = g_forced;
  for (int64_t e = 0; e < (int64_t)s * b; ++e) Lt[e] = 0.0;
  for (int l = 0; l < b / s; ++l) {
    const int c0 = l * s;
    double* Ll = Lt + (int64_t)c0 * s; /* Ltilde_l[r][c] at c*s + r */
    for (int c = c0; c < c0 + s; ++c) {
      const int jj = c - c0;
      int pr = -1;
      double best = fabs(E(U, c, c, b));
      for (int r = 0; r < b; ++r)
        if (fabs(E(A, r, c, b)) > best) { best = fabs(E(A, r, c, b)); pr = r; }
      if (forced) {
        const int fp = forced[c];
        pr = take_forced(pr, fp, best, fp < 0 ? fabs(E(U, c, c, b)) : fabs(E(A, fp, c, b)));
      }
      piv[c] = pr;
      if (pr >= 0) {
        for (int c2 = c0; c2 < c; ++c2) { /* L part: A's multipliers up, zeros down */
          Ll[(int64_t)(c2 - c0) * s + jj] = E(A, pr, c2, b);
          E(A, pr, c2, b) = 0.0;
        }
        swap_rows(U, b, c, A, b, pr, c, c0 + s);
      }
      const double d = E(U, c, c, b);
      if (d != 0.0)
        for (int r = 0; r < b; ++r) E(A, r, c, b) /= d;
      for (int c2 = c + 1; c2 < c0 + s; ++c2)
        for (int r = 0; r < b; ++r) E(A, r, c2, b) -= E(A, r, c, b) * E(U, c, c2, b);
    }
    ssssm_block(b, s, l, A, Lt, piv, U, A, c0 + s, b);
  }
  return 0;
}

/* SSSSM(k,i,j): every block of TSTRF(k,i) applied to [C1; C2] = [A_kj; A_ij], l ascending. */
int oracle_lu_ssssm(int b, int s, const double* V, const double* Lt, const int32_t* piv, double* C1, double* C2) {
  int rc = check_bs(b, s);
  if (rc) return rc;
  for (int l = 0; l < b / s; ++l) ssssm_block(b, s, l, V, Lt, piv, C1, C2, 0, b);
  return 0;
}

/* ---- tiled driver (the analogue of Algorithm 1) ------------------------ */
typedef struct {
  int64_t p, q, qb, b, s;
  const double* At;  /* factors */
  double* Aw;        /* factorization: the tiles being factored */
  double* Lt;
  int32_t* piv;
  double* Bt;        /* apply: the right-hand sides */
  int64_t k, j0, j1;
} lu_ctx;

/* step k, tile columns [j0, j1): GESSM(k,j), then SSSSM(k,i,j) for i ascending */
static void step_columns(const lu_ctx* X) {
  const int b = (int)X->b, s = (int)X->s;
  const int64_t p = X->p, k = X->k;
  for (int64_t j = X->j0; j < X->j1; ++j) {
    oracle_lu_gessm(b, s, TILE(X->Aw, k, k, p, b), PSLOT(X->piv, k, k, p, b), TILE(X->Aw, k, j, p, b));
    for (int64_t i = k + 1; i < p; ++i)
      oracle_lu_ssssm(b, s, TILE(X->Aw, i, k, p, b), LSLOT(X->Lt, i, k, p, s, b), PSLOT(X->piv, i, k, p, b),
                      TILE(X->Aw, k, j, p, b), TILE(X->Aw, i, j, p, b));
  }
}
static void* step_worker(void* a) { step_columns((const lu_ctx*)a); return NULL; }

static void for_columns(lu_ctx* X, int64_t jlo, int64_t jhi, int nthreads, void (*fn)(const lu_ctx*),
                        void* (*wk)(void*)) {
  const int64_t nj = jhi - jlo;
  if (nj <= 0) return;
  int nt = nthreads < 1 ? 1 : nthreads;
  if (nt > nj) nt = (int)nj;
  if (nt == 1) { X->j0 = jlo; X->j1 = jhi; fn(X); return; }
  lu_ctx* cx = (lu_ctx*)malloc(sizeof(lu_ctx) * nt);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nt);
  for (int t = 0; t < nt; ++t) {
    cx[t] = *X;
    cx[t].j0 = jlo + nj * t / nt;
    cx[t].j1 = jlo + nj * (t + 1) / nt;
    pthread_create(&th[t], NULL, wk, &cx[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  free(cx);
  free(th);
}

int oracle_lu_getrf_tiles(int64_t m, int64_t n, int b, int s, double* At, double* Lt, int32_t* piv, int nthreads) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  int rc = check_bs(b, s);
  if (rc) return rc - 2;
  if (nthreads < 1) return -8;
  const int64_t p = (m + b - 1) / b, q = (n + b - 1) / b, K = p < q ? p : q;
  for (int64_t e = 0; e < p * K * (int64_t)s * b; ++e) Lt[e] = 0.0;
  for (int64_t e = 0; e < p * K * (int64_t)b; ++e) piv[e] = 0;
  lu_ctx X = {p, q, 0, b, s, At, At, Lt, piv, NULL, 0, 0, 0};
  const int32_t* forced_all = g_forced;
  for (int64_t k = 0; k < K; ++k) {
    if (forced_all) g_forced = PSLOT(forced_all, k, k, p, b);
    oracle_lu_getrf(b, s, TILE(At, k, k, p, b), PSLOT(piv, k, k, p, b));
    /* TSTRF(k, i) reads only U_kk and A_ik: all of them first (i ascending: the flat chain on
     * U_kk), then the tile columns' GESSM + SSSSM chains, in parallel over j */
    for (int64_t i = k + 1; i < p; ++i) {
      if (forced_all) g_forced = PSLOT(forced_all, i, k, p, b);
      oracle_lu_tstrf(b, s, TILE(At, k, k, p, b), TILE(At, i, k, p, b), LSLOT(Lt, i, k, p, s, b),
                      PSLOT(piv, i, k, p, b));
    }
    g_forced = forced_all;
    X.k = k;
    for_columns(&X, k + 1, q, nthreads, step_columns, step_worker);
  }
  return 0;
}

int oracle_lu_getrf_tiles_forced(int64_t m, int64_t n, int b, int s, double* At, double* Lt, int32_t* piv,
                                  const int32_t* forced, double rel, int64_t* nearties, int64_t* invalid,
                                  int nthreads) {
  if (!forced) return -8;
  g_forced = forced;
  g_rel = rel;
  g_nearties = g_invalid = 0;
  int rc = oracle_lu_getrf_tiles(m, n, b, s, At, Lt, piv, nthreads);
  g_forced = NULL;
  if (nearties) *nearties = g_nearties;
  if (invalid) *invalid = g_invalid;
  return rc;
}

/* apply M to B: the same step sequence with the factors read-only, on B's tile columns */
static void apply_columns(const lu_ctx* X) {
  const int b = (int)X->b, s = (int)X->s;
  const int64_t p = X->p, K = X->p < X->q ? X->p : X->q;
  for (int64_t jb = X->j0; jb < X->j1; ++jb)
    for (int64_t k = 0; k < K; ++k) {
      oracle_lu_gessm(b, s, TILE(X->At, k, k, p, b), PSLOT(X->piv, k, k, p, b), TILE(X->Bt, k, jb, p, b));
      for (int64_t i = k + 1; i < p; ++i)
        oracle_lu_ssssm(b, s, TILE(X->At, i, k, p, b), LSLOT(X->Lt, i, k, p, s, b), PSLOT(X->piv, i, k, p, b),
                        TILE(X->Bt, k, jb, p, b), TILE(X->Bt, i, jb, p, b));
    }
}
static void* apply_worker(void* a) { apply_columns((const lu_ctx*)a); return NULL; }

int oracle_lu_apply(int64_t m, int64_t n, int b, int s, const double* At, const double* Lt, const int32_t* piv,
                    int64_t qb, double* Bt, int nthreads) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  int rc = check_bs(b, s);
  if (rc) return rc - 2;
  if (qb < 1) return -8;
  const int64_t p = (m + b - 1) / b, q = (n + b - 1) / b;
  lu_ctx X = {p, q, qb, b, s, At, NULL, (double*)Lt, (int32_t*)piv, Bt, 0, 0, 0};
  for_columns(&X, 0, qb, nthreads, apply_columns, apply_worker);
  return 0;
}

/* back substitution with the tiled U (upper triangle of the diagonal tiles, full tiles above):
 * for k descending: B(k) <- U_kk^{-1} B(k) (rows descending), B(i) -= U_ik B(k) for i < k */
static void backsub_columns(const lu_ctx* X) {
  const int64_t b = X->b, p = X->p;
  for (int64_t jb = X->j0; jb < X->j1; ++jb)
    for (int64_t k = p - 1; k >= 0; --k) {
      const double* Ukk = TILE(X->At, k, k, p, b);
      double* Bk = TILE(X->Bt, k, jb, p, b);
      for (int64_t t = 0; t < b; ++t)
        for (int64_t r = b - 1; r >= 0; --r) {
          double acc = E(Bk, r, t, b);
          for (int64_t c = r + 1; c < b; ++c) acc -= E(Ukk, r, c, b) * E(Bk, c, t, b);
          E(Bk, r, t, b) = acc / E(Ukk, r, r, b);
        }
      for (int64_t i = 0; i < k; ++i) {
        const double* Uik = TILE(X->At, i, k, p, b);
        double* Bi = TILE(X->Bt, i, jb, p, b);
        for (int64_t t = 0; t < b; ++t)
          for (int64_t r = 0; r < b; ++r) {
            double acc = 0.0;
            for (int64_t c = 0; c < b; ++c) acc += E(Uik, r, c, b) * E(Bk, c, t, b);
            E(Bi, r, t, b) -= acc;
          }
      }
    }
}
static void* backsub_worker(void* a) { backsub_columns((const lu_ctx*)a); return NULL; }

int oracle_lu_solve(int64_t n, int b, int s, const double* At, const double* Lt, const int32_t* piv, int64_t qb,
                    double* Bt, int nthreads) {
  if (n < 1) return -1;
  if (n % b != 0) return -1; /* the padded diagonal would be singular: square, whole tiles only */
  int rc = oracle_lu_apply(n, n, b, s, At, Lt, piv, qb, Bt, nthreads);
  if (rc) return rc;
  lu_ctx X = {n / b, n / b, qb, b, s, At, NULL, NULL, NULL, Bt, 0, 0, 0};
  for_columns(&X, 0, qb, nthreads, backsub_columns, backsub_worker);
  return 0;
}

/* ---- flop counts -------------------------------------------------------------------------- */
double oracle_lu_flops_standard(int64_t m, int64_t n) {
  const double M = (double)m, N = (double)n;
  if (m >= n) return M * N * N - N * N * N / 3.0;
  return N * M * M - M * M * M / 3.0;
}

/* per kernel, exactly as the routines above count them (a multiply-add = 2, a division = 1) */
static double fl_getrf(double b, double s) {
  double f = 0.0;
  for (double c0 = 0; c0 < b; c0 += s) {
    for (double c = c0; c < c0 + s; ++c) f += (b - c - 1) + 2.0 * (b - c - 1) * (c0 + s - c - 1);
    const double tc = b - c0 - s;
    f += s * (s - 1) * tc + 2.0 * (b - c0 - s) * s * tc;
  }
  return f;
}
static double fl_gessm(double b, double s) {
  double f = 0.0;
  for (double c0 = 0; c0 < b; c0 += s) f += s * (s - 1) * b + 2.0 * (b - c0 - s) * s * b;
  return f;
}
static double fl_tstrf(double b, double s) {
  double f = 0.0;
  for (double c0 = 0; c0 < b; c0 += s) {
    for (double c = c0; c < c0 + s; ++c) f += b + 2.0 * b * (c0 + s - c - 1);
    const double tc = b - c0 - s;
    f += s * (s - 1) * tc + 2.0 * b * s * tc;
  }
  return f;
}
static double fl_ssssm(double b, double s) { return (b / s) * (s * (s - 1) * b + 2.0 * b * s * b); }

double oracle_lu_flops_tiled(int64_t m, int64_t n, int b, int s) {
  const int64_t p = (m + b - 1) / b, q = (n + b - 1) / b, K = p < q ? p : q;
  const double fg = fl_getrf(b, s), fl = fl_gessm(b, s), ft = fl_tstrf(b, s), fs = fl_ssssm(b, s);
  double f = 0.0;
  for (int64_t k = 0; k < K; ++k) {
    const double nr = (double)(p - k - 1), nc = (double)(q - k - 1);
    f += fg + nc * fl + nr * ft + nr * nc * fs;
  }
  return f;
}
