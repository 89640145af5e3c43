/*
 * oracle.c -- plain CPU oracle for tiled QR (arXiv 0707.3548).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): loaded by tests/, smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, never by the product path.
 *
 * Every routine is a literal, loop-by-loop transcription of the step it cites;
 * there is no blocking, fusion or reordering beyond what the cited text or the
 * DESIGN.md reading states.  Compiled with -O2 -ffp-contract=off (no FMA
 * contraction, no reassociation).
 */
#include "oracle.h"
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define TILE(At, i, j, p, b) ((At) + ((int64_t)(i) + (int64_t)(j) * (p)) * (int64_t)(b) * (b))
#define TSLOT(T, i, k, p, s, b) ((T) + ((int64_t)(i) + (int64_t)(k) * (p)) * (int64_t)(s) * (b))

/* ---------------------------------------------------------------------------
 * Householder generator.  PAPER.md:141-149 ("applying min(m,n) Householder
 * reflections"); the generator itself is unstated, DESIGN.md
 * readings R2-R4:
 *   sigma = sum_{r} x_r^2 (ascending r)
 *   sigma == 0      : tau = 0, beta = alpha, v = 0            (R3, dlarfg)
 *   otherwise       : nu = sqrt(alpha^2 + sigma);
 *                     beta = -nu if alpha >= 0 (incl. -0.0), else +nu  (R2)
 *                     tau = (beta - alpha)/beta;  v = x / (alpha - beta)
 *   H = I - tau u u^T, u = (1, v), H (alpha, x)^T = (beta, 0)^T.
 * No overflow/underflow rescaling (R4).  v may alias x.
 * ------------------------------------------------------------------------- */
void oracle_house(double alpha, const double* x, int64_t L, double* beta, double* tau, double* v) {
  double sigma = 0.0;
  for (int64_t r = 0; r < L; ++r) sigma += x[r] * x[r];
  if (sigma == 0.0) {
    *tau = 0.0;
    *beta = alpha;
    for (int64_t r = 0; r < L; ++r) v[r] = 0.0;
    return;
  }
  double nu = sqrt(alpha * alpha + sigma);
  double bt = (alpha >= 0.0) ? -nu : nu;
  double denom = alpha - bt;
  *beta = bt;
  *tau = (bt - alpha) / bt;
  for (int64_t r = 0; r < L; ++r) v[r] = x[r] / denom;
}

/* T_l column j (forward, column-wise DLARFT; PAPER.md:153-157, 213-219;
 * DESIGN.md R6):  T_l[j][j] = tau;  T_l[0:j, j] = -tau * T_l[0:j, 0:j] * z. */
static void larft_column(double* Tl, int s, int j, double tau, const double* z) {
  Tl[(int64_t)j * s + j] = tau;
  for (int t = 0; t < j; ++t) {
    double acc = 0.0;
    for (int tp = t; tp < j; ++tp) acc += Tl[(int64_t)tp * s + t] * z[tp];
    Tl[(int64_t)j * s + t] = -tau * acc;
  }
}

/* W <- T_l^T W (trans=1) or W <- T_l W (trans=0), W of length s, T_l upper. */
static void apply_tl(const double* Tl, int s, double* W, double* W2, int trans) {
  for (int a = 0; a < s; ++a) {
    double acc = 0.0;
    if (trans) {
      for (int ap = 0; ap <= a; ++ap) acc += Tl[(int64_t)a * s + ap] * W[ap];
    } else {
      for (int ap = a; ap < s; ++ap) acc += Tl[(int64_t)ap * s + a] * W[ap];
    }
    W2[a] = acc;
  }
}

static int check_bs(int b, int s) {
  if (b < 1) return -1;
  if (s < 1 || s > b || b % s != 0) return -2;
  return 0;
}

/* ---------------------------------------------------------------------------
 * GEQRT / DGEQT2: A_kk <- V_kk, R_kk ; T_kk.
 * With inner blocking s (R5): for each block l of s
 * columns, an unblocked (rank-1 per column, R7) QR of the s columns, the T_l
 * column recurrence, then the level-3 update C -= U_l T_l^T U_l^T C of the
 * columns right of the block.  s == b is the paper's unblocked kernel.
 * ------------------------------------------------------------------------- */
int oracle_geqrt(int b, int s, double* A, double* T) {
  int rc = check_bs(b, s);
  if (rc) return rc;
  double* z = (double*)malloc(sizeof(double) * s);
  double* W = (double*)malloc(sizeof(double) * s);
  double* W2 = (double*)malloc(sizeof(double) * s);
#define Ak(r, c) A[(int64_t)(r) + (int64_t)(c) * b]
  for (int l = 0; l < b / s; ++l) {
    int c0 = l * s;
    double* Tl = T + (int64_t)l * s * s;
    for (int64_t e = 0; e < (int64_t)s * s; ++e) Tl[e] = 0.0;
    for (int c = c0; c < c0 + s; ++c) {
      double beta, tau;
      oracle_house(Ak(c, c), &Ak(c + 1, c), b - c - 1, &beta, &tau, &Ak(c + 1, c));
      Ak(c, c) = beta;
      for (int cp = c + 1; cp < c0 + s; ++cp) {
        double w = Ak(c, cp);
        for (int r = c + 1; r < b; ++r) w += Ak(r, c) * Ak(r, cp);
        Ak(c, cp) -= tau * w;
        for (int r = c + 1; r < b; ++r) Ak(r, cp) -= tau * w * Ak(r, c);
      }
      int j = c - c0;
      for (int t = 0; t < j; ++t) {
        /* z_t = u_{c0+t}^T u_c : u_c has 1 at row c, v below; u_{c0+t}[c] = A[c, c0+t]. */
        double acc = Ak(c, c0 + t);
        for (int r = c + 1; r < b; ++r) acc += Ak(r, c0 + t) * Ak(r, c);
        z[t] = acc;
      }
      larft_column(Tl, s, j, tau, z);
    }
    /* trailing columns t in [c0+s, b): W = U_l^T C; W <- T_l^T W; C -= U_l W. */
    for (int t = c0 + s; t < b; ++t) {
      for (int a = 0; a < s; ++a) {
        int ca = c0 + a;
        double acc = Ak(ca, t); /* unit diagonal of U_l */
        for (int r = ca + 1; r < b; ++r) acc += Ak(r, ca) * Ak(r, t);
        W[a] = acc;
      }
      apply_tl(Tl, s, W, W2, 1);
      for (int r = c0; r < b; ++r) {
        double acc = 0.0;
        for (int a = 0; a < s; ++a) {
          int ca = c0 + a;
          double u = (r == ca) ? 1.0 : (r > ca ? Ak(r, ca) : 0.0);
          acc += u * W2[a];
        }
        Ak(r, t) -= acc;
      }
    }
  }
#undef Ak
  free(z); free(W); free(W2);
  return 0;
}

/* ---------------------------------------------------------------------------
 * TSQRT / DTSQT2: QR of [R_kk; A_ik]; reflectors [I; V_ik].
 * `rows` rows in the lower block B (ld = rows): rows = b is the paper's square tile,
 * rows = h b its non-square 2b x b tiles (reading R30).
 * R = upper triangle (incl. diagonal) of the diagonal tile; the strict lower
 * part (V_kk) is never read or written.  SURVEY 8(c) c-4.
 * ------------------------------------------------------------------------- */
int oracle_tsqrt_rows(int b, int s, int rows, double* R, double* B, double* T) {
  int rc = check_bs(b, s);
  if (rc) return rc;
  if (rows < 1) return -3;
  double* z = (double*)malloc(sizeof(double) * s);
  double* W = (double*)malloc(sizeof(double) * s);
  double* W2 = (double*)malloc(sizeof(double) * s);
#define Rk(r, c) R[(int64_t)(r) + (int64_t)(c) * b]
#define Bk(r, c) B[(int64_t)(r) + (int64_t)(c) * rows]
  for (int l = 0; l < b / s; ++l) {
    int c0 = l * s;
    double* Tl = T + (int64_t)l * s * s;
    for (int64_t e = 0; e < (int64_t)s * s; ++e) Tl[e] = 0.0;
    for (int c = c0; c < c0 + s; ++c) {
      double beta, tau;
      oracle_house(Rk(c, c), &Bk(0, c), rows, &beta, &tau, &Bk(0, c));
      Rk(c, c) = beta;
      for (int cp = c + 1; cp < c0 + s; ++cp) {
        double w = Rk(c, cp);
        for (int r = 0; r < rows; ++r) w += Bk(r, c) * Bk(r, cp);
        Rk(c, cp) -= tau * w;
        for (int r = 0; r < rows; ++r) Bk(r, cp) -= tau * w * Bk(r, c);
      }
      int j = c - c0;
      for (int t = 0; t < j; ++t) {
        /* identity tops are orthogonal (e_{c0+t} . e_c = 0) */
        double acc = 0.0;
        for (int r = 0; r < rows; ++r) acc += Bk(r, c0 + t) * Bk(r, c);
        z[t] = acc;
      }
      larft_column(Tl, s, j, tau, z);
    }
    for (int t = c0 + s; t < b; ++t) {
      for (int a = 0; a < s; ++a) {
        double acc = Rk(c0 + a, t);
        for (int r = 0; r < rows; ++r) acc += Bk(r, c0 + a) * Bk(r, t);
        W[a] = acc;
      }
      apply_tl(Tl, s, W, W2, 1);
      for (int a = 0; a < s; ++a) Rk(c0 + a, t) -= W2[a];
      for (int r = 0; r < rows; ++r) {
        double acc = 0.0;
        for (int a = 0; a < s; ++a) acc += Bk(r, c0 + a) * W2[a];
        Bk(r, t) -= acc;
      }
    }
  }
#undef Rk
#undef Bk
  free(z); free(W); free(W2);
  return 0;
}

/* TSQRT of [R_kk; A_ik] with one b x b lower tile. */
int oracle_tsqrt(int b, int s, double* R, double* B, double* T) { return oracle_tsqrt_rows(b, s, b, R, B, T); }

/* ---------------------------------------------------------------------------
 * LARFB / DLARFB: A_kj <- Q_kk^T A_kj (trans=1, R1)
 * or Q_kk A_kj (trans=0).  Reads only the strict lower part of V (unit lower
 * U_l).
 * ------------------------------------------------------------------------- */
int oracle_larfb(int b, int s, const double* V, const double* T, double* C, int trans) {
  int rc = check_bs(b, s);
  if (rc) return rc;
  double* W = (double*)malloc(sizeof(double) * s);
  double* W2 = (double*)malloc(sizeof(double) * s);
  int nl = b / s;
  for (int li = 0; li < nl; ++li) {
    int l = trans ? li : nl - 1 - li;
    int c0 = l * s;
    const double* Tl = T + (int64_t)l * s * s;
    for (int t = 0; t < b; ++t) {
      double* Ct = C + (int64_t)t * b;
      for (int a = 0; a < s; ++a) {
        int ca = c0 + a;
        double acc = Ct[ca];
        for (int r = ca + 1; r < b; ++r) acc += V[r + (int64_t)ca * b] * Ct[r];
        W[a] = acc;
      }
      apply_tl(Tl, s, W, W2, trans);
      for (int r = c0; r < b; ++r) {
        double acc = 0.0;
        for (int a = 0; a < s; ++a) {
          int ca = c0 + a;
          double u = (r == ca) ? 1.0 : (r > ca ? V[r + (int64_t)ca * b] : 0.0);
          acc += u * W2[a];
        }
        Ct[r] -= acc;
      }
    }
  }
  free(W); free(W2);
  return 0;
}

/* ---------------------------------------------------------------------------
 * SSRFB / DSSRFB:
 * [A_kj; A_ij] <- (I - [I;V] T^T [I;V]^T) [A_kj; A_ij] per inner block l
 * (trans=1), or the Q form with T_l, l descending (trans=0).  SURVEY 8(c) c-6.
 * ------------------------------------------------------------------------- */
int oracle_ssrfb_rows(int b, int s, int rows, const double* V, const double* T, double* C1, double* C2, int trans) {
  int rc = check_bs(b, s);
  if (rc) return rc;
  if (rows < 1) return -3;
  double* W = (double*)malloc(sizeof(double) * s);
  double* W2 = (double*)malloc(sizeof(double) * s);
  int nl = b / s;
  for (int li = 0; li < nl; ++li) {
    int l = trans ? li : nl - 1 - li;
    int c0 = l * s;
    const double* Tl = T + (int64_t)l * s * s;
    for (int t = 0; t < b; ++t) {
      double* C1t = C1 + (int64_t)t * b;
      double* C2t = C2 + (int64_t)t * rows;
      for (int a = 0; a < s; ++a) {
        double acc = C1t[c0 + a];
        const double* Va = V + (int64_t)(c0 + a) * rows;
        for (int r = 0; r < rows; ++r) acc += Va[r] * C2t[r];
        W[a] = acc;
      }
      apply_tl(Tl, s, W, W2, trans);
      for (int a = 0; a < s; ++a) C1t[c0 + a] -= W2[a];
      for (int r = 0; r < rows; ++r) {
        double acc = 0.0;
        for (int a = 0; a < s; ++a) acc += V[r + (int64_t)(c0 + a) * rows] * W2[a];
        C2t[r] -= acc;
      }
    }
  }
  free(W); free(W2);
  return 0;
}

/* SSRFB with one b x b lower tile. */
int oracle_ssrfb(int b, int s, const double* V, const double* T, double* C1, double* C2, int trans) {
  return oracle_ssrfb_rows(b, s, b, V, T, C1, C2, trans);
}

/* ---------------------------------------------------------------------------
 * Block Data Layout with zero padding to tile multiples
 * (R9).
 * ------------------------------------------------------------------------- */
int oracle_pack(int64_t m, int64_t n, int b, const double* A, int64_t lda, double* At) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  if (b < 1) return -3;
  if (lda < m) return -5;
  int64_t p = (m + b - 1) / b, q = (n + b - 1) / b;
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = 0; i < p; ++i) {
      double* t = TILE(At, i, j, p, b);
      for (int64_t c = 0; c < b; ++c)
        for (int64_t r = 0; r < b; ++r) {
          int64_t gr = i * b + r, gc = j * b + c;
          t[r + c * b] = (gr < m && gc < n) ? A[gr + gc * lda] : 0.0;
        }
    }
  return 0;
}

int oracle_unpack(int64_t m, int64_t n, int b, const double* At, double* A, int64_t lda) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  if (b < 1) return -3;
  if (lda < m) return -5;
  int64_t p = (m + b - 1) / b;
  for (int64_t gc = 0; gc < n; ++gc)
    for (int64_t gr = 0; gr < m; ++gr)
      A[gr + gc * lda] = TILE(At, gr / b, gc / b, p, b)[(gr % b) + (gc % b) * b];
  return 0;
}

int oracle_get_r(int64_t m, int64_t n, int b, const double* At, double* R, int64_t ldr) {
  int64_t k = m < n ? m : n;
  if (ldr < k) return -5;
  int64_t p = (m + b - 1) / b;
  for (int64_t gc = 0; gc < n; ++gc)
    for (int64_t gr = 0; gr < k; ++gr)
      R[gr + gc * ldr] = (gr <= gc) ? TILE(At, gr / b, gc / b, p, b)[(gr % b) + (gc % b) * b] : 0.0;
  return 0;
}

/* ---------------------------------------------------------------------------
 * Algorithm 1, flat tree, 0-based:
 *   for k < min(p,q): GEQRT(k); LARFB(k,j) j>k; for i>k: TSQRT(k,i); SSRFB(k,i,j) j>k
 * ------------------------------------------------------------------------- */
enum { KG = 0, KT = 1, KL = 2, KS = 3 }; /* priority classes */

typedef struct {
  int64_t m, n, p, q;
  int b, s;
  double* At;
  double* T;
  int h;  /* tile rows per TSQRT/SSRFB unit (R30; 1 = the paper's square tiles) */
} qr_ctx;

static int64_t g_counts[4];

/* Units of step k (R30): the tile rows below the diagonal, k+1 .. p-1, in
 * consecutive groups of h starting at k+1 (the last group may be shorter).  Unit g covers
 * tile rows [unit_lo(k, g), unit_hi(k, g)); the tile row i lies in unit unit_of(k, i). */
static int64_t unit_lo(int64_t k, int64_t g, int h) { return k + 1 + (int64_t)h * g; }
static int64_t unit_hi(int64_t k, int64_t g, int h, int64_t p) {
  int64_t e = k + 1 + (int64_t)h * (g + 1);
  return e < p ? e : p;
}
static int64_t unit_of(int64_t k, int64_t i, int h) { return (i - k - 1) / h; }
static int64_t unit_count(int64_t k, int64_t p, int h) { return (p - k - 1 + h - 1) / h; }

/* The nt tiles (i0 .. i0+nt-1, j) stacked into a column-major (nt b) x b buffer, and back. */
static void gather(const qr_ctx* X, int64_t i0, int64_t nt, int64_t j, double* buf) {
  int b = X->b;
  for (int64_t t = 0; t < nt; ++t) {
    const double* tl = TILE(X->At, i0 + t, j, X->p, b);
    for (int64_t c = 0; c < b; ++c)
      for (int64_t r = 0; r < b; ++r) buf[t * b + r + c * nt * b] = tl[r + c * b];
  }
}
static void scatter(const qr_ctx* X, int64_t i0, int64_t nt, int64_t j, const double* buf) {
  int b = X->b;
  for (int64_t t = 0; t < nt; ++t) {
    double* tl = TILE(X->At, i0 + t, j, X->p, b);
    for (int64_t c = 0; c < b; ++c)
      for (int64_t r = 0; r < b; ++r) tl[r + c * b] = buf[t * b + r + c * nt * b];
  }
}

/* Task (kind, k, g, j); for T and S, g is the unit index (h = 1: the tile row k+1+g).  The T
 * factors of unit g live in the T slot of its first tile row. */
static void run_task(const qr_ctx* X, int kind, int64_t k, int64_t g, int64_t j) {
  int64_t p = X->p;
  int b = X->b, s = X->s;
  int64_t i0 = 0, nt = 0;
  if (kind == KT || kind == KS) {
    i0 = unit_lo(k, g, X->h);
    nt = unit_hi(k, g, X->h, p) - i0;
  }
  switch (kind) {
    case KG: oracle_geqrt(b, s, TILE(X->At, k, k, p, b), TSLOT(X->T, k, k, p, s, b)); break;
    case KL: oracle_larfb(b, s, TILE(X->At, k, k, p, b), TSLOT(X->T, k, k, p, s, b), TILE(X->At, k, j, p, b), 1); break;
    case KT:
      if (nt == 1) {
        oracle_tsqrt(b, s, TILE(X->At, k, k, p, b), TILE(X->At, i0, k, p, b), TSLOT(X->T, i0, k, p, s, b));
      } else {
        double* V = (double*)malloc(sizeof(double) * nt * b * b);
        gather(X, i0, nt, k, V);
        oracle_tsqrt_rows(b, s, (int)(nt * b), TILE(X->At, k, k, p, b), V, TSLOT(X->T, i0, k, p, s, b));
        scatter(X, i0, nt, k, V);
        free(V);
      }
      break;
    case KS:
      if (nt == 1) {
        oracle_ssrfb(b, s, TILE(X->At, i0, k, p, b), TSLOT(X->T, i0, k, p, s, b), TILE(X->At, k, j, p, b),
                     TILE(X->At, i0, j, p, b), 1);
      } else {
        double* V = (double*)malloc(sizeof(double) * nt * b * b);
        double* C2 = (double*)malloc(sizeof(double) * nt * b * b);
        gather(X, i0, nt, k, V);
        gather(X, i0, nt, j, C2);
        oracle_ssrfb_rows(b, s, (int)(nt * b), V, TSLOT(X->T, i0, k, p, s, b), TILE(X->At, k, j, p, b), C2, 1);
        scatter(X, i0, nt, j, C2);
        free(V);
        free(C2);
      }
      break;
  }
}

/* ---- DAG form: tasks, edges, 4-level priority ------------
 * Edges derived from each kernel's read/write sets (SPEC dag module):
 *   G(k)     <- S(k-1,k,k)
 *   L(k,j)   <- G(k), S(k-1,k,j)
 *   T(k,i)   <- G(k) if i == k+1 else T(k,i-1); S(k-1,i,k)
 *   S(k,i,j) <- T(k,i); L(k,j) if i == k+1 else S(k,i-1,j); S(k-1,i,j)
 * Priority G > T > L > S, ties by smaller k, then i, then j (R10).
 * With units of h tile rows (R30) the T/S tasks are indexed by unit g; a task of step k that
 * touches tile rows of step k-1's units depends on the LAST of those units (the step k-1
 * tasks of one column form a chain over the units).                              */
typedef struct {
  int kind;
  int64_t k, i, j;
  int npred;        /* remaining predecessors */
} dag_task;

typedef struct {
  qr_ctx X;
  dag_task* tasks;
  int64_t ntasks, ndone;
  int64_t* heap;
  int64_t heap_n;
  int64_t* idG; int64_t* idL; int64_t* idT; int64_t* idS;  /* index maps */
  int64_t* efrom; int64_t* eto; int64_t nedge;             /* edge list */
  int64_t* soff; int64_t* succ;                            /* CSR successors */
  pthread_mutex_t mu;
  pthread_cond_t cv;
} dag_ctx;

static int task_less(const dag_task* a, const dag_task* b) {
  if (a->kind != b->kind) return a->kind < b->kind;
  if (a->k != b->k) return a->k < b->k;
  if (a->i != b->i) return a->i < b->i;
  return a->j < b->j;
}
static void heap_push(dag_ctx* D, int64_t id) {
  int64_t x = D->heap_n++;
  D->heap[x] = id;
  while (x > 0) {
    int64_t par = (x - 1) / 2;
    if (!task_less(&D->tasks[D->heap[x]], &D->tasks[D->heap[par]])) break;
    int64_t t = D->heap[x]; D->heap[x] = D->heap[par]; D->heap[par] = t;
    x = par;
  }
}
static int64_t heap_pop(dag_ctx* D) {
  int64_t top = D->heap[0];
  D->heap[0] = D->heap[--D->heap_n];
  int64_t x = 0;
  for (;;) {
    int64_t l = 2 * x + 1, r = l + 1, m = x;
    if (l < D->heap_n && task_less(&D->tasks[D->heap[l]], &D->tasks[D->heap[m]])) m = l;
    if (r < D->heap_n && task_less(&D->tasks[D->heap[r]], &D->tasks[D->heap[m]])) m = r;
    if (m == x) break;
    int64_t t = D->heap[x]; D->heap[x] = D->heap[m]; D->heap[m] = t;
    x = m;
  }
  return top;
}

static void add_edge(dag_ctx* D, int64_t from, int64_t to) {
  D->efrom[D->nedge] = from;
  D->eto[D->nedge] = to;
  D->nedge++;
  D->tasks[to].npred++;
}

static void* dag_worker(void* arg) {
  dag_ctx* D = (dag_ctx*)arg;
  for (;;) {
    pthread_mutex_lock(&D->mu);
    while (D->heap_n == 0 && D->ndone < D->ntasks) pthread_cond_wait(&D->cv, &D->mu);
    if (D->heap_n == 0) { pthread_mutex_unlock(&D->mu); return NULL; }
    int64_t id = heap_pop(D);
    pthread_mutex_unlock(&D->mu);
    dag_task* t = &D->tasks[id];
    run_task(&D->X, t->kind, t->k, t->i, t->j);
    pthread_mutex_lock(&D->mu);
    g_counts[t->kind]++;
    D->ndone++;
    for (int64_t e = D->soff[id]; e < D->soff[id + 1]; ++e) {
      dag_task* u = &D->tasks[D->succ[e]];
      if (--u->npred == 0) heap_push(D, D->succ[e]);
    }
    pthread_cond_broadcast(&D->cv);
    pthread_mutex_unlock(&D->mu);
  }
}

/* Nodes in Algorithm 1's loop order and the edges of the comment above (the SPEC dag
 * module's rules).  Shared by the threaded executor and the oracle_dag_edges test hook. */
static void dag_build(dag_ctx* D, int64_t p, int64_t q, int h) {
  int64_t K = p < q ? p : q;
  int64_t nt = 0;
  for (int64_t k = 0; k < K; ++k) {
    const int64_t ng = unit_count(k, p, h);
    nt += 1 + (q - k - 1) + ng + ng * (q - k - 1);
  }
  D->ntasks = nt;
  D->tasks = (dag_task*)calloc(nt, sizeof(dag_task));
  D->heap = (int64_t*)malloc(sizeof(int64_t) * nt);
  D->idG = (int64_t*)malloc(sizeof(int64_t) * K);
  D->idL = (int64_t*)malloc(sizeof(int64_t) * K * q);
  D->idT = (int64_t*)malloc(sizeof(int64_t) * K * p);
  D->idS = (int64_t*)malloc(sizeof(int64_t) * K * p * q);
  D->efrom = (int64_t*)malloc(sizeof(int64_t) * 3 * nt);
  D->eto = (int64_t*)malloc(sizeof(int64_t) * 3 * nt);
#define IDL(k, j) D->idL[(k) * q + (j)]
#define IDT(k, g) D->idT[(k) * p + (g)]
#define IDS(k, g, j) D->idS[((k) * p + (g)) * q + (j)]
  int64_t id = 0;
  for (int64_t k = 0; k < K; ++k) {
    D->tasks[id] = (dag_task){KG, k, k, k, 0}; D->idG[k] = id++;
    for (int64_t j = k + 1; j < q; ++j) { D->tasks[id] = (dag_task){KL, k, k, j, 0}; IDL(k, j) = id++; }
    for (int64_t g = 0; g < unit_count(k, p, h); ++g) {
      D->tasks[id] = (dag_task){KT, k, g, k, 0}; IDT(k, g) = id++;
      for (int64_t j = k + 1; j < q; ++j) { D->tasks[id] = (dag_task){KS, k, g, j, 0}; IDS(k, g, j) = id++; }
    }
  }
  for (int64_t k = 0; k < K; ++k) {
    if (k > 0) add_edge(D, IDS(k - 1, unit_of(k - 1, k, h), k), D->idG[k]);
    for (int64_t j = k + 1; j < q; ++j) {
      add_edge(D, D->idG[k], IDL(k, j));
      if (k > 0) add_edge(D, IDS(k - 1, unit_of(k - 1, k, h), j), IDL(k, j));
    }
    for (int64_t g = 0; g < unit_count(k, p, h); ++g) {
      const int64_t gp = k > 0 ? unit_of(k - 1, unit_hi(k, g, h, p) - 1, h) : 0;  /* last unit of step k-1 */
      add_edge(D, g == 0 ? D->idG[k] : IDT(k, g - 1), IDT(k, g));
      if (k > 0) add_edge(D, IDS(k - 1, gp, k), IDT(k, g));
      for (int64_t j = k + 1; j < q; ++j) {
        add_edge(D, IDT(k, g), IDS(k, g, j));
        add_edge(D, g == 0 ? IDL(k, j) : IDS(k, g - 1, j), IDS(k, g, j));
        if (k > 0) add_edge(D, IDS(k - 1, gp, j), IDS(k, g, j));
      }
    }
  }
#undef IDL
#undef IDT
#undef IDS
}

static void dag_free(dag_ctx* D) {
  free(D->tasks); free(D->heap); free(D->idG); free(D->idL); free(D->idT); free(D->idS);
  free(D->efrom); free(D->eto); free(D->soff); free(D->succ);
}

/* Test hook: the DAG's edges for a p x q tile grid, 8 int64 per edge {kind, k, i, j} of the
 * predecessor then of the successor (kind 0 G, 1 T, 2 L, 3 S; T(k,i) has j = k, G and L
 * have i = k); returns the edge count, writes min(cap, count) edges. */
int64_t oracle_dag_edges_h(int64_t p, int64_t q, int h, int64_t* out, int64_t cap) {
  if (p < 1 || q < 1 || h < 1) return -1;
  dag_ctx D;
  memset(&D, 0, sizeof(D));
  dag_build(&D, p, q, h);
  for (int64_t e = 0; e < D.nedge && e < cap; ++e) {
    const dag_task* a = &D.tasks[D.efrom[e]];
    const dag_task* b = &D.tasks[D.eto[e]];
    int64_t* o = out + 8 * e;
    /* T / S tasks report the FIRST tile row of their unit */
    o[0] = a->kind; o[1] = a->k; o[2] = (a->kind == KT || a->kind == KS) ? unit_lo(a->k, a->i, h) : a->i; o[3] = a->j;
    o[4] = b->kind; o[5] = b->k; o[6] = (b->kind == KT || b->kind == KS) ? unit_lo(b->k, b->i, h) : b->i; o[7] = b->j;
  }
  int64_t n = D.nedge;
  dag_free(&D);
  return n;
}
int64_t oracle_dag_edges(int64_t p, int64_t q, int64_t* out, int64_t cap) { return oracle_dag_edges_h(p, q, 1, out, cap); }

static int geqrf_dag(const qr_ctx* X, int nthreads) {
  dag_ctx D;
  memset(&D, 0, sizeof(D));
  D.X = *X;
  dag_build(&D, X->p, X->q, X->h);
  const int64_t nt = D.ntasks;
  D.soff = (int64_t*)calloc(nt + 1, sizeof(int64_t));
  D.succ = (int64_t*)malloc(sizeof(int64_t) * (D.nedge + 1));
  for (int64_t e = 0; e < D.nedge; ++e) D.soff[D.efrom[e] + 1]++;
  for (int64_t t = 0; t < nt; ++t) D.soff[t + 1] += D.soff[t];
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (nt + 1));
    memcpy(fill, D.soff, sizeof(int64_t) * (nt + 1));
    for (int64_t e = 0; e < D.nedge; ++e) D.succ[fill[D.efrom[e]]++] = D.eto[e];
    free(fill);
  }
  for (int64_t t = 0; t < nt; ++t)
    if (D.tasks[t].npred == 0) heap_push(&D, t);
  pthread_mutex_init(&D.mu, NULL);
  pthread_cond_init(&D.cv, NULL);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  for (int w = 0; w < nthreads; ++w) pthread_create(&th[w], NULL, dag_worker, &D);
  for (int w = 0; w < nthreads; ++w) pthread_join(th[w], NULL);
  pthread_mutex_destroy(&D.mu);
  pthread_cond_destroy(&D.cv);
  int ok = (D.ndone == nt);
  free(th);
  dag_free(&D);
  return ok ? 0 : -99;
}

int oracle_geqrf_tiles_h(int64_t m, int64_t n, int b, int s, int h, double* At, double* T, int nthreads) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  int rc = check_bs(b, s);
  if (rc) return rc - 2;
  if (h < 1) return -5;
  if (nthreads < 1) return -8;
  qr_ctx X = {m, n, (m + b - 1) / b, (n + b - 1) / b, b, s, At, T, h};
  int64_t p = X.p, q = X.q, K = p < q ? p : q;
  memset(g_counts, 0, sizeof(g_counts));
  for (int64_t e = 0; e < p * q * (int64_t)s * b; ++e) T[e] = 0.0;
  if (nthreads > 1) return geqrf_dag(&X, nthreads);
  for (int64_t k = 0; k < K; ++k) {
    run_task(&X, KG, k, k, k); g_counts[KG]++;
    for (int64_t j = k + 1; j < q; ++j) { run_task(&X, KL, k, k, j); g_counts[KL]++; }
    for (int64_t g = 0; g < unit_count(k, p, h); ++g) {
      run_task(&X, KT, k, g, k); g_counts[KT]++;
      for (int64_t j = k + 1; j < q; ++j) { run_task(&X, KS, k, g, j); g_counts[KS]++; }
    }
  }
  return 0;
}

int oracle_geqrf_tiles(int64_t m, int64_t n, int b, int s, double* At, double* T, int nthreads) {
  int rc = oracle_geqrf_tiles_h(m, n, b, s, 1, At, T, nthreads);
  return rc <= -5 ? rc + 1 : rc;  /* (argument numbering of the h-less signature) */
}

void oracle_last_task_counts(int64_t counts[4]) {
  counts[0] = g_counts[KG]; counts[1] = g_counts[KL]; counts[2] = g_counts[KT]; counts[3] = g_counts[KS];
}

/* ---------------------------------------------------------------------------
 * Apply Q^T / Q to a tile-major B (R8).
 * Q = product of all reflectors in creation order (GEQRT(k), TSQRT(k,k+1..p-1),
 * k ascending).  Q^T B replays the factorization's LARFB/SSRFB on B's tiles;
 * Q B runs the reverse order with T_l un-transposed.  Tile columns of B are
 * independent, so nthreads > 1 splits them across threads.
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t m, n, p, q, qb, j0, j1;
  int b, s, trans, h;
  const double* At; const double* T; double* Bt;
} orm_ctx;

/* SSRFB-type application of unit g of step k (R30) to tile column j of B. */
static void orm_unit(const orm_ctx* X, int64_t k, int64_t g, int64_t j, int trans) {
  int64_t p = X->p;
  int b = X->b, s = X->s;
  const int64_t i0 = unit_lo(k, g, X->h), nt = unit_hi(k, g, X->h, p) - i0;
  if (nt == 1) {
    oracle_ssrfb(b, s, TILE(X->At, i0, k, p, b), TSLOT(X->T, i0, k, p, s, b), TILE(X->Bt, k, j, p, b),
                 TILE(X->Bt, i0, j, p, b), trans);
    return;
  }
  double* V = (double*)calloc(nt * b * b, sizeof(double));
  double* C2 = (double*)calloc(nt * b * b, sizeof(double));
  for (int64_t t = 0; t < nt; ++t)
    for (int64_t c = 0; c < b; ++c)
      for (int64_t r = 0; r < b; ++r) {
        V[t * b + r + c * nt * b] = TILE(X->At, i0 + t, k, p, b)[r + c * b];
        C2[t * b + r + c * nt * b] = TILE(X->Bt, i0 + t, j, p, b)[r + c * b];
      }
  oracle_ssrfb_rows(b, s, (int)(nt * b), V, TSLOT(X->T, i0, k, p, s, b), TILE(X->Bt, k, j, p, b), C2, trans);
  for (int64_t t = 0; t < nt; ++t)
    for (int64_t c = 0; c < b; ++c)
      for (int64_t r = 0; r < b; ++r) TILE(X->Bt, i0 + t, j, p, b)[r + c * b] = C2[t * b + r + c * nt * b];
  free(V);
  free(C2);
}

static void orm_columns(const orm_ctx* X) {
  int64_t p = X->p, K = X->p < X->q ? X->p : X->q;
  int b = X->b, s = X->s;
  for (int64_t j = X->j0; j < X->j1; ++j) {
    if (X->trans) {
      for (int64_t k = 0; k < K; ++k) {
        oracle_larfb(b, s, TILE(X->At, k, k, p, b), TSLOT(X->T, k, k, p, s, b), TILE(X->Bt, k, j, p, b), 1);
        for (int64_t g = 0; g < unit_count(k, p, X->h); ++g) orm_unit(X, k, g, j, 1);
      }
    } else {
      for (int64_t k = K - 1; k >= 0; --k) {
        for (int64_t g = unit_count(k, p, X->h) - 1; g >= 0; --g) orm_unit(X, k, g, j, 0);
        oracle_larfb(b, s, TILE(X->At, k, k, p, b), TSLOT(X->T, k, k, p, s, b), TILE(X->Bt, k, j, p, b), 0);
      }
    }
  }
}
static void* orm_worker(void* a) { orm_columns((const orm_ctx*)a); return NULL; }

int oracle_ormqr_tiles_h(int64_t m, int64_t n, int b, int s, int h, const double* At, const double* T,
                         int trans, int64_t nrhs, double* Bt, int nthreads) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  int rc = check_bs(b, s);
  if (rc) return rc - 2;
  if (h < 1) return -5;
  if (trans != 0 && trans != 1) return -8;
  if (nrhs < 1) return -9;
  if (nthreads < 1) return -11;
  int64_t p = (m + b - 1) / b, q = (n + b - 1) / b, qb = (nrhs + b - 1) / b;
  if (nthreads > qb) nthreads = (int)qb;
  orm_ctx* X = (orm_ctx*)malloc(sizeof(orm_ctx) * nthreads);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  for (int w = 0; w < nthreads; ++w) {
    X[w] = (orm_ctx){m, n, p, q, qb, qb * w / nthreads, qb * (w + 1) / nthreads, b, s, trans, h, At, T, Bt};
    if (nthreads == 1) orm_columns(&X[w]);
    else pthread_create(&th[w], NULL, orm_worker, &X[w]);
  }
  if (nthreads > 1)
    for (int w = 0; w < nthreads; ++w) pthread_join(th[w], NULL);
  free(X); free(th);
  return 0;
}

int oracle_ormqr_tiles(int64_t m, int64_t n, int b, int s, const double* At, const double* T,
                       int trans, int64_t nrhs, double* Bt, int nthreads) {
  int rc = oracle_ormqr_tiles_h(m, n, b, s, 1, At, T, trans, nrhs, Bt, nthreads);
  return rc <= -5 ? rc + 1 : rc;
}

/* ---------------------------------------------------------------------------
 * Flop models.
 * ------------------------------------------------------------------------- */
double oracle_flops_standard(int64_t m, int64_t n) {
  /* QR requires 2n^2(m - n/3) (m >= n); by symmetry
   * 2m^2(n - m/3) when m < n. */
  double M = (double)m, N = (double)n;
  if (m >= n) return 2.0 * N * N * (M - N / 3.0);
  return 2.0 * M * M * (N - M / 3.0);
}

double oracle_kernel_flops(int kind, double b) {
  double b3 = b * b * b;
  switch (kind) {
    case 0: return 2.0 * b3;          /* DGEQT2 */
    case 1: return 3.0 * b3;          /* DLARFB */
    case 2: return 10.0 / 3.0 * b3;   /* DTSQT2 */
    case 3: return 5.0 * b3;          /* DSSRFB */
  }
  return -1.0;
}

/* Eq. (4) with units of h tile rows (R30), s = b: per unit of nt tiles TSQRT (3 nt + 1/3) b^3
 * (h = 1: 10/3 b^3) and SSRFB (4 nt + 1) b^3 (h = 1: 5 b^3). */
double oracle_flops_eq4_h(int64_t p, int64_t q, double b, int h) {
  double tot = 0.0, b3 = b * b * b;
  int64_t K = p < q ? p : q;
  for (int64_t k = 0; k < K; ++k) {
    tot += 2.0 * b3 + (double)(q - k - 1) * 3.0 * b3;
    for (int64_t g = 0; g < unit_count(k, p, h); ++g) {
      const double nt = (double)(unit_hi(k, g, h, p) - unit_lo(k, g, h));
      tot += (3.0 * nt + 1.0 / 3.0) * b3 + (double)(q - k - 1) * (4.0 * nt + 1.0) * b3;
    }
  }
  return tot;
}

double oracle_flops_eq4(int64_t p, int64_t q, double b) {
  /* Eq. (4), exact sum over k = 1..min(p,q). */
  double tot = 0.0;
  int64_t K = p < q ? p : q;
  for (int64_t k = 1; k <= K; ++k)
    tot += oracle_kernel_flops(0, b) + (double)(q - k) * oracle_kernel_flops(1, b) +
           (double)(p - k) * oracle_kernel_flops(2, b) + (double)(p - k) * (double)(q - k) * oracle_kernel_flops(3, b);
  return tot;
}
