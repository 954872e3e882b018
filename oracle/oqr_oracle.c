/*
 * oqr_oracle.c -- CPU FP64 ORACLE for the oblique-QR normal-equation hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_1401_5171_b200/) never imports, links or executes it; the two share no code.
 *
 * Plain, slow, obviously-correct FP64 implementations written from the paper:
 *   Lowery & Langou, "Stability Analysis of QR factorization in an Oblique Inner Product"
 *   (/root/reference/PAPER.md).  Citations are PAPER.md line numbers.
 *
 * Arithmetic rules: IEEE binary64, round-to-nearest, no FMA contraction
 * (-ffp-contract=off), no -ffast-math.  Every sum runs in ascending index order
 * as written; OpenMP only splits DISJOINT outputs across threads, so results are
 * independent of the thread count.
 *
 * Storage: column-major; element (i,j) of a matrix with leading dimension ld is p[j*ld+i].
 *
 * Pins (tests/test_oracle_pins.py): Theorem 1, the normal equation
 * Z^T A Z = R^T R, A = I reducing to Euclidean QR
 * (PAPER.md:82-83), brute force with an explicit A^{1/2} on tiny inputs,
 * exact rational arithmetic on tiny inputs, and the paper's s7 closed forms
 * (PAPER.md:693-742).  Nothing here is "parity unpinned" except the breakdown INDEX on
 * near-singular G.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* Algorithm 1 (CHOLQR) step 1-2:  B = A Z;  C = Z^T B.      */
/* B[i,l] = sum_{j=0}^{m-1} A[i,j] Z[j,l]   (j ascending)                      */
/* G[k,l] = sum_{i=0}^{m-1} Z[i,k] B[i,l]   (i ascending)                      */
/* ------------------------------------------------------------------------- */
void orc_gram(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
              double* G, int64_t ldg) {
  double* B = (double*)malloc(sizeof(double) * m * n);
  double* Zt = (double*)malloc(sizeof(double) * m * n); /* row-major copy: Zt[j*n+l] = Z[j,l] */
  for (int64_t l = 0; l < n; l++)
    for (int64_t j = 0; j < m; j++) Zt[j * n + l] = Z[l * ldz + j];
  const int64_t RB = 64;
  const int64_t nblk = (m + RB - 1) / RB;
#pragma omp parallel for schedule(static)
  for (int64_t ib = 0; ib < nblk; ib++) {
    int64_t i0 = ib * RB, i1 = i0 + RB < m ? i0 + RB : m;
    for (int64_t l = 0; l < n; l++)
      for (int64_t i = i0; i < i1; i++) B[l * m + i] = 0.0;
    for (int64_t j = 0; j < m; j++) {
      const double* acol = A + j * lda;
      const double* zrow = Zt + j * n;
      for (int64_t l = 0; l < n; l++) {
        const double z = zrow[l];
        double* b = B + l * m;
        for (int64_t i = i0; i < i1; i++) b[i] += acol[i] * z; /* B[i,l] += A[i,j]*Z[j,l] */
      }
    }
  }
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t l = 0; l < n; l++)
    for (int64_t k = 0; k < n; k++) {
      const double* zk = Z + k * ldz;
      const double* bl = B + l * m;
      double s = 0.0;
      for (int64_t i = 0; i < m; i++) s += zk[i] * bl[i];
      G[l * ldg + k] = s;
    }
  free(B);
  free(Zt);
}

/* Euclidean Gram (the pre-QR step of PRE-CHOLQR done as Cholesky-QR, north_star;
 * PAPER.md:321 with the DESIGN.md reading R2):  G[k,l] = sum_i Z[i,k] Z[i,l]. */
void orc_gram_euclid(int64_t m, int64_t n, const double* Z, int64_t ldz, double* G, int64_t ldg) {
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t l = 0; l < n; l++)
    for (int64_t k = 0; k < n; k++) {
      const double* zk = Z + k * ldz;
      const double* zl = Z + l * ldz;
      double s = 0.0;
      for (int64_t i = 0; i < m; i++) s += zk[i] * zl[i];
      G[l * ldg + k] = s;
    }
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1 step 3, PAPER.md:182 (R = chol(C), upper, R^T R = C).           */
/* Unblocked, reads only the upper triangle of G (readings R4, R5):  */
/*   for j: d = G[j,j] - sum_{k<j} R[k,j]^2;  if !(d > 0) return j+1;          */
/*          R[j,j] = sqrt(d);                                                  */
/*          R[j,l] = (G[j,l] - sum_{k<j} R[k,j] R[k,l]) / R[j,j],  l > j.      */
/* Strictly lower part of R is set to zero.  Returns 0 or the 1-based pivot.   */
/* ------------------------------------------------------------------------- */
int orc_potrf(int64_t n, const double* G, int64_t ldg, double* R, int64_t ldr) {
  for (int64_t l = 0; l < n; l++)
    for (int64_t k = 0; k < n; k++) R[l * ldr + k] = 0.0;
  for (int64_t j = 0; j < n; j++) {
    double dot = 0.0;
    for (int64_t k = 0; k < j; k++) dot += R[j * ldr + k] * R[j * ldr + k];
    double d = G[j * ldg + j] - dot;
    if (!(d > 0.0)) return (int)(j + 1);
    double rjj = sqrt(d);
    R[j * ldr + j] = rjj;
    for (int64_t l = j + 1; l < n; l++) {
      double s = 0.0;
      for (int64_t k = 0; k < j; k++) s += R[j * ldr + k] * R[l * ldr + k];
      R[l * ldr + j] = (G[l * ldg + j] - s) / rjj;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1 step 4, PAPER.md:183 (Q = Z / R), row-wise substitution as in   */
/* the backward-error statement PAPER.md:197-198:                              */
/*   q_ij = (z_ij - sum_{k<j} q_ik r_kj) / r_jj.                               */
/* Q may alias Z (rows are independent; each row is read before it is written) */
/* ------------------------------------------------------------------------- */
void orc_trsm(int64_t m, int64_t n, const double* Z, int64_t ldz, const double* R, int64_t ldr,
              double* Q, int64_t ldq) {
#pragma omp parallel
  {
    double* q = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
#pragma omp for schedule(static)
    for (int64_t i = 0; i < m; i++) {
      for (int64_t j = 0; j < n; j++) {
        double s = 0.0;
        for (int64_t k = 0; k < j; k++) s += q[k] * R[j * ldr + k];
        q[j] = (Z[j * ldz + i] - s) / R[j * ldr + j];
      }
      for (int64_t j = 0; j < n; j++) Q[j * ldq + i] = q[j];
    }
    free(q);
  }
}

/* R = R2 * R1 for upper-triangular n x n ("R = US"; normal2: R = R2 R1).
 * R[i,j] = sum_{k=i}^{j} R2[i,k] R1[k,j], k ascending; lower part zero. */
void orc_trmm(int64_t n, const double* R2, int64_t ld2, const double* R1, int64_t ld1, double* R, int64_t ldr) {
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < n; i++) {
      double s = 0.0;
      if (i <= j)
        for (int64_t k = i; k <= j; k++) s += R2[k * ld2 + i] * R1[j * ld1 + k];
      R[j * ldr + i] = s;
    }
}

/* ------------------------------------------------------------------------- */
/* The three variants.  Q: m x n (ld m), R: n x n (ld n).                      */
/* Status: 0 ok; k in 1..n breakdown of the first Cholesky; n+k of the second. */
/* ------------------------------------------------------------------------- */

/* Algorithm 1, CHOLQR. */
int orc_normal(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
               double* Q, double* R) {
  double* G = (double*)malloc(sizeof(double) * n * n);
  orc_gram(m, n, A, lda, Z, ldz, G, n);
  int info = orc_potrf(n, G, n, R, n);
  free(G);
  if (info) return info;
  orc_trsm(m, n, Z, ldz, R, n, Q, m);
  return 0;
}

/* Repeated CHOLQR (north_star; reading R1): two full passes, R = R2 R1. */
int orc_normal2(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                double* Q, double* R) {
  double* R1 = (double*)malloc(sizeof(double) * n * n);
  double* R2 = (double*)malloc(sizeof(double) * n * n);
  double* Q1 = (double*)malloc(sizeof(double) * m * n);
  int info = orc_normal(m, n, A, lda, Z, ldz, Q1, R1);
  if (!info) {
    int info2 = orc_normal(m, n, A, lda, Q1, m, Q, R2);
    if (info2) info = (int)n + info2;
    else orc_trmm(n, R2, n, R1, n, R, n);
  }
  free(R1); free(R2); free(Q1);
  return info;
}

/* Algorithm 2, PRE-CHOLQR with the Euclidean pre-step done by
 * Cholesky-QR (north_star; reading R2): [Y,S] = cholqr_I(Z);
 * [Q,U] = CHOLQR(A,Y); R = U S. */
int orc_prequr(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
               double* Q, double* R) {
  double* G = (double*)malloc(sizeof(double) * n * n);
  double* S = (double*)malloc(sizeof(double) * n * n);
  double* U = (double*)malloc(sizeof(double) * n * n);
  double* Y = (double*)malloc(sizeof(double) * m * n);
  orc_gram_euclid(m, n, Z, ldz, G, n);
  int info = orc_potrf(n, G, n, S, n);
  if (!info) {
    orc_trsm(m, n, Z, ldz, S, n, Y, m);
    int info2 = orc_normal(m, n, A, lda, Y, m, Q, U);
    if (info2) info = (int)n + info2;
    else orc_trmm(n, U, n, S, n, R, n);
  }
  free(G); free(S); free(U); free(Y);
  return info;
}

/* ------------------------------------------------------------------------- */
/* Checkers (double-double; TwoSum / TwoProd with an explicit fma()).          */
/* Needed because for the stable variants the measured error is the size of   */
/* the FP64 error of forming the check itself.            */
/* ------------------------------------------------------------------------- */
typedef struct { double hi, lo; } dd_t;

static inline dd_t two_sum(double a, double b) {
  double s = a + b, bb = s - a;
  dd_t r = {s, (a - (s - bb)) + (b - bb)};
  return r;
}
static inline dd_t dd_add_prod(dd_t acc, double a, double b) {
  double p = a * b, pe = fma(a, b, -p);      /* exact product p + pe */
  dd_t s = two_sum(acc.hi, p);
  double lo = s.lo + acc.lo + pe;
  dd_t r = two_sum(s.hi, lo);
  return r;
}
static inline dd_t dd_add_dd_prod(dd_t acc, double a, dd_t b) {
  /* acc + a*(b.hi + b.lo) */
  acc = dd_add_prod(acc, a, b.hi);
  double t = a * b.lo;
  dd_t s = two_sum(acc.hi, t);
  return two_sum(s.hi, s.lo + acc.lo);
}

/* E = Q^T A Q - I (n x n, ld n) accumulated in double-double, rounded at the end. */
void orc_dd_orth(int64_t m, int64_t n, const double* A, int64_t lda, const double* Q, int64_t ldq,
                 double* E) {
  dd_t* AQ = (dd_t*)malloc(sizeof(dd_t) * m * n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++) {
    for (int64_t l = 0; l < n; l++) {
      dd_t s = {0.0, 0.0};
      for (int64_t j = 0; j < m; j++) s = dd_add_prod(s, A[j * lda + i], Q[l * ldq + j]);
      AQ[l * m + i] = s;
    }
  }
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t l = 0; l < n; l++)
    for (int64_t k = 0; k < n; k++) {
      dd_t s = {k == l ? -1.0 : 0.0, 0.0};
      for (int64_t i = 0; i < m; i++) s = dd_add_dd_prod(s, Q[k * ldq + i], AQ[l * m + i]);
      E[l * n + k] = s.hi + s.lo;
    }
  free(AQ);
}

/* G = Z^T A Z in double-double (rounded) and M = |Z|^T |A| |Z| in FP64 (for the
 * eq.mult1-2 componentwise tolerance). */
void orc_dd_gram(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                 double* G, double* M) {
  dd_t* B = (dd_t*)malloc(sizeof(dd_t) * m * n);
  double* Babs = (double*)malloc(sizeof(double) * m * n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++) {
    for (int64_t l = 0; l < n; l++) {
      dd_t s = {0.0, 0.0};
      double sa = 0.0;
      for (int64_t j = 0; j < m; j++) {
        double a = A[j * lda + i], z = Z[l * ldz + j];
        s = dd_add_prod(s, a, z);
        sa += fabs(a) * fabs(z);
      }
      B[l * m + i] = s;
      Babs[l * m + i] = sa;
    }
  }
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t l = 0; l < n; l++)
    for (int64_t k = 0; k < n; k++) {
      dd_t s = {0.0, 0.0};
      double sa = 0.0;
      for (int64_t i = 0; i < m; i++) {
        s = dd_add_dd_prod(s, Z[k * ldz + i], B[l * m + i]);
        sa += fabs(Z[k * ldz + i]) * Babs[l * m + i];
      }
      G[l * n + k] = s.hi + s.lo;
      M[l * n + k] = sa;
    }
  free(B);
  free(Babs);
}

/* D = Z - Q R (double-double, rounded) and QR_abs = |Q| |R| (FP64), both m x n (ld m).
 * Inputs for the Theorem 2 representativity checks. */
void orc_dd_resid(int64_t m, int64_t n, const double* Z, int64_t ldz, const double* Q, int64_t ldq,
                  const double* R, int64_t ldr, double* D, double* QRabs) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++) {
    for (int64_t j = 0; j < n; j++) {
      dd_t s = {Z[j * ldz + i], 0.0};
      double sa = 0.0;
      for (int64_t k = 0; k <= j; k++) {
        double q = Q[k * ldq + i], r = R[j * ldr + k];
        s = dd_add_prod(s, -q, r);
        sa += fabs(q) * fabs(r);
      }
      D[j * m + i] = s.hi + s.lo;
      QRabs[j * m + i] = sa;
    }
  }
}

/* |G - R^T R| and |R|^T |R| over the upper triangle (Cholesky backward error,
 * eq:normal:chol PAPER.md:195-196), double-double. Outputs n x n (ld n). */
void orc_dd_chol_resid(int64_t n, const double* G, int64_t ldg, const double* R, int64_t ldr,
                       double* D, double* RRabs) {
  for (int64_t l = 0; l < n; l++)
    for (int64_t k = 0; k < n; k++) {
      dd_t s = {G[l * ldg + k], 0.0};
      double sa = 0.0;
      int64_t kmax = k < l ? k : l;
      for (int64_t p = 0; p <= kmax; p++) {
        double a = R[k * ldr + p], b = R[l * ldr + p];
        s = dd_add_prod(s, -a, b);
        sa += fabs(a) * fabs(b);
      }
      D[l * n + k] = s.hi + s.lo;
      RRabs[l * n + k] = sa;
    }
}

/* E_S = Q_S^T A Q_S - I for the column subset S (ns columns, indices cols[]), n_s x n_s (ld ns),
 * double-double.  Identical per-entry arithmetic to orc_dd_orth (AQ[i,l] accumulated over j
 * ascending, then E[k,l] over i ascending); only the loop order over (i, j) is interchanged so
 * that column-major A is streamed once (rows i are split across threads).  Used for sampled
 * orthogonality checks at the full BASELINE sizes. */
void orc_dd_orth_cols(int64_t m, int64_t ns, const int64_t* cols, const double* A, int64_t lda,
                      const double* Q, int64_t ldq, double* E) {
  dd_t* AQ = (dd_t*)malloc(sizeof(dd_t) * m * ns);
#pragma omp parallel
  {
    int nt = 1, t = 0;
#ifdef _OPENMP
    nt = omp_get_num_threads();
    t = omp_get_thread_num();
#endif
    int64_t i0 = m * t / nt, i1 = m * (t + 1) / nt;
    for (int64_t l = 0; l < ns; l++)
      for (int64_t i = i0; i < i1; i++) { AQ[l * m + i].hi = 0.0; AQ[l * m + i].lo = 0.0; }
    for (int64_t j = 0; j < m; j++) {
      const double* acol = A + j * lda;
      for (int64_t l = 0; l < ns; l++) {
        const double q = Q[cols[l] * ldq + j];
        dd_t* aq = AQ + l * m;
        for (int64_t i = i0; i < i1; i++) aq[i] = dd_add_prod(aq[i], acol[i], q);
      }
    }
  }
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t l = 0; l < ns; l++)
    for (int64_t k = 0; k < ns; k++) {
      dd_t s = {k == l ? -1.0 : 0.0, 0.0};
      const double* qk = Q + cols[k] * ldq;
      for (int64_t i = 0; i < m; i++) s = dd_add_dd_prod(s, qk[i], AQ[l * m + i]);
      E[l * ns + k] = s.hi + s.lo;
    }
  free(AQ);
}

/* ========================================================================= */
/* NEXT-N3: symmetric tridiagonal A = tridiag(e, d, e). */
/* B = A Z by the 3-point definition, terms in ascending column order j = i-1, i, */
/* i+1 starting from 0.0 -- the same operations as orc_gram on the densified A   */
/* (whose other terms add exact zeros), so the two agree bitwise (pinned).       */
/* ========================================================================= */
void orc_gram_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Z, int64_t ldz,
                      double* G, int64_t ldg) {
  double* B = (double*)malloc(sizeof(double) * m * n);
#pragma omp parallel for schedule(static)
  for (int64_t l = 0; l < n; l++) {
    const double* z = Z + l * ldz;
    for (int64_t i = 0; i < m; i++) {
      double b = 0.0;
      if (i > 0) b += e[i - 1] * z[i - 1];
      b += d[i] * z[i];
      if (i < m - 1) b += e[i] * z[i + 1];
      B[l * m + i] = b;
    }
  }
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t l = 0; l < n; l++)
    for (int64_t k = 0; k < n; k++) {
      const double* zk = Z + k * ldz;
      const double* bl = B + l * m;
      double s = 0.0;
      for (int64_t i = 0; i < m; i++) s += zk[i] * bl[i];
      G[l * ldg + k] = s;
    }
  free(B);
}

/* Algorithm 1 with the tridiagonal Gram. */
int orc_normal_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Z, int64_t ldz,
                       double* Q, double* R) {
  double* G = (double*)malloc(sizeof(double) * n * n);
  orc_gram_tridiag(m, n, d, e, Z, ldz, G, n);
  int info = orc_potrf(n, G, n, R, n);
  free(G);
  if (info) return info;
  orc_trsm(m, n, Z, ldz, R, n, Q, m);
  return 0;
}

/* Repeated CHOLQR (reading R1) with the tridiagonal Gram. */
int orc_normal2_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Z, int64_t ldz,
                        double* Q, double* R) {
  double* R1 = (double*)malloc(sizeof(double) * n * n);
  double* R2 = (double*)malloc(sizeof(double) * n * n);
  double* Q1 = (double*)malloc(sizeof(double) * m * n);
  int info = orc_normal_tridiag(m, n, d, e, Z, ldz, Q1, R1);
  if (!info) {
    int info2 = orc_normal_tridiag(m, n, d, e, Q1, m, Q, R2);
    if (info2) info = (int)n + info2;
    else orc_trmm(n, R2, n, R1, n, R, n);
  }
  free(R1); free(R2); free(Q1);
  return info;
}

/* PRE-CHOLQR (Algorithm 2, reading R2) with the tridiagonal A-stage. */
int orc_prequr_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Z, int64_t ldz,
                       double* Q, double* R) {
  double* G = (double*)malloc(sizeof(double) * n * n);
  double* S = (double*)malloc(sizeof(double) * n * n);
  double* U = (double*)malloc(sizeof(double) * n * n);
  double* Y = (double*)malloc(sizeof(double) * m * n);
  orc_gram_euclid(m, n, Z, ldz, G, n);
  int info = orc_potrf(n, G, n, S, n);
  if (!info) {
    orc_trsm(m, n, Z, ldz, S, n, Y, m);
    int info2 = orc_normal_tridiag(m, n, d, e, Y, m, Q, U);
    if (info2) info = (int)n + info2;
    else orc_trmm(n, U, n, S, n, R, n);
  }
  free(G); free(S); free(U); free(Y);
  return info;
}

/* E = Q^T A Q - I for tridiagonal A, double-double (the same checker as orc_dd_orth). */
void orc_dd_orth_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Q, int64_t ldq,
                         double* E) {
  dd_t* AQ = (dd_t*)malloc(sizeof(dd_t) * m * n);
#pragma omp parallel for schedule(static)
  for (int64_t l = 0; l < n; l++) {
    const double* q = Q + l * ldq;
    for (int64_t i = 0; i < m; i++) {
      dd_t s = {0.0, 0.0};
      if (i > 0) s = dd_add_prod(s, e[i - 1], q[i - 1]);
      s = dd_add_prod(s, d[i], q[i]);
      if (i < m - 1) s = dd_add_prod(s, e[i], q[i + 1]);
      AQ[l * m + i] = s;
    }
  }
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t l = 0; l < n; l++)
    for (int64_t k = 0; k < n; k++) {
      dd_t s = {k == l ? -1.0 : 0.0, 0.0};
      for (int64_t i = 0; i < m; i++) s = dd_add_dd_prod(s, Q[k * ldq + i], AQ[l * m + i]);
      E[l * n + k] = s.hi + s.lo;
    }
  free(AQ);
}

/* ========================================================================= */
/* NEXT-N1: PRE-CHOLQR with a STABLE Euclidean pre-step (reading R21). */
/* Theorem 3 assumes a backward-stable Euclidean QR of Z; the */
/* pre-step here is shifted CholeskyQR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto,  */
/* Yanagisawa, SIAM J. Sci. Comput. 42 (2020)), stable for kappa(Z) <~ 1/u:       */
/*   G = Z^T Z;  s = 11 (m n + n (n+1)) u tr(G)   (tr(G) = ||Z||_F^2 >= ||Z||_2^2,  */
/*   summed i ascending);  R1 = chol(G + s I);  Q1 = Z / R1;                        */
/*   [Q2, R2] = CholQR(Q1);  [Y, R3] = CholQR(Q2);  S = R3 R2 R1;                   */
/* then the A-stage [Q, U] = CHOLQR(A, Y) and R = U S.          */
/* Breakdown in any pre-step Cholesky -> k; in the A-stage -> n + k.              */
/* ========================================================================= */
static int orc_cholqr_euclid(int64_t m, int64_t n, const double* Z, int64_t ldz, double* Q, double* R,
                             double shift_factor) {
  double* G = (double*)malloc(sizeof(double) * n * n);
  orc_gram_euclid(m, n, Z, ldz, G, n);
  if (shift_factor > 0.0) {
    double tr = 0.0;
    for (int64_t i = 0; i < n; i++) tr += G[i * n + i];
    const double s = shift_factor * tr;
    for (int64_t i = 0; i < n; i++) G[i * n + i] += s;
  }
  int info = orc_potrf(n, G, n, R, n);
  free(G);
  if (info) return info;
  orc_trsm(m, n, Z, ldz, R, n, Q, m);
  return 0;
}

int orc_scqr3(int64_t m, int64_t n, const double* Z, int64_t ldz, double* Y, double* S) {
  const double u = 0x1.0p-53;
  const double shift_factor = 11.0 * ((double)m * (double)n + (double)n * (double)(n + 1)) * u;
  double* R1 = (double*)malloc(sizeof(double) * n * n);
  double* R2 = (double*)malloc(sizeof(double) * n * n);
  double* R3 = (double*)malloc(sizeof(double) * n * n);
  double* T = (double*)malloc(sizeof(double) * n * n);
  double* Q1 = (double*)malloc(sizeof(double) * m * n);
  double* Q2 = (double*)malloc(sizeof(double) * m * n);
  int info = orc_cholqr_euclid(m, n, Z, ldz, Q1, R1, shift_factor);
  if (!info) info = orc_cholqr_euclid(m, n, Q1, m, Q2, R2, 0.0);
  if (!info) info = orc_cholqr_euclid(m, n, Q2, m, Y, R3, 0.0);
  if (!info) {
    orc_trmm(n, R3, n, R2, n, T, n);   /* T = R3 R2 */
    orc_trmm(n, T, n, R1, n, S, n);    /* S = T R1  */
  }
  free(R1); free(R2); free(R3); free(T); free(Q1); free(Q2);
  return info;
}

int orc_prequr_stable(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                      double* Q, double* R) {
  double* S = (double*)malloc(sizeof(double) * n * n);
  double* U = (double*)malloc(sizeof(double) * n * n);
  double* Y = (double*)malloc(sizeof(double) * m * n);
  int info = orc_scqr3(m, n, Z, ldz, Y, S);
  if (!info) {
    int info2 = orc_normal(m, n, A, lda, Y, m, Q, U);
    if (info2) info = (int)n + info2;
    else orc_trmm(n, U, n, S, n, R, n);
  }
  free(S); free(U); free(Y);
  return info;
}

/* ========================================================================= */
/* NEXT-N1 (paper-faithful): PRE-CHOLQR with a Householder Euclidean pre-step. */
/* Algorithm 2 line 1: "[Y,S] = qr(Z)" with "a stable       */
/* Euclidean QR factorization (such as Householder QR)".    */
/* Plain unblocked Householder QR (LAPACK dgeqr2 / dlarfg convention) and the  */
/* explicit first n columns of Q (dorg2r: reflectors applied to I[:, :n] in    */
/* reverse order), then the positive-diagonal normalisation of the problem     */
/* statement (R with positive diagonal): for r_jj < 0 the row  */
/* j of S and the column j of Y change sign (exact).                           */
/*   column j:  alpha = X[j,j];  nrm2 = sum_{i>=j} X[i,j]^2 (i ascending);     */
/*     if nrm2 == alpha^2 (x below the diagonal is zero): tau_j = 0, beta = alpha */
/*     else beta = -sign(alpha) sqrt(nrm2);  tau_j = (beta - alpha) / beta;    */
/*          v_j = 1, v_i = X[i,j] / (alpha - beta) (i > j);  X[j,j] = beta;    */
/*     for l > j:  w = X[j,l] + sum_{i>j} v_i X[i,l];  X[i,l] -= tau_j v_i w.  */
/* ========================================================================= */
void orc_geqr2(int64_t m, int64_t n, double* X, int64_t ldx, double* tau) {
  for (int64_t j = 0; j < n; j++) {
    double* xj = X + j * ldx;
    const double alpha = xj[j];
    double tail = 0.0;
    for (int64_t i = j + 1; i < m; i++) tail += xj[i] * xj[i];
    if (tail == 0.0) { tau[j] = 0.0; continue; }
    const double nrm = sqrt(alpha * alpha + tail);
    const double beta = alpha >= 0.0 ? -nrm : nrm;
    tau[j] = (beta - alpha) / beta;
    const double scal = 1.0 / (alpha - beta);
    for (int64_t i = j + 1; i < m; i++) xj[i] *= scal;
    xj[j] = beta;
    /* the columns l > j are independent: OpenMP splits them (disjoint outputs, same arithmetic) */
#pragma omp parallel for schedule(static)
    for (int64_t l = j + 1; l < n; l++) {
      double* xl = X + l * ldx;
      double w = xl[j];
      for (int64_t i = j + 1; i < m; i++) w += xj[i] * xl[i];
      xl[j] -= tau[j] * w;
      for (int64_t i = j + 1; i < m; i++) xl[i] -= tau[j] * xj[i] * w;
    }
  }
}

/* Y (m x n, ld m) = H_0 H_1 ... H_{n-1} I[:, :n] with H_j = I - tau_j v_j v_j^T (v_j stored
 * below the diagonal of X, unit at j): the reflectors applied to I[:, :n] last to first. */
void orc_org2r(int64_t m, int64_t n, const double* X, int64_t ldx, const double* tau, double* Y) {
  for (int64_t l = 0; l < n; l++)
    for (int64_t i = 0; i < m; i++) Y[l * m + i] = (i == l) ? 1.0 : 0.0;
  for (int64_t j = n - 1; j >= 0; j--) {
    const double* v = X + j * ldx;
#pragma omp parallel for schedule(static)
    for (int64_t l = j; l < n; l++) {
      double* y = Y + l * m;
      double w = y[j];
      for (int64_t i = j + 1; i < m; i++) w += v[i] * y[i];
      y[j] -= tau[j] * w;
      for (int64_t i = j + 1; i < m; i++) y[i] -= tau[j] * v[i] * w;
    }
  }
}

/* [Y, S] = Householder QR of Z with positive-diagonal S (Y: m x n ld m, S: n x n ld n). */
int orc_hhqr(int64_t m, int64_t n, const double* Z, int64_t ldz, double* Y, double* S) {
  double* X = (double*)malloc(sizeof(double) * m * n);
  double* tau = (double*)malloc(sizeof(double) * n);
  for (int64_t l = 0; l < n; l++) memcpy(X + l * m, Z + l * ldz, sizeof(double) * m);
  orc_geqr2(m, n, X, m, tau);
  orc_org2r(m, n, X, m, tau, Y);
  for (int64_t l = 0; l < n; l++)
    for (int64_t k = 0; k < n; k++) S[l * n + k] = (k <= l) ? X[l * m + k] : 0.0;
  for (int64_t j = 0; j < n; j++)
    if (S[j * n + j] < 0.0) {
      for (int64_t l = j; l < n; l++) S[l * n + j] = -S[l * n + j];
      for (int64_t i = 0; i < m; i++) Y[j * m + i] = -Y[j * m + i];
    }
  free(X); free(tau);
  return 0;
}

/* PRE-CHOLQR (Algorithm 2) exactly as the paper states it: Householder pre-step, then
 * [Q, U] = CHOLQR(A, Y) and R = U S.  A-stage breakdown -> n + k. */
int orc_prequr_hh(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                  double* Q, double* R) {
  double* S = (double*)malloc(sizeof(double) * n * n);
  double* U = (double*)malloc(sizeof(double) * n * n);
  double* Y = (double*)malloc(sizeof(double) * m * n);
  int info = orc_hhqr(m, n, Z, ldz, Y, S);
  if (!info) {
    int info2 = orc_normal(m, n, A, lda, Y, m, Q, U);
    if (info2) info = (int)n + info2;
    else orc_trmm(n, U, n, S, n, R, n);
  }
  free(S); free(U); free(Y);
  return info;
}

/* E = Y^T Y - I (n x n, ld n), double-double (Euclidean orthogonality of a pre-step factor). */
void orc_dd_orth_euclid(int64_t m, int64_t n, const double* Y, int64_t ldy, double* E) {
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t l = 0; l < n; l++)
    for (int64_t k = 0; k < n; k++) {
      dd_t s = {k == l ? -1.0 : 0.0, 0.0};
      for (int64_t i = 0; i < m; i++) s = dd_add_prod(s, Y[k * ldy + i], Y[l * ldy + i]);
      E[l * n + k] = s.hi + s.lo;
    }
}
