/*
 * oqr_gen.c -- seeded synthetic input generator for the oblique-QR hot path.
 *
 * INPUT GENERATION ONLY.  This module holds none of the method's arithmetic
 * (no A*Z product, no Gram matrix, no Cholesky, no triangular solve).  It is
 * shared by the CUDA path's tests/bench and by the oracle, and by nothing else.
 *
 * Recipe (BASELINE.json configs[0..4]; paper s7):
 *   A = V diag(d) V^T,  V = H1 H2 H3 H4 = I - Y T Y^T  (4 Householder reflectors,
 *       Gaussian unit vectors, compact WY; T upper triangular, T_jj = 2,
 *       T(1:j-1,j) = -2 T(1:j-1,1:j-1) Y(:,1:j-1)^T v_j),
 *       d_i = kappa_A^{-(i-1)/(m-1)}  (1 down to 1/kappa_A; reading R11).
 *   Z = U diag(s) W^T,  s_k = kappa_Z^{-(k-1)/(n-1)}  (reading R10),
 *       W = 4-reflector product of order n,
 *       U depends on `ucase`:
 *         OQR_GEN_REFLECT (0): first n columns of a fresh 4-reflector product of order m
 *                              (the BASELINE.json configs);
 *         OQR_GEN_TOP     (2): columns of V for the n largest eigenvalues (paper case 2);
 *         OQR_GEN_BOTTOM  (1): columns of V for the n smallest eigenvalues (paper case 1);
 *         OQR_GEN_SPLIT   (3): floor(n/2) largest and ceil(n/2) smallest (paper case 3);
 *         OQR_GEN_AORTH   (5): the case-3 columns with s_k = d_{J_k}^{-1/2} (paper case 5).
 *       Singular values are paired in descending order with descending selected d.
 *   A is computed for i <= j and mirrored, so it is bitwise symmetric.
 *
 * RNG: SplitMix64 (counter-based: draw k of stream s is splitmix64 of
 * seed + (s << 40) + k), 53-bit uniforms in (0,1), Box-Muller normals.
 * Substreams: 1 = V, 2 = U, 3 = W.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OQR_GEN_REFLECT 0
#define OQR_GEN_BOTTOM 1
#define OQR_GEN_TOP 2
#define OQR_GEN_SPLIT 3
#define OQR_GEN_AORTH 5
#define NREFL 4

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* uniform in (0,1): (k + 0.5) * 2^-53 */
static double unif(uint64_t seed, uint64_t stream, uint64_t k) {
  uint64_t r = splitmix64(seed + (stream << 40) + k) >> 11;
  return ((double)r + 0.5) * 0x1.0p-53;
}

/* k-th standard normal of a stream (Box-Muller, cosine branch). */
double oqr_gen_normal(uint64_t seed, uint64_t stream, uint64_t k) {
  double u1 = unif(seed, stream, 2 * k);
  double u2 = unif(seed, stream, 2 * k + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* NREFL Gaussian unit vectors of length len (Y, len x NREFL col-major) and the
 * WY triangular factor T (NREFL x NREFL col-major, upper) with
 * H1 H2 ... H_NREFL = I - Y T Y^T,  H_j = I - 2 v_j v_j^T. */
void oqr_gen_wy(int64_t len, uint64_t seed, uint64_t stream, double* Y, double* T) {
  for (int j = 0; j < NREFL; j++) {
    double nrm2 = 0.0;
    for (int64_t i = 0; i < len; i++) {
      double g = oqr_gen_normal(seed, stream, (uint64_t)j * (uint64_t)len + (uint64_t)i);
      Y[j * len + i] = g;
      nrm2 += g * g;
    }
    double inv = 1.0 / sqrt(nrm2);
    for (int64_t i = 0; i < len; i++) Y[j * len + i] *= inv;
  }
  memset(T, 0, sizeof(double) * NREFL * NREFL);
  for (int j = 0; j < NREFL; j++) {
    double w[NREFL]; /* w = Y(:,0:j-1)^T v_j */
    for (int a = 0; a < j; a++) {
      double s = 0.0;
      for (int64_t i = 0; i < len; i++) s += Y[a * len + i] * Y[j * len + i];
      w[a] = s;
    }
    for (int a = 0; a < j; a++) {
      double s = 0.0;
      for (int b = a; b < j; b++) s += T[b * NREFL + a] * w[b];
      T[j * NREFL + a] = -2.0 * s;
    }
    T[j * NREFL + j] = 2.0;
  }
}

/* d_i = kappa^{-(i)/(m-1)}, i = 0..m-1 (descending from 1 to 1/kappa). */
void oqr_gen_logspace(int64_t m, double kappa, double* d) {
  for (int64_t i = 0; i < m; i++)
    d[i] = (m == 1) ? 1.0 : pow(kappa, -(double)i / (double)(m - 1));
}

/* column c of I - Y T Y^T at row i: delta_ic - y_i^T (T y_c). */
static double wy_entry(const double* Y, int64_t len, const double* Tyc, int64_t i, int64_t c) {
  double s = 0.0;
  for (int a = 0; a < NREFL; a++) s += Y[a * len + i] * Tyc[a];
  return (i == c ? 1.0 : 0.0) - s;
}

static void T_times_y(const double* T, const double* Y, int64_t len, int64_t c, double* out) {
  for (int a = 0; a < NREFL; a++) {
    double s = 0.0;
    for (int b = a; b < NREFL; b++) s += T[b * NREFL + a] * Y[b * len + c];
    out[a] = s;
  }
}

/* Selected eigen-indices (descending d <=> ascending index) for the cases. */
static void select_cols(int64_t m, int64_t n, int ucase, int64_t* J) {
  if (ucase == OQR_GEN_TOP) {
    for (int64_t k = 0; k < n; k++) J[k] = k;
  } else if (ucase == OQR_GEN_BOTTOM) {
    for (int64_t k = 0; k < n; k++) J[k] = m - n + k;
  } else { /* split / aorth: floor(n/2) largest, ceil(n/2) smallest */
    int64_t nl = n / 2, ns = n - nl;
    for (int64_t k = 0; k < nl; k++) J[k] = k;
    for (int64_t k = 0; k < ns; k++) J[nl + k] = m - ns + k;
  }
}

/* Per-row coefficients of the closed form of A = V diag(d) V^T (V = I - Y T Y^T):
 * K = Y^T diag(d) Y, M = T K T^T, and for each row i: p_i = T y_i, q_i = T^T y_i, r_i = M y_i
 * (P[i*12 + 0..3 | 4..7 | 8..11]).  Caller frees. */
static double* a_prep(int64_t m, const double* Yv, const double* Tv, const double* d) {
  double K[NREFL * NREFL], TK[NREFL * NREFL], M[NREFL * NREFL];
  for (int a = 0; a < NREFL; a++)
    for (int b = 0; b < NREFL; b++) {
      double s = 0.0;
      for (int64_t i = 0; i < m; i++) s += Yv[a * m + i] * d[i] * Yv[b * m + i];
      K[b * NREFL + a] = s;
    }
  for (int a = 0; a < NREFL; a++)
    for (int b = 0; b < NREFL; b++) {
      double s = 0.0;
      for (int c = 0; c < NREFL; c++) s += Tv[c * NREFL + a] * K[b * NREFL + c];
      TK[b * NREFL + a] = s;
    }
  for (int a = 0; a < NREFL; a++)
    for (int b = 0; b < NREFL; b++) {
      double s = 0.0;
      for (int c = 0; c < NREFL; c++) s += TK[c * NREFL + a] * Tv[c * NREFL + b];
      M[b * NREFL + a] = s;
    }
  double* P = (double*)malloc(sizeof(double) * m * 3 * NREFL);
  for (int64_t i = 0; i < m; i++) {
    double* pi = P + i * 3 * NREFL;
    for (int a = 0; a < NREFL; a++) {
      double sp = 0.0, sq = 0.0, sr = 0.0;
      for (int b = 0; b < NREFL; b++) {
        double yb = Yv[b * m + i];
        sp += Tv[b * NREFL + a] * yb;
        sq += Tv[a * NREFL + b] * yb;
        sr += M[b * NREFL + a] * yb;
      }
      pi[a] = sp;
      pi[NREFL + a] = sq;
      pi[2 * NREFL + a] = sr;
    }
  }
  return P;
}

/* A_ij for i <= j: d_i delta_ij - d_i (T y_i).y_j - d_j (T^T y_i).y_j + (M y_i).y_j.
 * The stored matrix uses this value for both (i, j) and (j, i): bitwise symmetric. */
static inline double a_entry(const double* P, const double* Yv, const double* d, int64_t m, int64_t i,
                             int64_t j) {
  const double* pi = P + i * 3 * NREFL;
  double t1 = 0.0, t2 = 0.0, t3 = 0.0;
  for (int a = 0; a < NREFL; a++) {
    const double yja = Yv[a * m + j];
    t1 += pi[a] * yja;
    t2 += pi[NREFL + a] * yja;
    t3 += pi[2 * NREFL + a] * yja;
  }
  return (i == j ? d[i] : 0.0) - d[i] * t1 - d[j] * t2 + t3;
}

/* Rows [r0, r1) of the same A as oqr_gen_problem (bitwise identical entries), stored as an
 * (r1 - r0) x m column-major block with leading dimension lda >= r1 - r0 -- the row shard of
 * one rank in the row-sharded multi-GPU path.  Returns 0 or -1. */
int oqr_gen_A_rows(int64_t m, double kappa_a, uint64_t seed, int64_t r0, int64_t r1, double* A, int64_t lda) {
  if (m < 1 || kappa_a < 1.0 || r0 < 0 || r1 > m || r1 <= r0 || lda < r1 - r0 || !A) return -1;
  double* Yv = (double*)malloc(sizeof(double) * m * NREFL);
  double* d = (double*)malloc(sizeof(double) * m);
  double Tv[NREFL * NREFL];
  oqr_gen_wy(m, seed, 1, Yv, Tv);
  oqr_gen_logspace(m, kappa_a, d);
  double* P = a_prep(m, Yv, Tv, d);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < m; j++)
    for (int64_t i = r0; i < r1; i++)
      A[j * lda + (i - r0)] = (i <= j) ? a_entry(P, Yv, d, m, i, j) : a_entry(P, Yv, d, m, j, i);
  free(P);
  free(Yv);
  free(d);
  return 0;
}

/*
 * Fill A (m x m, lda) and/or Z (m x n, ldz); either may be NULL.
 * Outputs (each may be NULL): Yv (m x 4), Tv (4 x 4) of V; d (m); s (n);
 * Yu (m x 4), Tu (4 x 4) of U (REFLECT case); Yw (n x 4), Tw (4 x 4) of W;
 * cols (n) the V-columns used for U (or -1).
 * Returns 0, or -1 on bad arguments.
 */
int oqr_gen_problem(int64_t m, int64_t n, double kappa_a, double kappa_z, uint64_t seed, int ucase,
                    double* A, int64_t lda, double* Z, int64_t ldz,
                    double* Yv_out, double* Tv_out, double* d_out, double* s_out,
                    double* Yu_out, double* Tu_out, double* Yw_out, double* Tw_out, int64_t* cols_out) {
  if (m < 1 || n < 1 || n > m || kappa_a < 1.0 || kappa_z < 1.0) return -1;
  if (A && lda < m) return -1;
  if (Z && ldz < m) return -1;
  if (ucase != OQR_GEN_REFLECT && ucase != OQR_GEN_TOP && ucase != OQR_GEN_BOTTOM &&
      ucase != OQR_GEN_SPLIT && ucase != OQR_GEN_AORTH) return -1;

  double* Yv = (double*)malloc(sizeof(double) * m * NREFL);
  double* d = (double*)malloc(sizeof(double) * m);
  double Tv[NREFL * NREFL];
  oqr_gen_wy(m, seed, 1, Yv, Tv);
  oqr_gen_logspace(m, kappa_a, d);

  if (A) {
    double* P = a_prep(m, Yv, Tv, d);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t j = 0; j < m; j++) {
      for (int64_t i = 0; i <= j; i++) {
        const double v = a_entry(P, Yv, d, m, i, j);
        A[j * lda + i] = v;
        A[i * lda + j] = v;
      }
    }
    free(P);
  }

  double* s = (double*)malloc(sizeof(double) * n);
  int64_t* J = (int64_t*)malloc(sizeof(int64_t) * n);
  double Tu[NREFL * NREFL];
  double* Yu = NULL;
  double* Yw = (double*)malloc(sizeof(double) * n * NREFL);
  double Tw[NREFL * NREFL];
  oqr_gen_wy(n, seed, 3, Yw, Tw);
  if (ucase == OQR_GEN_REFLECT) {
    Yu = (double*)malloc(sizeof(double) * m * NREFL);
    oqr_gen_wy(m, seed, 2, Yu, Tu);
    for (int64_t k = 0; k < n; k++) J[k] = -1;
  } else {
    select_cols(m, n, ucase, J);
    memset(Tu, 0, sizeof(Tu));
  }
  if (ucase == OQR_GEN_AORTH) {
    for (int64_t k = 0; k < n; k++) s[k] = 1.0 / sqrt(d[J[k]]);
  } else {
    oqr_gen_logspace(n, kappa_z, s);
  }

  if (Z) {
    /* W (n x n) explicit; U column k evaluated entrywise. Z_il = sum_k U_ik s_k W_lk. */
    double* W = (double*)malloc(sizeof(double) * n * n);
    for (int64_t c = 0; c < n; c++) {
      double Tyc[NREFL];
      T_times_y(Tw, Yw, n, c, Tyc);
      for (int64_t l = 0; l < n; l++) W[c * n + l] = wy_entry(Yw, n, Tyc, l, c);
    }
    double* Tyk = (double*)malloc(sizeof(double) * n * NREFL);
    for (int64_t k = 0; k < n; k++) {
      if (ucase == OQR_GEN_REFLECT) T_times_y(Tu, Yu, m, k, Tyk + k * NREFL);
      else T_times_y(Tv, Yv, m, J[k], Tyk + k * NREFL);
    }
#pragma omp parallel
    {
      double* zrow = (double*)malloc(sizeof(double) * n);
#pragma omp for schedule(static)
      for (int64_t i = 0; i < m; i++) {
        for (int64_t l = 0; l < n; l++) zrow[l] = 0.0;
        for (int64_t k = 0; k < n; k++) {
          double uik = (ucase == OQR_GEN_REFLECT) ? wy_entry(Yu, m, Tyk + k * NREFL, i, k)
                                                  : wy_entry(Yv, m, Tyk + k * NREFL, i, J[k]);
          double us = uik * s[k];
          for (int64_t l = 0; l < n; l++) zrow[l] += us * W[k * n + l];
        }
        for (int64_t l = 0; l < n; l++) Z[l * ldz + i] = zrow[l];
      }
      free(zrow);
    }
    free(Tyk);
    free(W);
  }

  if (Yv_out) memcpy(Yv_out, Yv, sizeof(double) * m * NREFL);
  if (Tv_out) memcpy(Tv_out, Tv, sizeof(Tv));
  if (d_out) memcpy(d_out, d, sizeof(double) * m);
  if (s_out) memcpy(s_out, s, sizeof(double) * n);
  if (Yu_out && Yu) memcpy(Yu_out, Yu, sizeof(double) * m * NREFL);
  if (Tu_out) memcpy(Tu_out, Tu, sizeof(Tu));
  if (Yw_out) memcpy(Yw_out, Yw, sizeof(double) * n * NREFL);
  if (Tw_out) memcpy(Tw_out, Tw, sizeof(Tw));
  if (cols_out) memcpy(cols_out, J, sizeof(int64_t) * n);
  free(Yv); free(d); free(s); free(J); free(Yw);
  if (Yu) free(Yu);
  return 0;
}

/*
 * The paper's s7 construction with DENSE random orthogonal factors:
 *   V = orth(randn(m)) (Haar), U = the case's columns of V, or orth(randn(m, n)) for case 4
 *   (random Z), W = orth(randn(n)) (Haar), A = V diag(d) V^T, Z = U diag(s) W^T.
 * orth() is classical Gram-Schmidt applied twice ("twice is enough") to seeded Gaussian columns,
 * each column normalised to a positive diagonal of the implied R: the Q factor of a Gaussian
 * matrix with positive-diagonal R is Haar distributed.  (Gram-Schmidt is NOT on the library's or
 * the oracle's path; it is used here only to draw random orthogonal matrices.)
 * Substreams: 4 = V, 5 = U (case 4), 6 = W.  A is formed for i <= j and mirrored (bitwise
 * symmetric).  O(m^3): for the s7 sweeps (m = 80) and small parity cases (m <= 4096).
 * Outputs (each may be NULL): V (m x m col-major), d (m), s (n), W (n x n), cols (n).
 */
#define OQR_GEN_RANDOM 4

static void orth_gaussian(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, double* Q) {
  for (int64_t j = 0; j < cols; j++)
    for (int64_t i = 0; i < rows; i++) Q[j * rows + i] = oqr_gen_normal(seed, stream, (uint64_t)(j * rows + i));
  double* h = (double*)malloc(sizeof(double) * (cols > 0 ? cols : 1));
  for (int64_t j = 0; j < cols; j++) {
    double* q = Q + j * rows;
    for (int pass = 0; pass < 2; pass++) {
      for (int64_t k = 0; k < j; k++) {
        const double* qk = Q + k * rows;
        double s = 0.0;
        for (int64_t i = 0; i < rows; i++) s += qk[i] * q[i];
        h[k] = s;
      }
      for (int64_t k = 0; k < j; k++) {
        const double* qk = Q + k * rows;
        for (int64_t i = 0; i < rows; i++) q[i] -= h[k] * qk[i];
      }
    }
    double nrm = 0.0;
    for (int64_t i = 0; i < rows; i++) nrm += q[i] * q[i];
    nrm = sqrt(nrm);
    for (int64_t i = 0; i < rows; i++) q[i] /= nrm;
  }
  free(h);
}

int oqr_gen_problem_haar(int64_t m, int64_t n, double kappa_a, double kappa_z, uint64_t seed, int ucase,
                         double* A, int64_t lda, double* Z, int64_t ldz, double* V_out, double* d_out,
                         double* s_out, double* W_out, int64_t* cols_out) {
  if (m < 1 || n < 1 || n > m || m > 4096 || kappa_a < 1.0 || kappa_z < 1.0) return -1;
  if (A && lda < m) return -1;
  if (Z && ldz < m) return -1;
  if (ucase != OQR_GEN_RANDOM && ucase != OQR_GEN_TOP && ucase != OQR_GEN_BOTTOM && ucase != OQR_GEN_SPLIT &&
      ucase != OQR_GEN_AORTH) return -1;
  double* V = (double*)malloc(sizeof(double) * m * m);
  double* d = (double*)malloc(sizeof(double) * m);
  double* s = (double*)malloc(sizeof(double) * n);
  double* W = (double*)malloc(sizeof(double) * n * n);
  double* Uc = (double*)malloc(sizeof(double) * m * n);
  int64_t* J = (int64_t*)malloc(sizeof(int64_t) * n);
  orth_gaussian(m, m, seed, 4, V);
  oqr_gen_logspace(m, kappa_a, d);
  orth_gaussian(n, n, seed, 6, W);
  if (ucase == OQR_GEN_RANDOM) {
    orth_gaussian(m, n, seed, 5, Uc);
    for (int64_t k = 0; k < n; k++) J[k] = -1;
  } else {
    select_cols(m, n, ucase, J);
    for (int64_t k = 0; k < n; k++) memcpy(Uc + k * m, V + J[k] * m, sizeof(double) * m);
  }
  if (ucase == OQR_GEN_AORTH) {
    for (int64_t k = 0; k < n; k++) s[k] = 1.0 / sqrt(d[J[k]]);
  } else {
    oqr_gen_logspace(n, kappa_z, s);
  }
  if (A) {
    /* rows of V contiguous (Vt[i*m + k] = V[i, k]): the same sums, k ascending, cache-friendly */
    double* Vt = (double*)malloc(sizeof(double) * m * m);
    for (int64_t k = 0; k < m; k++)
      for (int64_t i = 0; i < m; i++) Vt[i * m + k] = V[k * m + i];
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t j = 0; j < m; j++)
      for (int64_t i = 0; i <= j; i++) {
        const double* vi = Vt + i * m;
        const double* vj = Vt + j * m;
        double v = 0.0;
        for (int64_t k = 0; k < m; k++) v += vi[k] * d[k] * vj[k];
        A[j * lda + i] = v;
        A[i * lda + j] = v;
      }
    free(Vt);
  }
  if (Z) {
    for (int64_t l = 0; l < n; l++)
      for (int64_t i = 0; i < m; i++) {
        double v = 0.0;
        for (int64_t k = 0; k < n; k++) v += Uc[k * m + i] * s[k] * W[k * n + l];
        Z[l * ldz + i] = v;
      }
  }
  if (V_out) memcpy(V_out, V, sizeof(double) * m * m);
  if (d_out) memcpy(d_out, d, sizeof(double) * m);
  if (s_out) memcpy(s_out, s, sizeof(double) * n);
  if (W_out) memcpy(W_out, W, sizeof(double) * n * n);
  if (cols_out) memcpy(cols_out, J, sizeof(int64_t) * n);
  free(V); free(d); free(s); free(W); free(Uc); free(J);
  return 0;
}
