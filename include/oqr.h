/*
 * oqr.h -- C ABI of liboqr.so, the B200 (sm_100a) oblique-QR normal-equation library.
 *
 * Problem (s1 "Introduction"): given A (m x m) symmetric positive definite
 * and Z (m x n) of full column rank, m >= n, find Q (m x n) and R (n x n, upper triangular,
 * positive diagonal) with  Z = Q R  and  Q^T A Q = I.
 *
 * Method: Algorithm 1 "CHOLQR" (s2):
 *     B = A Z;  C = Z^T B;  R = chol(C);  Q = Z / R.
 * The library fuses lines 1-2 into one kernel that streams A once and never stores B.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - FP64 (IEEE binary64, round-to-nearest), column-major.  Element (i, j) of a matrix with
 *    leading dimension ld is p[j*ld + i].  All matrix pointers are DEVICE pointers owned by
 *    the caller; the library never frees or retains them.
 *  - A is read in full as given (both triangles); it is never written.  Z is never written.
 *  - lda, ldz >= m; all pointers 8-byte aligned.  FAST PATH: A 16-byte aligned and lda even --
 *    the fused Gram kernel then moves each 64 x KS tile of A with one tensor-TMA request
 *    (m % 8 == 0: a 4-D view that lands the tile bank-conflict-free; otherwise the 2-D view);
 *    with a misaligned A or odd lda it falls back to plain loads for every tile (same results,
 *    much slower).
 *  - 1 <= n <= min(m, OQR_NMAX).
 *  - Q: m x n output with leading dimension m.  R: n x n output with leading dimension n,
 *    upper triangular with positive diagonal; its strictly lower part is written as zero.
 *  - Outputs must not overlap the inputs or each other.
 *  - All work is enqueued on `stream` (0 = legacy default stream).  Scratch memory is
 *    stream-ordered (cudaMallocFromPoolAsync / cudaFreeAsync on a memory pool the library owns;
 *    the device's default pool is not touched), so concurrent calls on different streams are safe.
 *
 * Status codes (LAPACK conventions):
 *     0        success
 *     1..n     Cholesky breakdown at pivot k (1-based) of the FIRST Cholesky: oqr_normal,
 *              pass 1 of oqr_normal2, the Euclidean pre-step of oqr_prequr.  A pivot
 *              breaks down when it is <= 0 or NaN (reading R4).
 *     n+1..2n  breakdown at pivot k of the SECOND Cholesky (pass 2 of oqr_normal2, the
 *              A-stage of oqr_prequr); the code is n + k (LAPACK xSYGV's INFO = N + i idiom).
 *    -i        argument i is invalid: -1 m, -2 n, -3 A (null or not 8-byte aligned), -4 lda
 *              (< m), -5 Z, -6 ldz, -7 Q, -8 R.  Nothing is launched.
 *   -100       a CUDA error occurred (launch or runtime); -101 workspace allocation failed;
 *   -102       caller-provided workspace too small or misaligned (async calls).
 *  On any nonzero status the contents of Q and R are unspecified.
 *
 * Preconditions that are NOT checked (reading R17): that A is SPD and
 * that Z has full rank.  A violation surfaces as a breakdown status or as a large
 * ||Q^T A Q - I||, exactly as in the CPU oracle.
 */
#ifndef OQR_H
#define OQR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OQR_NMAX 240

/* cudaStream_t without pulling in the CUDA headers. */
typedef struct CUstream_st* oqr_stream_t;

/*
 * oqr_normal -- CHOLQR, Algorithm 1.
 *   G = Z^T (A Z) (lines 1-2, fused; A streamed once), R = chol(G) (line 3),
 *   Q = Z R^{-1} by row-wise substitution (line 4).
 * Synchronous: enqueues on `stream`, then synchronises `stream` and returns the status.
 * Small problems (m*m*n <= 1.1e10; all synchronous dense variants -- and the synchronous
 * tridiagonal oqr_normal/normal2/prequr_tridiag with m*n*n <= 2e10): from the second call with the
 * same arguments (sizes, pointers, stream, device) on, the call replays a CUDA graph of its
 * asynchronous form captured once, with its own cached workspace (same kernels, bitwise the same
 * results; at most 8 such graphs per process; oqr_pool_trim releases them; never while the
 * timing hook is on).
 */
int oqr_normal(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
               double* Q, double* R, oqr_stream_t stream);

/*
 * oqr_normal_host -- oqr_normal on HOST arrays: the same Algorithm 1 for a
 * caller whose A, Z live in host memory and who wants Q, R back in host memory.  A (lda >= m),
 * Z (ldz >= m) are read; Q (leading dimension m) and R (n x n, leading dimension n) are written.
 * Page-locked host memory (cudaHostAlloc / cudaHostRegister) gives full PCIe bandwidth and the
 * overlap below; pageable memory works, serialised.  The library streams A through a ring of
 * three device chunk buffers from its pool, `chunk_cols` columns each (0: automatic -- the ring
 * is ~1 GiB whatever m is, at most m/8 columns a chunk; rounded up to a multiple of 64), on its
 * own copy stream, and runs the fused Gram on each chunk as soon as it has landed
 * (G = sum_J Z^T A[:, J] Z[J, :], chunks summed in order into the same per-CTA slots:
 * deterministic for a given chunk size, within the same T1 bound as oqr_normal but not bitwise
 * equal to it), so the A transfer -- the bound of a host-to-host factorisation -- hides all
 * but the last chunk's Gram, and the device footprint does not grow with A (an A larger than
 * the GPU's memory factors).  Synchronous on `stream`.  Status and argument codes as oqr_normal
 * (-3 / -5 / -7 / -8: null host pointer), plus -9 for chunk_cols < 0.
 */
int oqr_normal_host(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                    double* Q, double* R, int64_t chunk_cols, oqr_stream_t stream);

/*
 * oqr_normal2 -- repeated CHOLQR (north_star; reading R1, the CGS2 analogue of
 * PAPER.md:673-681):  [Q1, R1] = CHOLQR(A, Z);  [Q, R2] = CHOLQR(A, Q1);  R = R2 R1.
 * The second pass re-streams A (it must see A * dQ1).  Q1 lives in Q.
 */
int oqr_normal2(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                double* Q, double* R, oqr_stream_t stream);

/*
 * oqr_prequr -- PRE-CHOLQR, Algorithm 2 with the Euclidean pre-QR done by
 * Cholesky-QR as north_star specifies (reading R2):
 *   S = chol(Z^T Z), Y = Z S^{-1};  [Q, U] = CHOLQR(A, Y);  R = U S.
 * Y lives in Q and is overwritten in place by Q = Y U^{-1}.
 */
int oqr_prequr(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
               double* Q, double* R, oqr_stream_t stream);

/*
 * Symmetric-A variants.  A is SPD, hence symmetric: these read
 * only the block-lower triangle of A (64 x 64 blocks: A[i, j] for floor(j/64) <= floor(i/64))
 * -- half the bytes and half the flops of the dense calls.  With A = L + D + L^T by blocks,
 * G = Z^T A Z = T + T^T where T = sum_I Z_I^T (sum_{J<I} A_IJ Z_J + (1/2) A_II Z_I); the 1/2 is
 * applied exactly to Z.  G is bitwise symmetric.  Same arguments, outputs and status codes as
 * the dense calls; for an A that is not symmetric they factor the block-lower symmetrisation.
 */
int oqr_normal_sym(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                   double* Q, double* R, oqr_stream_t stream);
int oqr_normal2_sym(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                    double* Q, double* R, oqr_stream_t stream);
int oqr_prequr_sym(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                   double* Q, double* R, oqr_stream_t stream);
/* Host -> device copy of exactly what the *_sym calls read: the block-lower triangle of a
 * column-major host A (lda >= m; pinned memory for asynchrony) into A_dev (ldda >= m), one 2-D copy
 * per 64-column panel (rows from the panel's first row to m): ~half of A's bytes.  Asynchronous on
 * `stream`; the block-upper part of A_dev is left untouched.  Status: 0, -1 m, -2 A_host, -3 lda,
 * -4 A_dev, -5 ldda, -100 CUDA. */
int oqr_upload_sym(int64_t m, const double* A_host, int64_t lda, double* A_dev, int64_t ldda, oqr_stream_t stream);

/* Step export of the symmetric Gram (asynchronous). */
int oqr_gram_sym(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz, double* G,
                 oqr_stream_t stream);

/*
 * Tridiagonal A (the paper's second workload):
 * A = tridiag(e, d, e) symmetric positive definite, d: m diagonal entries, e: m-1 off-diagonal
 * entries (device pointers; e may be NULL when m == 1).  Same algorithms, outputs and status
 * codes as the dense calls; argument codes: -1 m, -2 n, -3 d, -4 e, -5 Z, -6 ldz, -7 Q, -8 R.
 * The A-product is the 3-point stencil (O(mn)), fused into the packing of the Gram operand;
 * the Gram Z^T (A Z) then runs on the FP64 tensor pipe.  Synchronous, like oqr_normal.
 */
int oqr_normal_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Z, int64_t ldz,
                       double* Q, double* R, oqr_stream_t stream);
int oqr_normal2_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Z,
                        int64_t ldz, double* Q, double* R, oqr_stream_t stream);
int oqr_prequr_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Z, int64_t ldz,
                       double* Q, double* R, oqr_stream_t stream);

/*
 * oqr_prequr_stable -- PRE-CHOLQR (Algorithm 2) with a STABLE Euclidean pre-step
 * (reading R21): shifted CholeskyQR3 (Fukaya et al., SIAM J. Sci.
 * Comput. 42, 2020) -- G = Z^T Z, R1 = chol(G + 11 (m n + n(n+1)) u tr(G) I), Q1 = Z R1^{-1}, two
 * Cholesky-QR passes on Q1 (R2, R3), Y = Q3, S = R3 R2 R1 -- a backward-stable QR of Z for
 * kappa(Z) up to ~1/u, which is what Theorem 3 assumes of the pre-step; then
 * [Q, U] = CHOLQR(A, Y) and R = U S.  Removes the kappa(Z) <~ 1e7.5 limit of oqr_prequr.
 * Breakdown in any pre-step Cholesky: code k; in the A-stage: n + k.  Y lives in Q.
 * _sym / _tridiag: the same with the symmetric (block-lower) or tridiagonal A-stage.
 */
int oqr_prequr_stable(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                      double* Q, double* R, oqr_stream_t stream);
int oqr_prequr_stable_sym(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                          double* Q, double* R, oqr_stream_t stream);
int oqr_prequr_stable_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Z,
                              int64_t ldz, double* Q, double* R, oqr_stream_t stream);

/*
 * oqr_prequr_hh -- PRE-CHOLQR exactly as Algorithm 2 states it: the pre-step
 * [Y, S] = qr(Z) is a Householder QR, "a stable Euclidean QR factorization (such as Householder
 * QR)", the pre-step Theorem 3 is proved for; then
 * [Q, U] = CHOLQR(A, Y) and R = U S.  The pre-step is backward stable for EVERY
 * full-rank Z (no kappa(Z) limit: ||Y^T Y - I|| = O(m n u), ||Z - Y S|| = O(m n u) ||Z||) and never
 * breaks down; only the A-stage can (status n + k).  S has a positive diagonal (LAPACK dlarfg
 * reflectors, then row/column sign flips, exact).  Y lives in Q.  Householder QR runs as one
 * cooperative kernel (all CTAs co-resident, grid barriers) whose per-CTA row block must fit in
 * shared memory: m up to ~1.5e5 at n = 240 (larger m: status -1).
 * _sym / _tridiag: the same with the symmetric (block-lower) or tridiagonal A-stage.
 */
int oqr_prequr_hh(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                  double* Q, double* R, oqr_stream_t stream);
int oqr_prequr_hh_sym(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                      double* Q, double* R, oqr_stream_t stream);
int oqr_prequr_hh_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Z,
                          int64_t ldz, double* Q, double* R, oqr_stream_t stream);

/*
 * Asynchronous variants (CUDA-graph capturable).  Same computation as the synchronous calls, but
 * nothing is synchronised: the call enqueues its kernels on `stream` and returns 0 (or a negative
 * argument status, nothing enqueued); the factorisation status (0, k, n + k as above) is written to
 * the device int *d_status when the stream reaches it.  workspace: caller-provided device memory of
 * at least oqr_workspace_bytes(m, n) bytes, 256-byte aligned (then no allocation happens inside and
 * the call can be captured into a CUDA graph), or NULL for a stream-ordered allocation from the
 * library's pool.  Extra statuses: -9 d_status null, -102 workspace too small / misaligned.
 */
size_t oqr_workspace_bytes(int64_t m, int64_t n);
int oqr_normal_async(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz, double* Q,
                     double* R, void* workspace, size_t workspace_bytes, int* d_status, oqr_stream_t stream);
int oqr_normal2_async(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz, double* Q,
                      double* R, void* workspace, size_t workspace_bytes, int* d_status, oqr_stream_t stream);
int oqr_prequr_async(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz, double* Q,
                     double* R, void* workspace, size_t workspace_bytes, int* d_status, oqr_stream_t stream);
int oqr_prequr_stable_async(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                            double* Q, double* R, void* workspace, size_t workspace_bytes, int* d_status,
                            oqr_stream_t stream);
int oqr_prequr_hh_async(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
                        double* Q, double* R, void* workspace, size_t workspace_bytes, int* d_status,
                        oqr_stream_t stream);

/* The library's device memory pool (current device).  Scratch of the calls is stream-ordered from
 * it; up to 4 GiB of freed blocks stay cached between calls (no driver allocation per call), larger
 * transient staging (oqr_normal_host's device copy of A) is returned to the driver at the call's
 * final synchronisation.  oqr_pool_trim synchronises the device, drops the idle cached CUDA graphs
 * of small synchronous calls (with their workspaces; see oqr_normal) and releases cached pool
 * blocks down to keep_bytes (0: everything not in use); status 0 or -100.  oqr_pool_reserved:
 * bytes the pool currently holds from the driver (or -100). */
int oqr_pool_trim(size_t keep_bytes);
int64_t oqr_pool_reserved(void);

/* Which path the fused Gram kernel takes for an A (m x m, lda): 1 = FAST (16-byte aligned A, even
 * lda: tensor-TMA tiles), 0 = SLOW (8-byte aligned A or odd lda: plain loads for every tile, same
 * results, several times slower); -1 m < 1, -3 A null or not 8-byte aligned, -4 lda < m.  The
 * factorisations accept both paths (the argument checks reject only what neither path can read);
 * callers that need the fast path check it here. */
int oqr_gram_fast_path(int64_t m, const double* A, int64_t lda);

/* Human-readable text for a status code (static storage; never NULL). */
const char* oqr_status_string(int status);

/* ---- Step exports (test and measurement only).  ASYNCHRONOUS: they enqueue and return 0
 *      (or a negative argument / CUDA status) without synchronising.  Workspace is
 *      stream-ordered, so the caller may free nothing until the stream has drained. ---- */

/* G = Z^T (A Z), Algorithm 1 lines 1-2.  G: n x n, ld n, both triangles
 * written (G is not forced symmetric: G[k,l] = sum_i Z[i,k] (AZ)[i,l]).  Summation order is
 * fixed for a given (m, n, SM count), so repeated calls are bitwise identical. */
int oqr_gram(int64_t m, int64_t n, const double* A, int64_t lda, const double* Z, int64_t ldz,
             double* G, oqr_stream_t stream);

/* G = Z^T (T Z) for tridiagonal T = tridiag(e, d, e) (asynchronous step export). */
int oqr_gram_tridiag(int64_t m, int64_t n, const double* d, const double* e, const double* Z, int64_t ldz,
                     double* G, oqr_stream_t stream);

/* G = Z^T Z, the Euclidean Gram of the PRE-CHOLQR pre-step (reading R2).  Unlike the
 * factorisations, n > m is allowed (a row block of the row-sharded path may hold fewer rows than
 * columns): -2 only for n < 1 or n > OQR_NMAX. */
int oqr_gram_euclid(int64_t m, int64_t n, const double* Z, int64_t ldz, double* G,
                    oqr_stream_t stream);

/* R = chol(G), upper, R^T R = G, reading only the upper triangle of G (n x n, ld n);
 * Algorithm 1 line 3.  *d_info (device int) receives 0 or the 1-based pivot
 * of breakdown (pivot <= 0 or NaN).  R: n x n, ld n, strictly lower part zero. */
int oqr_potrf(int64_t n, const double* G, double* R, int* d_info, oqr_stream_t stream);

/* Q = Z R^{-1} by row-wise substitution, Algorithm 1 line 4:
 * q_ij = (z_ij - sum_{k<j} q_ik r_kj) / r_jj.  R: n x n, ld n, upper.  Q: m x n, ld m.
 * Q may equal Z when ldz == m (in-place).  n > m is allowed (rows are independent; a row block of
 * the row-sharded path may hold fewer rows than columns): -2 only for n < 1 or n > OQR_NMAX. */
int oqr_trsm(int64_t m, int64_t n, const double* Z, int64_t ldz, const double* R, double* Q,
             oqr_stream_t stream);

/* R = R2 R1 for upper triangular n x n R2, R1 (ld n): the R of repeated CHOLQR and R = U S of
 * PRE-CHOLQR; R[k, l] = sum_{p=k}^{l} R2[k, p] R1[p, l], strictly lower part zero.
 * Asynchronous.  Status 0, -1 n, -2 R2, -3 R1, -4 R, -100 CUDA. */
int oqr_trmm(int64_t n, const double* R2, const double* R1, double* R, oqr_stream_t stream);

/* [Y, S] = Householder QR of Z (Algorithm 2 line 1; the pre-step of oqr_prequr_hh):
 * Y m x n (ld m) with orthonormal columns, S n x n (ld n) upper triangular with positive diagonal,
 * Z = Y S.  Y must not overlap Z.  Asynchronous.  Status 0, -1 m (too large, see oqr_prequr_hh),
 * -2 n, -5 Z, -6 ldz, -7 Y, -8 S, -100 CUDA, -101 workspace. */
int oqr_hhqr(int64_t m, int64_t n, const double* Z, int64_t ldz, double* Y, double* S, oqr_stream_t stream);

/* ---- Row-sharded multi-GPU path.  Rank r holds rows
 *      R_r = [r0, r0 + mr) of A and all of Z.  Because G = sum_r Z_{R_r}^T (A_{R_r,:} Z) for any
 *      partition of the rows (bilinearity of Algorithm 1 lines 1-2), each rank
 *      computes its partial with oqr_gram_rows, the partials are exchanged once (all-gather,
 *      n x n each), every rank sums them in rank order with oqr_sum_partials (bitwise-identical G
 *      and R everywhere), factors with oqr_potrf and solves its own rows with oqr_trsm. ---- */

/* G_r = Z_{R}^T (A_{R,:} Z), R = rows [r0, r0 + mr) of A.  Ar: the row block, mr x m column-major,
 * leading dimension ldar >= mr (element (i, j) of the block = A[r0 + i, j]); Z: all m rows, ldz >= m.
 * G: n x n, ld n.  Asynchronous.  Status: 0, -1 m, -2 n, -3 Ar, -4 ldar, -5 Z, -6 ldz, -7 G,
 * -9 row range, -100 CUDA, -101 workspace.  With r0 = 0, mr = m this equals oqr_gram. */
int oqr_gram_rows(int64_t m, int64_t n, int64_t r0, int64_t mr, const double* Ar, int64_t ldar,
                  const double* Z, int64_t ldz, double* G, oqr_stream_t stream);

/* G = sum_{c=0}^{count-1} P_c in c order (fixed order => reproducible bits); P holds count
 * consecutive n x n matrices (ld n), G is n x n (ld n).  Asynchronous. */
int oqr_sum_partials(int64_t n, int64_t count, const double* P, double* G, oqr_stream_t stream);

/* ---- Measurement hook: per-launch CUDA-event timing of the fused Gram kernel (K1).
 *      When enabled, every K1 launch is bracketed by events recorded on the caller's stream;
 *      oqr_timing_read returns the accumulated milliseconds and launch count since the last
 *      reset (it synchronises on the recorded events).  Not thread-safe; off by default.
 *      While it is on, the factorisations run every kernel one after the other: neither the cached
 *      CUDA graphs of small calls nor the overlapped Cholesky / solve pair (the solve is otherwise
 *      launched as a programmatic dependent of the Cholesky and runs concurrently with it) are
 *      taken; the results are bitwise the same either way. */
void oqr_timing_enable(int enable);
void oqr_timing_reset(void);
int oqr_timing_read(double* gram_ms, int64_t* gram_launches, int64_t* total_launches);
/* The same hook for one kernel family: OQR_TIMING_K1 (fused Gram, as oqr_timing_read),
 * OQR_TIMING_K4 (packed tall-skinny Gram: Euclidean / tridiagonal), OQR_TIMING_K3 (triangular
 * solve), OQR_TIMING_K2 (Cholesky), OQR_TIMING_K6 (Householder QR).  Status 0, -1 unknown kernel,
 * -100 CUDA. */
#define OQR_TIMING_K1 0
#define OQR_TIMING_K4 1
#define OQR_TIMING_K3 2
#define OQR_TIMING_K2 3
#define OQR_TIMING_K6 4
int oqr_timing_read_kernel(int kernel, double* ms, int64_t* launches);

/* Number of kernels this library has launched since load (all entry points). */
int64_t oqr_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* OQR_H */
