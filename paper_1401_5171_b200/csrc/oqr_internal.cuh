// oqr_internal.cuh -- shared constants, PTX wrappers and launchers of liboqr (sm_100a only).
//
// Nothing here is shared with oracle/ (the CPU checker); see DESIGN.md s3.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/oqr.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "liboqr is written for sm_100a (B200) only"
#endif

namespace oqr {

// ---- Tiling of the fused Gram kernel (K1) and its packed Z layout ----------
constexpr int BM = 64;        // rows of A (and of W = AZ) per panel: NRG row groups x 8 rows
constexpr int BK = 16;        // rows of Z per packed block (a K1 stage moves KS/BK of them)
constexpr int NRG = 8;        // row groups per panel: 8 rows each (BM = 8 * NRG)
constexpr int NCH = 2;        // column halves: warp (rg, ch) owns rows rg*8.. and half the n-tiles
constexpr int NCW = NRG * NCH;  // 16 DMMA warps per CTA (4 per SM sub-partition)
#ifndef OQR_LG
#define OQR_LG 4
#endif
constexpr int LG = OQR_LG;    // n-tiles per warp per contraction chunk (reduction granule)
constexpr int NTMAX = 30;     // n <= 8 * NTMAX = 240 = OQR_NMAX
constexpr int SMEM_MAX = 227 * 1024;
constexpr int FRAG = 32;      // doubles per DMMA operand fragment (one per lane)

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Packed Z ("Zp") in DMMA B-fragment order, no padding.  Block b holds rows [b*BK, b*BK+BK)
// of Z; inside it, fragment (lt, kk) (n-tile lt = 8 columns, k-step kk = 4 rows) is 32
// consecutive doubles, lane-indexed as the B operand of mma.m8n8k4 wants them:
//   Zp[((b*NT + lt)*4 + kk)*32 + lane] = Z[b*BK + kk*4 + lane%4, lt*8 + lane/4]
// (zero for rows >= m and columns >= n).  One pipeline stage's Z tile is then one contiguous
// bulk copy of NT KiB, and every warp fragment load is 256 consecutive bytes (conflict-free).
// Blocks cover every panel row: nblk = ceil(m/BM)*BM/BK.
inline int64_t zp_blocks(int64_t m) { return cdiv(m, BM) * (BM / BK); }
inline int64_t zp_doubles(int64_t m, int NP) { return zp_blocks(m) * (NP / 8) * 4 * FRAG; }

// ---- launch bookkeeping (oqr_abi.cu) ----
void note_launch();
// Raise a kernel's dynamic shared-memory limit once per (kernel, device) -- thread-safe.
cudaError_t ensure_smem_attr(const void* func, int bytes);
// kind: OQR_TIMING_K1 / _K4 / _K3 / _K2 (include/oqr.h)
void timing_begin(cudaStream_t s, int kind);
void timing_end(cudaStream_t s);

// ---- launchers (return cudaError_t of the launch) ----
// Z (m x n, ldz) -> Zp (packed, NP = 8*ceil(n/8) columns)
cudaError_t launch_pack_z(int64_t m, int n, const double* Z, int64_t ldz, double* Zp, cudaStream_t s,
                          double scale = 1.0);
// Per-CTA partial Gram slots P[g][NP][NP] of Z^T (A Z); returns the grid size used in *g_out.
// A is moved by tensor TMA when it is 16-byte aligned with an even lda; otherwise by plain
// loads (same results, slow).  accum: add to the slots instead of overwriting them (a later
// column chunk of A; the grid must not exceed the first chunk's).
// Rows [0, mr) of A (or of a row block of A holding mr rows, all m columns): slots of
// Z_rows^T (A_rows Z) where Zp packs all m rows of Z (B operand) and Zc packs the mr rows of Z
// that match the A rows (contraction operand; Zc == Zp on one GPU).  Zh != nullptr selects the
// symmetric schedule (NEXT-N4; mr == m): only the block-lower triangle of A is read, Zh = Z/2
// packed, and the slots hold T with G = T + T^T (launch_gram_reduce(..., sym = true)).
cudaError_t launch_gram_fused(int64_t m, int64_t mr, int n, const double* A, int64_t lda, const double* Zp,
                              const double* Zc, const double* Zh, double* P, int* g_out, cudaStream_t s,
                              bool accum = false);
// G (n x n, ldg) = sum_{c<count} P_c, P_c = n x n (ld n) consecutive, c ascending.
cudaError_t launch_sum_partials(int n, int count, const double* P, double* G, int64_t ldg, cudaStream_t s);
// Zp and W = T Z (T = tridiag(e, d, e)), both packed, in one pass over Z.
cudaError_t launch_pack_zw_tridiag(int64_t m, int n, const double* d, const double* e, const double* Z, int64_t ldz,
                                   double* Zp, double* Wp, cudaStream_t s);
// Slots of the upper triangle of X^T Y for two packed m x n operands whose product is symmetric
// in exact arithmetic (X = Y = Zp: the Euclidean Gram; Zp and T Z: the tridiagonal one); reduce
// with mirror = true.
cudaError_t launch_gram_packed(int64_t m, int n, const double* Xp, const double* Yp, double* P, int* g_out,
                               cudaStream_t s);
// K4t: slots of the upper triangle of Z^T (T Z), T = tridiag(e, d, e), streaming the column-major
// Z once by tensor TMA with the stencil fused in (no packed copies).  *done = false (nothing
// launched) when Z cannot be described to TMA (16-byte alignment, even ldz): the caller then packs.
// Reduce with mirror = true.
cudaError_t launch_gram_tridiag(int64_t m, int n, const double* d, const double* e, const double* Z, int64_t ldz,
                                double* P, int* g_out, cudaStream_t s, bool* done);
// K4e: slots of the upper triangle of Z^T Z streaming the column-major Z once by tensor TMA (no
// packed copy).  *done = false (nothing launched) when TMA cannot describe Z: the caller packs and
// takes launch_gram_packed (bitwise the same slots).  Reduce with mirror = true.
cudaError_t launch_gram_euclid_box(int64_t m, int n, const double* Z, int64_t ldz, double* P, int* g_out,
                                   cudaStream_t s, bool* done);
// G (n x n, ldg) = sum_{c<g} P[c] in fixed c order.
cudaError_t launch_gram_reduce(int n, int g, const double* P, double* G, int64_t ldg, cudaStream_t s,
                               bool sym = false,
                               bool mirror = false);
// K3's shared-memory image of R, in this order: the strictly upper 8x8 tiles in DMMA B-fragment
// order, block row by block row (NT(NT-1)/2 * 64 doubles), the reciprocals of the diagonal (NT * 8; 1 beyond n), the
// diagonal tiles (NT * 64; only when the whole image fits in shared memory, NT <= 29).
__host__ __device__ constexpr size_t trsm_img_doubles_rd(int NT, bool rd) {
  return (size_t)NT * (NT - 1) / 2 * 64 + (size_t)NT * 8 + (rd ? (size_t)NT * 64 : 0);
}
__host__ __device__ constexpr bool trsm_img_has_rd(int NT) { return trsm_img_doubles_rd(NT, true) * 8 <= (size_t)SMEM_MAX; }
__host__ __device__ constexpr size_t trsm_img_doubles(int NT) { return trsm_img_doubles_rd(NT, trsm_img_has_rd(NT)); }
// R = chol(G) (upper).  first: *info = 0 on success, info_off + k on breakdown.  !first: does
// nothing if *info != 0 already (an earlier stage broke down), else writes info_off + k on breakdown.
// img != nullptr: also write K3's image of R there (trsm_img_doubles(ceil(n/8)) doubles, 16-byte
// aligned) for a launch_trsm with the same R.
// prog != nullptr (needs img): the OVERLAPPED pair -- the launch_trsm that follows on the same
// stream with the same img and prog starts while this kernel runs and consumes R's image tile
// column by tile column (*prog = columns complete, -1 = do nothing); trsm_overlap_ok(n) must hold.
cudaError_t launch_potrf(int n, const double* G, int64_t ldg, double* R, int64_t ldr, int* info,
                         int info_off, cudaStream_t s, bool first = true, double* img = nullptr,
                         int* prog = nullptr);
bool trsm_overlap_ok(int n);
// G += factor * tr(G) * I (skipped when *info != 0).
cudaError_t launch_shift_diag(int n, double* G, int64_t ldg, double factor, const int* info, cudaStream_t s);
// Q = Z R^{-1}; skipped when info != nullptr && *info != 0.  img: the image launch_potrf wrote for
// this R (each CTA lands it with one bulk copy), or nullptr (each CTA stages it from R).
cudaError_t launch_trsm(int64_t m, int n, const double* Z, int64_t ldz, const double* R, int64_t ldr,
                        double* Q, int64_t ldq, const int* info, cudaStream_t s, const double* img = nullptr,
                        const int* prog = nullptr);
// R = R2 * R1 (upper x upper); skipped when *info != 0.
cudaError_t launch_trmm(int n, const double* R2, const double* R1, double* R, const int* info,
                        cudaStream_t s);

// K6: Householder QR of Z (m x n, ldz) -> Y (m x n, ld m), S (n x n, ld n, positive diagonal);
// X: m x n working matrix (ld m); scratch: hh_scratch_doubles(m, n) doubles, 16-byte aligned.
// One cooperative launch (grid barriers).  hh_supported: the per-CTA row block fits in shared memory.
cudaError_t launch_hhqr(int64_t m, int n, const double* Z, int64_t ldz, double* X, double* Y, double* S,
                        double* scratch, cudaStream_t s);
size_t hh_scratch_doubles(int64_t m, int n);
bool hh_supported(int64_t m, int n);

// Workspace size (bytes) for the Gram of an (m, n) problem on a grid of g CTAs.
int gram_grid(int64_t m);
size_t slots_doubles(int n, int g);

}  // namespace oqr
