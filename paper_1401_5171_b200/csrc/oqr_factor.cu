// oqr_factor.cu -- K2 single-CTA Cholesky, K3 row-wise triangular solve, K5 triangular product.
#include "oqr_internal.cuh"

namespace oqr {

// ------------------------------------------------------------------ K2 --------------------
// R = chol(G), upper, R^T R = G: Algorithm 1 line 3, backward error
// eq:normal:chol.  One CTA of 1024 threads; the upper triangle of G lives
// packed in shared memory (column-major packed index l(l+1)/2 + k, k <= l), padded to a
// multiple of 8 with an identity block (n = 240 -> 231,360 B).  Blocked right-looking with 8x8
// blocks -- the same operations as the unblocked algorithm in a different order:
//   1. warp 0 factors the diagonal block: pivot d = a_pp, breakdown iff !(d > 0) (LAPACK rule,
//      catches NaN; reading R4), r_pp = sqrt(d), row p of the block scaled by 1/r_pp
//      (as LAPACK dpotf2), the block's trailing triangle updated;
//   2. one thread per column l solves the block row: r_pl = (a_pl - sum_{c'<c} r_c'p r_c'l)/r_pp
//      (multiplying by the block's reciprocals);
//   3. the trailing upper triangle is updated tile by tile on the FP64 tensor pipe:
//      A_kl -= R_{j,k}^T R_{j,l} (8x8x8 per tile, mma.m8n8k4 x 2).
// Only the upper triangle of G is read.
__device__ __forceinline__ int pk(int k, int l) { return l * (l + 1) / 2 + k; }

__device__ __forceinline__ void dmma_c(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

#ifdef OQR_EXP_POTRF_TRACE  // experiment build only: per-step clock64 stamps of K2's phases
__device__ long long oqr_k2_trace[4 * 64];
extern "C" int oqr_exp_k2_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, oqr_k2_trace, sizeof(oqr_k2_trace)) == cudaSuccess ? 0 : -1;
}
#define K2_STAMP(i)                                                      \
  do {                                                                   \
    if ((i) < 4 * 64) oqr_k2_trace[(i)] = clock64();                     \
  } while (0)
#else
#define K2_STAMP(i) \
  do {              \
  } while (0)
#endif
#ifdef OQR_EXP_POTRF_TRACE2  // experiment build only: per-(step, warp) stamps of K2's phases
__device__ long long oqr_k2_trace2[32 * 32 * 4];
extern "C" int oqr_exp_k2_trace2(long long* out) {
  return cudaMemcpyFromSymbol(out, oqr_k2_trace2, sizeof(oqr_k2_trace2)) == cudaSuccess ? 0 : -1;
}
#define K2W_STAMP(j, k)                                                         \
  do {                                                                          \
    if (lane == 0 && (j) < 32) oqr_k2_trace2[((j) * 32 + warp) * 4 + (k)] = clock64(); \
  } while (0)
#else
#define K2W_STAMP(j, k) \
  do {                  \
  } while (0)
#endif

__device__ __forceinline__ double lds_f64_k2(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f64_k2(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// K3's image of R keeps the strictly upper 8 x 8 tiles (kt, jt), kt < jt, in BLOCK-ROW-major order:
// tile index trsm_tix = kt (2 NT - kt - 1) / 2 + (jt - kt - 1), so the NT - 1 - kt tiles of block
// row kt -- what the right-looking solve needs once tile kt is solved, and what K2 finalises in
// its step kt -- are contiguous (one bulk copy per block row in the overlapped K2 -> K3 pair).
__host__ __device__ constexpr int trsm_tix(int NT, int kt, int jt) { return kt * (2 * NT - kt - 1) / 2 + (jt - kt - 1); }
__device__ __forceinline__ void trsm_tile_of(int NT, int t, int* kt_out, int* jt_out) {
  const float b = (float)(2 * NT - 1);
  int kt = (int)((b - sqrtf(fmaxf(b * b - 8.0f * (float)t, 0.0f))) * 0.5f);
  if (kt < 0) kt = 0;
  if (kt > NT - 2) kt = NT - 2;
  while (kt > 0 && trsm_tix(NT, kt, kt + 1) > t) --kt;
  while (kt < NT - 2 && trsm_tix(NT, kt + 1, kt + 2) <= t) ++kt;
  *kt_out = kt;
  *jt_out = t - trsm_tix(NT, kt, kt + 1) + kt + 1;
}

// progress word of the overlapped K2 -> K3 pair (gpu-scope release / acquire)
__device__ __forceinline__ void prog_store(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int prog_load(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(1024, 1)
potrf_kernel(int n, const double* __restrict__ G, int64_t ldg, double* __restrict__ R, int64_t ldr,
             int* info, int info_off, bool first, double* __restrict__ img, int* prog) {
  extern __shared__ double S[];
  __shared__ int s_brk;
  const int NT = (n + 7) / 8, NP = NT * 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  // prog != nullptr: K3 runs CONCURRENTLY (launched as a programmatic dependent, session 4): this
  // kernel publishes K3's image of R block row by block row and raises *prog to the number of
  // complete block rows (release); -1 tells K3 to do nothing (breakdown, here or earlier).
  const bool skip = !first && *info != 0;  // an earlier stage already broke down: keep its code
  if (prog != nullptr) {
    if (tid == 0) {
      prog_store(prog, skip ? -1 : 0);
      __threadfence();
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  if (skip) return;
  {  // packed upper triangle of G, padded with an identity block; 8 loads in flight per thread
    const int tot = NP * (NP + 1) / 2;
    for (int e0 = tid; e0 < tot; e0 += 8 * 1024) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * 1024;
        v[u] = 0.0;
        if (e < tot) {
          int l = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
          while (l * (l + 1) / 2 > e) --l;
          while ((l + 1) * (l + 2) / 2 <= e) ++l;
          const int k = e - l * (l + 1) / 2;
          v[u] = (l < n) ? G[(int64_t)l * ldg + k] : (k == l ? 1.0 : 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (e0 + u * 1024 < tot) S[e0 + u * 1024] = v[u];
    }
  }
  if (tid == 0) s_brk = 0;
  __syncthreads();
  if (tid == 0) K2_STAMP(0);
  __shared__ double s_inv[2][8];  // reciprocals of the diagonal blocks' pivots (double-buffered)
  // warp 0: factor diagonal block jb (rows/cols jb*8..+8) in place; row p scaled by 1/r_pp as
  // LAPACK dpotf2 (DSCAL by ONE/AJJ); breakdown (LAPACK rule) recorded in s_brk.
  auto factor_diag = [&](int jb) {
    const int b0 = jb * 8;
    double* inv_out = s_inv[jb & 1];
#ifdef OQR_EXP_POTRF_NOFACTOR  // experiment build only: time of everything but the diagonal factor
    if (lane < 8) inv_out[lane] = 1.0;
    __syncwarp();
    return;
#endif
    // The 8 x 8 block in registers: lane L holds entries (L/8, L%8) and (L/8 + 4, L%8) (upper
    // part meaningful); pivots and scaled rows travel by shuffles -- the same operations, in the
    // same order, as the unblocked LAPACK loop on the block.
    const int ra = lane >> 3, cb = lane & 7;
    double v0 = (cb >= ra) ? S[pk(b0 + ra, b0 + cb)] : 0.0;
    double v1 = (cb >= ra + 4) ? S[pk(b0 + ra + 4, b0 + cb)] : 0.0;
    double dA = 1.0, dB = 1.0;  // the pivots of this lane's rows ra, ra + 4 (for the deferred sqrt)
    int brk = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      // pivot (c, c): lane 9c (c < 4, v0) or 9c - 32 (c >= 4, v1)
      const double d = __shfl_sync(0xffffffffu, c < 4 ? v0 : v1, c < 4 ? 9 * c : 9 * c - 32);
      if (!(d > 0.0)) {  // uniform across the warp
        brk = b0 + c + 1;
        break;
      }
      // The row is scaled by 1/sqrt(d) from one rsqrt (<= 1 ulp; LAPACK dpotf2 scales by
      // ONE/AJJ), which is what the next pivot waits for (inside the gamma_{n+1} of
      // eq:normal:chol).  r_cc = sqrt(d), correctly rounded (IEEE sqrt, SURVEY
      // s8(a) S2 -- the same pivot as the oracle's), is needed by no later operation of the
      // block: it is taken after the loop for all 8 pivots at once (in-order issue would
      // otherwise hold the chain behind each sqrt's own dependent sequence -- session 3).
      const double inv = rsqrt(d);
      // row c: (c, b > c) *= inv; (c, c) keeps d until the deferred sqrt
      if (c < 4) {
        if (ra == c) {
          v0 = cb > c ? v0 * inv : v0;
          dA = d;
        }
      } else {
        if (ra + 4 == c) {
          v1 = cb > c ? v1 * inv : v1;
          dB = d;
        }
      }
      if (lane == 0) inv_out[c] = inv;
      // trailing: (a, b) -= r_ca r_cb for c < a <= b; r_cx lives in lane c*8 + x (mod 32)
      const double rc0 = c < 4 ? v0 : v1;
      const int src = (c & 3) * 8;
      const double ra0 = __shfl_sync(0xffffffffu, rc0, src + ra);        // r_{c, ra}
      const double ra1 = __shfl_sync(0xffffffffu, rc0, src + ((ra + 4) & 7));  // r_{c, ra+4}
      const double rb = __shfl_sync(0xffffffffu, rc0, src + cb);         // r_{c, cb}
      if (ra > c && cb >= ra) v0 -= ra0 * rb;
      if (ra + 4 > c && cb >= ra + 4) v1 -= ra1 * rb;
    }
    if (cb == ra) v0 = sqrt(dA);  // r_cc, c = ra
    if (cb == ra + 4) v1 = sqrt(dB);  // r_cc, c = ra + 4
    if (cb >= ra) S[pk(b0 + ra, b0 + cb)] = v0;
    if (cb >= ra + 4) S[pk(b0 + ra + 4, b0 + cb)] = v1;
    if (brk && lane == 0) s_brk = brk;
    __syncwarp();
  };
  // one 8x8 tile of the trailing update: A_{k0.., l0..} -= R_{j0.., k0..}^T R_{j0.., l0..}
  auto update_tile = [&](int j0, int k0, int l0) {
#ifdef OQR_EXP_POTRF_NOTRAIL  // experiment build only: no trailing update
    return;
#endif
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int p = j0 + 4 * h + (lane & 3);
      dmma_c(acc, S[pk(p, k0 + (lane >> 2))], S[pk(p, l0 + (lane >> 2))]);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int k = k0 + (lane >> 2), l = l0 + 2 * (lane & 3) + e;
      if (k <= l) S[pk(k, l)] -= acc[e];
    }
  };
  if (warp == 0) factor_diag(0);
#ifdef OQR_EXP_POTRF_LOADSTORE  // experiment build only: launch + staging of G + write of R
  for (int j = 0; j < 0; ++j) {
#else
  for (int j = 0; j < NT; ++j) {
#endif
    const int j0 = j * 8;
    __syncthreads();  // diagonal block j factored (look-ahead by warp 0)
    if (tid == 0) K2_STAMP(4 + 3 * j);
    K2W_STAMP(j, 0);
    if (s_brk) break;
    const double* inv = s_inv[j & 1];
    // 2. block row j: columns l >= j0 + 8 (one thread each), forward substitution with R_jj^T
    for (int l = j0 + 8 + tid; l < NP; l += blockDim.x) {
      double x[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = S[pk(j0 + c, l)];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        x[c] *= inv[c];
#pragma unroll
        for (int c2 = c + 1; c2 < 8; ++c2) x[c2] -= S[pk(j0 + c, j0 + c2)] * x[c];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) S[pk(j0 + c, l)] = x[c];
    }
    K2W_STAMP(j, 1);
    __syncthreads();
    if (tid == 0) K2_STAMP(5 + 3 * j);
    K2W_STAMP(j, 2);
    // 3. trailing update on DMMA, tiles (kt, lt), j < kt <= lt < NT.  Look-ahead: warp 0 updates
    //    the next diagonal tile (t = 0) and factors it at once; warps 1.. take the other tiles.
    const int rem = NT - j - 1;
    const int ntiles = rem * (rem + 1) / 2;
    if (warp == 0) {
      if (rem > 0) {
        update_tile(j0, j0 + 8, j0 + 8);
        __syncwarp();
        factor_diag(j + 1);
        if (lane == 0) K2_STAMP(6 + 3 * j);
      }
    } else if (warp == 4 && prog != nullptr) {
      // Block row j of R and diagonal block j are final: publish their part of K3's image (the
      // same values as the end-of-kernel image below) and raise the progress word.  Warp 4 idles
      // in this phase anyway (sub-partition 0 is kept free of DMMAs for warp 0's pivot chain).
      const int ntri = NT * (NT - 1) / 2 * 64;
      for (int jt = j + 1; jt < NT; ++jt) {
        double* dst = img + (size_t)trsm_tix(NT, j, jt) * 64;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          dst[h * 32 + lane] = S[pk(j0 + 4 * h + (lane & 3), jt * 8 + (lane >> 2))];
      }
      if (lane < 8) img[ntri + j0 + lane] = (j0 + lane < n) ? 1.0 / S[pk(j0 + lane, j0 + lane)] : 1.0;
      if (trsm_img_has_rd(NT)) {
        double* Rd = img + ntri + NT * 8 + j * 64;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = h * 32 + lane, c = e >> 3, c2 = e & 7;
          Rd[e] = c <= c2 ? S[pk(j0 + c, j0 + c2)] : 0.0;
        }
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) prog_store(prog, j + 1);
    } else if (warp & 3) {
      // the trailing tiles go to the warps of sub-partitions 1-3 only (warp w runs on sub-partition
      // w % 4): DMMA and DFMA share the FP64 pipe, and warp 0's pivot chain (the critical path)
      // would otherwise queue behind its sub-partition's DMMAs (K2 phase trace,
      // tools/exp/k2_trace.py: a diagonal factor took up to 9.5k clocks under a full trailing
      // update, 4.2k without; K2 at n = 200: 100.6 -> 96.6 us)
      // Row strips: the trailing tiles in row-major order (tile row kt = 0..rem-1 local, columns
      // lt = kt..rem-1; tile 0 = the next diagonal tile is warp 0's), one contiguous run per warp,
      // so a warp loads the A fragments R_{j,kt} once per tile row it touches.  The update is
      // shared-memory bound: the per-warp phase trace (tools/exp/k2_trace2.py) put the step-0
      // trailing update at ~11.7k clocks, and the packed-triangle accesses of a tile cost 36
      // wavefronts (A 10, B 10, C read+write 16; 16 conflict-free) -- 10.8k for its 300 tiles.
      // The operations per tile are update_tile's (the same two DMMAs from zero, the same
      // subtractions), on shared-window offsets.
      const int widx = warp - (warp >> 2) - 1, nwork = nwarp - (nwarp >> 2);
      const int T1 = ntiles - 1;  // tiles other than the next diagonal one
      const int t0 = 1 + (widx * T1) / nwork, t1 = 1 + ((widx + 1) * T1) / nwork;
      if (t0 < t1) {
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(S);
        const int c8 = lane >> 2, r4 = lane & 3;
        int kt = 0, rs = 0;  // rs: row-major index of tile (kt, kt)
        while (t0 >= rs + (rem - kt)) {
          rs += rem - kt;
          ++kt;
        }
        int lt = kt + (t0 - rs);
        int ka = (j + 1 + kt) * 8 + c8;  // output row k = A-fragment column
        uint32_t ta = sb + 4u * (uint32_t)(ka * (ka + 1)) + 8u * (uint32_t)(j0 + r4);
        double a0 = lds_f64_k2(ta), a1 = lds_f64_k2(ta + 32u);
        for (int t = t0;;) {
          const int kb = (j + 1 + lt) * 8 + c8;  // B-fragment column
          const uint32_t tb = sb + 4u * (uint32_t)(kb * (kb + 1)) + 8u * (uint32_t)(j0 + r4);
          double acc[2] = {0.0, 0.0};
          dmma_c(acc, a0, lds_f64_k2(tb));
          dmma_c(acc, a1, lds_f64_k2(tb + 32u));
          const int l = (j + 1 + lt) * 8 + 2 * r4;
          const uint32_t tc = sb + 4u * (uint32_t)(l * (l + 1)) + 8u * (uint32_t)ka;  // (ka, l)
          if (ka <= l) sts_f64_k2(tc, lds_f64_k2(tc) - acc[0]);
          if (ka <= l + 1) {
            const uint32_t tc1 = tc + 8u * (uint32_t)(l + 1);  // (ka, l + 1)
            sts_f64_k2(tc1, lds_f64_k2(tc1) - acc[1]);
          }
          if (++t == t1) break;
          if (++lt == rem) {  // next tile row
            ++kt;
            lt = kt;
            ka += 8;
            ta = sb + 4u * (uint32_t)(ka * (ka + 1)) + 8u * (uint32_t)(j0 + r4);
            a0 = lds_f64_k2(ta);
            a1 = lds_f64_k2(ta + 32u);
          }
        }
      }
    }
    K2W_STAMP(j, 3);
  }
  if (s_brk) {
    if (tid == 0) {
      *info = info_off + s_brk;
      if (prog != nullptr) prog_store(prog, -1);
    }
    return;
  }
  if (tid == 0) K2_STAMP(1);
  for (int l = warp; l < n; l += nwarp)
    for (int k = lane; k < n; k += 32) R[(int64_t)l * ldr + k] = (k <= l) ? S[pk(k, l)] : 0.0;
  if (img != nullptr && prog == nullptr) {
    // K3's shared-memory image of R (trsm_img_*): the same values K3's prologue would stage from
    // R -- off-diagonal tiles in B-fragment order, the reciprocals of the diagonal, the diagonal
    // tiles -- written once here, so that every K3 CTA lands it with one bulk copy
    const int ntri = NT * (NT - 1) / 2 * 64;
    for (int e = tid; e < ntri; e += blockDim.x) {
      int kt, jt;
      trsm_tile_of(NT, e >> 6, &kt, &jt);
      const int ln = e & 31, h = (e >> 5) & 1;
      const int k = kt * 8 + 4 * h + (ln & 3), col = jt * 8 + (ln >> 2);
      img[e] = col < n ? S[pk(k, col)] : 0.0;
    }
    double* Ri = img + ntri;
    for (int e = tid; e < NT * 8; e += blockDim.x) Ri[e] = (e < n) ? 1.0 / S[pk(e, e)] : 1.0;
    if (trsm_img_has_rd(NT)) {
      double* Rd = Ri + NT * 8;
      for (int e = tid; e < NT * 64; e += blockDim.x) {
        const int jt = e >> 6, c = (e >> 3) & 7, c2 = e & 7;
        const int r = jt * 8 + c, col = jt * 8 + c2;
        Rd[e] = c <= c2 ? (col < n ? S[pk(r, col)] : (c == c2 ? 1.0 : 0.0)) : 0.0;
      }
    }
  }
  if (tid == 0 && first) *info = 0;
  if (tid == 0) K2_STAMP(2);
}

cudaError_t launch_potrf(int n, const double* G, int64_t ldg, double* R, int64_t ldr, int* info,
                         int info_off, cudaStream_t s, bool first, double* img, int* prog) {
  const int NP = 8 * ((n + 7) / 8);
  const size_t bytes = (size_t)NP * (NP + 1) / 2 * sizeof(double);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(potrf_kernel), SMEM_MAX - 1024);
  if (e != cudaSuccess) return e;
  timing_begin(s, OQR_TIMING_K2);
  potrf_kernel<<<1, 1024, bytes, s>>>(n, G, ldg, R, ldr, info, info_off, first, img, prog);
  note_launch();
  e = cudaGetLastError();
  timing_end(s);
  return e;
}

// ------------------------------------------------------------------ shift -----------------
// G += s I with s = factor * tr(G), tr summed in ascending order (shifted CholeskyQR, reading
// R21: factor = 11 (m n + n (n + 1)) u, tr(G) = ||Z||_F^2 bounds ||Z||_2^2 from above).
__global__ void shift_diag_kernel(int n, double* G, int64_t ldg, double factor, const int* info) {
  __shared__ double s_shift;
  if (info != nullptr && *info != 0) return;
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int i = 0; i < n; ++i) tr += G[(int64_t)i * ldg + i];
    s_shift = factor * tr;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) G[(int64_t)i * ldg + i] += s_shift;
}

cudaError_t launch_shift_diag(int n, double* G, int64_t ldg, double factor, const int* info, cudaStream_t s) {
  shift_diag_kernel<<<1, 256, 0, s>>>(n, G, ldg, factor, info);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K3 --------------------
// Q = Z R^{-1}: Algorithm 1 line 4 as the row-wise substitution whose backward
// error is stated at PAPER.md:197-198:  q_ij = (z_ij - sum_{k<j} q_ik r_kj) / r_jj.
// One warp per 8 rows; columns in tiles of 8 (jt).  Right-looking: as soon as tile kt of the
// row block is solved, its contributions q_kt R[kt, jt] to every later tile jt are added on the
// FP64 tensor pipe (mma.m8n8k4) into per-tile accumulators S[jt] held in registers, so when tile
// jt is reached only q_{jt-1}'s two DMMAs stand between it and its diagonal solve, and the
// updates of the later tiles overlap that solve; then the 8 x 8 diagonal block is solved by
// plain substitution: column c of the tile is (z - s - sum_{c'<c} q_c' r_c'c) / r_cc.
// (Left-looking with the finished q's kept as A-fragments measured 0.20 / 0.38 ms at
// m = 4e4 / 1e5, n = 200; this form with LDS-addressed R: 0.15 / 0.28 ms.)
// This is the substitution formula with the sum split into pieces (a summation order), never an
// explicit inverse, so the componentwise bound |dR^i| <= gamma_n |R| still holds.
__device__ __forceinline__ void dmma_f(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// R is staged once per (persistent) CTA in shared memory in DMMA B-fragment order:
//   Rt[(trsm_tix(NT, kt, jt)*2 + h)*32 + lane] = R[kt*8 + 4h + lane%4, jt*8 + lane/4]   (kt < jt;
//   tiles in block-row-major order, trsm_tix above)
//   Rd[(jt*8 + c)*8 + c2] = R[jt*8 + c, jt*8 + c2]  (diagonal tiles, upper part)
//   Ri[jt*8 + c] = 1 / R[jt*8 + c, jt*8 + c]       (1 beyond n)
// so every fragment load is 256 consecutive bytes.  At NT = 30 Rd does not fit as well (238 KB):
// the diagonal tiles are then read from global memory (L1/L2).
// Diagonal 8 x 8 block: the row's 8 partial values are gathered into all 4 lanes of the row's
// quad (8 independent shuffles) and each lane solves the row redundantly with an FMA chain,
// q_c = (t_c - sum_{c'<c} q_c' r_c'c) * (1 / r_cc): no shuffles and no divisions on the chain.
// (Multiplying by the rounded reciprocal adds one rounding per entry: the row-wise backward error
// becomes |dR^i| <= gamma_{n+1} |R|, the bound the parity gates use.)
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
// v[q] for the lane's quad position q (0..3) by three predicated selects: written as a C
// ternary chain, ptxas turned the choice into divergent branches with a reconvergence barrier
// (BSSY/BSYNC) around every A-fragment and Q selection of every tile (cuobjdump; ncu
// "branch_resolving" 10% of K3's stall samples)
__device__ __forceinline__ double sel4(int q, double v0, double v1, double v2, double v3) {
  double r;
  asm("{\n\t.reg .pred p1, p2, p3;\n\t"
      "setp.eq.s32 p1, %5, 1;\n\tsetp.eq.s32 p2, %5, 2;\n\tsetp.eq.s32 p3, %5, 3;\n\t"
      "selp.f64 %0, %2, %1, p1;\n\tselp.f64 %0, %3, %0, p2;\n\tselp.f64 %0, %4, %0, p3;\n\t}"
      : "=&d"(r)
      : "d"(v0), "d"(v1), "d"(v2), "d"(v3), "r"(q));
  return r;
}

// Overlapped K2 -> K3 (session 4): before tile jt of a warp's first row block.  Warp 0 polls K2's
// progress word and issues the bulk copies of every newly complete block row c of the image (its
// NT - 1 - c off-diagonal tiles, contiguous; its 8 reciprocals; its diagonal tile) onto colbar[c];
// then every warp waits for colbar[jt]: solving tile jt and applying q_jt to the later tiles needs
// exactly block row jt.  Returns the new `issued`, or NT + 1 when the solve
// must be abandoned (K2 broke down or was skipped: *prog < 0; or -- a safety net, never seen -- no
// progress for ~2 s).
__device__ __noinline__ int trsm_follow_issue(const int* prog, const double* img, double* rsm, uint64_t* colbar,
                                              int* s_abort, int NT, int jt, int lane, int issued) {
  // warp 0 only (out of line: it runs a handful of times per CTA, and inlined at every tile it
  // made the unrolled body miss in the instruction cache -- ncu no_inst 4% -> 11%)
  int v = 0;
  if (lane == 0) {
    const long long t0 = clock64();
    for (;;) {
      v = prog_load(prog);
      if (v < 0 || v > jt) break;
      if (clock64() - t0 > 4000000000LL) {
        v = -1;
        break;
      }
      __nanosleep(64);
    }
    if (v < 0) {
      *reinterpret_cast<volatile int*>(s_abort) = 1;
    } else {
      asm volatile("fence.proxy.async;" ::: "memory");  // K2's generic-proxy writes before the async-proxy reads
      const size_t ntri = (size_t)NT * (NT - 1) / 2 * 64;
      for (int c = issued; c < v; ++c) {
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&colbar[c]);
        const uint32_t rowb = (uint32_t)(NT - 1 - c) * 512u;  // block row c: its NT - 1 - c off-diagonal tiles
        const uint32_t bytes = rowb + 64u + 512u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        const size_t o_t = (size_t)trsm_tix(NT, c, c + 1) * 64, o_i = ntri + (size_t)c * 8, o_d = ntri + (size_t)NT * 8 + (size_t)c * 64;
        if (rowb > 0)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(rsm + o_t)),
                       "l"(img + o_t), "r"(rowb), "r"(bar)
                       : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(rsm + o_i)),
                     "l"(img + o_i), "r"(64u), "r"(bar)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(rsm + o_d)),
                     "l"(img + o_d), "r"(512u), "r"(bar)
                     : "memory");
      }
    }
  }
  v = __shfl_sync(0xffffffffu, v, 0);
  return v > issued ? v : issued;
}
__device__ __forceinline__ int trsm_follow(const int* prog, const double* img, double* rsm, uint64_t* colbar,
                                           int* s_abort, int NT, int jt, int warp, int lane, int issued) {
  if (warp == 0 && issued <= jt) issued = trsm_follow_issue(prog, img, rsm, colbar, s_abort, NT, jt, lane, issued);
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&colbar[jt]);
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar)
        : "memory");
    if (ok) return issued;
    if (*reinterpret_cast<volatile int*>(s_abort)) return NT + 1;
  }
}

// Warps per CTA: as many as the per-tile register accumulators allow without spills (ptxas:
// 16 warps <= 128 registers up to NT = 16, 12 warps <= 168 up to NT = 29, else 8).
#ifndef OQR_EXP_TRSM_T16
#define OQR_EXP_TRSM_T16 16
#endif
#ifdef OQR_EXP_TRSM_THREADS  // experiment build only (tools/exp/build_k3d.sh)
__host__ __device__ constexpr int trsm_threads(int) { return OQR_EXP_TRSM_THREADS; }
#else
__host__ __device__ constexpr int trsm_threads(int NT) { return NT <= OQR_EXP_TRSM_T16 ? 512 : (NT <= 29 ? 384 : 256); }
#endif

template <int NT>
constexpr size_t trsm_smem_doubles(bool with_rd) {
  return (size_t)NT * (NT - 1) / 2 * 64 + (size_t)NT * 8 + (with_rd ? (size_t)NT * 64 : 0);
}

template <int NT, bool SMEM_RD>
__global__ void __launch_bounds__(trsm_threads(NT), 1)
trsm_dmma_kernel(int64_t m, int n, const double* Z, int64_t ldz,  // Z may alias Q (in place)
                 const double* __restrict__ R, int64_t ldr, double* Q, int64_t ldq, const int* info,
                 const double* __restrict__ img, const int* prog) {
  // prog != nullptr (SMEM_RD only): this grid runs concurrently with the K2 that produces R
  // (programmatic dependent launch, session 4).  K2 raises *prog to the number of complete block
  // rows of the image (-1: breakdown, do nothing); warp 0 lands each new block row's part of the
  // image with bulk copies on that row's mbarrier, and every warp waits for block row jt's
  // barrier before tile jt.  info is not consulted in that mode (K2 writes it at its end).
  if (prog == nullptr && info != nullptr && *info != 0) return;
  extern __shared__ __align__(16) double rsm[];
  double* const Rt_base = rsm;
  double* const Ri_base = rsm + (size_t)NT * (NT - 1) / 2 * 64;
  double* const Rd_base = Ri_base + (size_t)NT * 8;
  __shared__ __align__(8) uint64_t colbar[NT];
  __shared__ int s_abort;
  if (prog != nullptr) {
    if (threadIdx.x == 0) {
      s_abort = 0;
      for (int c = 0; c < NT; ++c)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&colbar[c])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  } else if (img != nullptr) {
    // K2 wrote this CTA's shared-memory image of R: one bulk copy (SASS UBLKCP) instead of
    // ~20k scattered L2 loads per CTA (the staging loop below: ~10% of K3 at c3)
    __shared__ __align__(8) uint64_t bar;
    constexpr uint32_t BYTES = (uint32_t)(trsm_img_doubles_rd(NT, SMEM_RD) * sizeof(double));
    const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(BYTES) : "memory");
      constexpr uint32_t CH = 32768;
      for (uint32_t o = 0; o < BYTES; o += CH) {
        const uint32_t len = BYTES - o < CH ? BYTES - o : CH;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(rsm) + o),
            "l"(reinterpret_cast<const char*>(img) + o), "r"(len), "r"(sbar)
            : "memory");
      }
    }
    __syncthreads();  // the barrier is initialised before anyone polls it
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(sbar)
          : "memory");
  } else {
    // staged with 8 independent loads in flight per thread (a plain loop waits one L2 round trip
    // per element: ~7% of K3 at m = 1e5)
    constexpr int TOT = NT * (NT - 1) / 2 * 64;
    for (int e0 = threadIdx.x; e0 < TOT; e0 += 8 * trsm_threads(NT)) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * trsm_threads(NT);
        v[u] = 0.0;
        if (e < TOT) {
          int kt, jt;  // tile e / 64 of the block-row-major order (trsm_tix)
          trsm_tile_of(NT, e >> 6, &kt, &jt);
#ifdef OQR_EXP_TRSM_LDS128
          const int ln = (e >> 1) & 31, h = e & 1;
#else
          const int ln = e & 31, h = (e >> 5) & 1;
#endif
          const int k = kt * 8 + 4 * h + (ln & 3), col = jt * 8 + (ln >> 2);
          if (col < n) v[u] = R[(int64_t)col * ldr + k];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * trsm_threads(NT);
        if (e < TOT) Rt_base[e] = v[u];
      }
    }
    if (SMEM_RD) {
      for (int e = threadIdx.x; e < NT * 64; e += blockDim.x) {
        const int jt = e >> 6, c = (e >> 3) & 7, c2 = e & 7;
        const int r = jt * 8 + c, col = jt * 8 + c2;
        double v = 0.0;
        if (c <= c2) v = (col < n) ? R[(int64_t)col * ldr + r] : (c == c2 ? 1.0 : 0.0);
        Rd_base[e] = v;
      }
    }
    for (int e = threadIdx.x; e < NT * 8; e += blockDim.x)
      Ri_base[e] = (e < n) ? 1.0 / R[(int64_t)e * ldr + e] : 1.0;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int q4 = lane & 3;                // quad position: C columns 2*q4, 2*q4 + 1
  const int gbase = lane & ~3;            // first lane of this row's quad
  bool follow = prog != nullptr;          // first row block of the overlapped mode: columns arrive
  int issued = 0;                         // warp 0: image columns whose copies are in flight
#pragma unroll 1
#ifndef OQR_EXP_TRSM_MAP
#define OQR_EXP_TRSM_MAP 1
#endif
  // First 8-row block of this warp.  1 (default) = warp-major: block w * gridDim + cta, so the last,
  // partly filled round of the persistent loop spreads one warp per SM over all SMs instead of
  // filling a few CTAs (a lone warp runs its block ~2x faster than one of twelve sharing an SM):
  // m = 1e5: n = 200 0.257 -> 0.248 ms, n = 100 0.091 -> 0.086; m = 2e4, n = 100 0.036 -> 0.029
  // (session 4; bitwise the same Q).  0 = CTA-major (adjacent blocks in one CTA), 2 = warp-pair-major
  // (as 1 with adjacent pairs, measured equal to 1): experiment builds.
  const int64_t first_block = OQR_EXP_TRSM_MAP == 1   ? (int64_t)warp * gridDim.x + blockIdx.x
                              : OQR_EXP_TRSM_MAP == 2 ? ((int64_t)(warp >> 1) * gridDim.x + blockIdx.x) * 2 + (warp & 1)
                                                      : (int64_t)blockIdx.x * nw + warp;
  for (int64_t r0 = first_block * 8; r0 < m; r0 += (int64_t)gridDim.x * nw * 8) {
    const int64_t row = r0 + (lane >> 2);
    const bool row_ok = row < m;
    // opaque per-iteration copies: stop the compiler from hoisting loop-invariant R loads and
    // per-column offsets/predicates out of the row loop into hundreds of registers
    // (shared-window addresses, so the loads stay LDS: a generic pointer made opaque would turn
    // them into generic loads with long-scoreboard latency)
    uint32_t Rt = (uint32_t)__cvta_generic_to_shared(Rt_base);
    uint32_t Rd = (uint32_t)__cvta_generic_to_shared(Rd_base);
    uint32_t Ri = (uint32_t)__cvta_generic_to_shared(Ri_base);
    int64_t ldz_l = ldz, ldq_l = ldq;
    int n_l = n;
    const double* Rg = R;
    asm volatile("" : "+r"(Rt), "+r"(Rd), "+r"(Ri), "+l"(ldz_l), "+l"(ldq_l), "+r"(n_l), "+l"(Rg));
    // Right-looking: S[jt] accumulates sum_{kt<jt} q_kt R[kt, jt] (C layout) as soon as each q_kt
    // is known, so when tile jt is reached only q_{jt-1}'s two DMMAs are still on its critical
    // path; the updates of the later tiles overlap the next diagonal solves.
    double S[NT][2];
#pragma unroll
    for (int jt = 0; jt < NT; ++jt) S[jt][0] = S[jt][1] = 0.0;
    // Z of tiles jt+1, jt+2 is loaded before tile jt's Q stores: different columns, so this is
    // safe even in place (Q == Z); the compiler must assume Q aliases Z and would not reorder them.
#ifndef OQR_EXP_TRSM_PD
#define OQR_EXP_TRSM_PD 2
#endif
    constexpr int PD = OQR_EXP_TRSM_PD;  // Z prefetch distance in tiles
    double zq[PD][2];
    // Running pointers instead of col * ld + row per access: a smaller unrolled body (-9% SASS), and
    // the size of this body is itself a cost (instruction cache): m = 1e5, n = 200 0.225 -> 0.217 ms,
    // n = 232 0.305 -> 0.287 (session 4; bitwise the same Q).  OQR_EXP_TRSM_NOPTR: the indexed form.
#if !defined(OQR_EXP_TRSM_NOPTR) && !defined(OQR_EXP_TRSM_PTR)
#define OQR_EXP_TRSM_PTR 1
#endif
#ifndef OQR_EXP_TRSM_PF
#define OQR_EXP_TRSM_PF 8
#endif
#ifdef OQR_EXP_TRSM_PTR
    const double* zp = Z + (int64_t)(2 * q4) * ldz_l + row;  // (row, column 2 q4) of the tile being loaded
    double* qp = Q + (int64_t)(2 * q4) * ldq_l + row;        // ... of the tile being stored
    const int64_t zstep = 8 * ldz_l, qstep = 8 * ldq_l;
#endif
#pragma unroll
    for (int d = 0; d < PD; ++d) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = d * 8 + 2 * q4 + e;
#ifdef OQR_EXP_TRSM_NOLDG  // timing-only diagnostic build: no Z loads (wrong Q)
        zq[d][e] = (double)(col + lane);
#elif defined(OQR_EXP_TRSM_PTR)
        zq[d][e] = (row_ok && (d < NT - 1 || col < n_l)) ? zp[e ? ldz_l : 0] : 0.0;
#else
        zq[d][e] = (row_ok && col < n_l) ? Z[(int64_t)col * ldz_l + row] : 0.0;
#endif
      }
#ifdef OQR_EXP_TRSM_PTR
      zp += zstep;
#endif
    }
#pragma unroll
    for (int jt = 0; jt < NT; ++jt) {
      const double zc0 = zq[jt % PD][0], zc1 = zq[jt % PD][1];
      if (jt + PD < NT) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = (jt + PD) * 8 + 2 * q4 + e;
#ifdef OQR_EXP_TRSM_NOLDG
          zq[jt % PD][e] = (double)(col + lane);
#elif defined(OQR_EXP_TRSM_PTR)
          zq[jt % PD][e] = (row_ok && (jt + PD < NT - 1 || col < n_l)) ? zp[e ? ldz_l : 0] : 0.0;
#else
          zq[jt % PD][e] = (row_ok && col < n_l) ? Z[(int64_t)col * ldz_l + row] : 0.0;
#endif
        }
#ifdef OQR_EXP_TRSM_PTR
        zp += zstep;
#endif
      }
      // L2 prefetch of this warp's Z chunk (8 columns x 64 B) OQR_EXP_TRSM_PF tiles ahead, running on
      // into its next row block: costs no registers (a register prefetch distance of 3 or 6 tiles was
      // slower: spills) and takes 2-5% off K3 (session 4: ncu put 22% of K3's stall samples on the
      // DADD that consumes a tile's Z values, long scoreboard; distance 4-16 and L1/L2 measured equal)
#if OQR_EXP_TRSM_PF > 0
      {
        const int tp = (jt + OQR_EXP_TRSM_PF) % NT;
        const int64_t rp = (jt + OQR_EXP_TRSM_PF < NT) ? r0 : r0 + (int64_t)gridDim.x * nw * 8;
        const int colp = tp * 8 + (lane & 7);
        if (lane < 8 && colp < n_l && rp < m) {
          const double* ap = Z + (int64_t)colp * ldz_l + rp;
#ifdef OQR_EXP_TRSM_PFL1
          asm volatile("prefetch.global.L1 [%0];" ::"l"(ap));
#else
          asm volatile("prefetch.global.L2 [%0];" ::"l"(ap));
#endif
        }
      }
#endif
      if (SMEM_RD && follow) {
        issued = trsm_follow(prog, img, rsm, colbar, &s_abort, NT, jt, warp, lane, issued);
        // Abandoned (K2 broke down or was skipped): stop following and run on over whatever the
        // image holds -- Q is unspecified on a nonzero status (include/oqr.h) -- rather than leave:
        // a CTA must not exit while bulk copies into its shared memory may still be in flight.
        if (issued > NT) follow = false;
        // the R loads below are plain (non-volatile) asm: tie their addresses to this point so that
        // none of tile jt's is scheduled before its column has landed
        asm volatile("" : "+r"(Rt), "+r"(Rd), "+r"(Ri) : : "memory");
      }
      double t0 = zc0 - S[jt][0];
      double t1 = zc1 - S[jt][1];
      // gather the row's 8 values into every lane of its quad
      double tt[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        tt[2 * q] = __shfl_sync(0xffffffffu, t0, gbase | q);
        tt[2 * q + 1] = __shfl_sync(0xffffffffu, t1, gbase | q);
      }
      // diagonal 8 x 8 block: right-looking substitution, redundantly in the 4 lanes of the quad
      double qv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int dc = jt * 8 + c;
#if defined(OQR_EXP_TRSM_NOCHAIN) || defined(OQR_EXP_TRSM_FMAONLY)  // timing-only diagnostic builds (wrong Q)
        qv[c] = tt[c];
        (void)dc;
#else
        qv[c] = tt[c] * lds_f64(Ri + 8u * dc);
#endif
#ifndef OQR_EXP_TRSM_NOCHAIN
#pragma unroll
        for (int c2 = c + 1; c2 < 8; ++c2) {
          double rcj;
          if (SMEM_RD) rcj = lds_f64(Rd + 8u * ((jt * 8 + c) * 8 + c2));
          else rcj = (jt * 8 + c2) < n_l ? Rg[(int64_t)(jt * 8 + c2) * ldr + dc] : 0.0;
          tt[c2] = fma(-qv[c], rcj, tt[c2]);
        }
#endif
      }
      // the tile's A fragments (row lane/4, cols 4h + lane%4), then the updates of every later
      // tile, the next one first
      const double a0 = sel4(q4, qv[0], qv[1], qv[2], qv[3]);
      const double a1 = sel4(q4, qv[4], qv[5], qv[6], qv[7]);
#ifdef OQR_EXP_TRSM_LDS128  // experiment build: both halves' B values in one LDS.128 (h-interleaved Rt)
#pragma unroll
      for (int j2 = jt + 1; j2 < NT; ++j2) {
        double b0, b1;
        asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(b0), "=d"(b1) : "r"(Rt + 16u * (trsm_tix(NT, jt, j2) * 32 + lane)));
        dmma_f(S[j2], a0, b0);
        dmma_f(S[j2], a1, b1);
      }
#else
      // all first-half k-steps, then all second-half ones: consecutive DMMAs are independent
#ifdef OQR_EXP_TRSM_NOBATCH  // timing-only diagnostic build: only the next tile's two DMMAs (wrong Q)
      const int JEND = (jt + 2 < NT) ? jt + 2 : NT;
#else
      const int JEND = NT;
#endif
#pragma unroll
      for (int j2 = jt + 1; j2 < JEND; ++j2)
        dmma_f(S[j2], a0, lds_f64(Rt + 8u * (trsm_tix(NT, jt, j2) * 64 + lane)));
#pragma unroll
      for (int j2 = jt + 1; j2 < JEND; ++j2)
        dmma_f(S[j2], a1, lds_f64(Rt + 8u * (trsm_tix(NT, jt, j2) * 64 + 32 + lane)));
#endif
      // this lane's two C entries -> Q
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = jt * 8 + 2 * q4 + e;
        const double qe = sel4(q4, qv[e], qv[2 + e], qv[4 + e], qv[6 + e]);
#ifdef OQR_EXP_TRSM_NOSTG  // timing-only diagnostic build: no Q stores except a never-true one
        if (row_ok && col < n_l && qe == 1.2345e300) Q[(int64_t)col * ldq_l + row] = qe;
#elif defined(OQR_EXP_TRSM_PTR)
        if (row_ok && (jt < NT - 1 || col < n_l)) qp[e ? ldq_l : 0] = qe;
#else
        if (row_ok && col < n_l) Q[(int64_t)col * ldq_l + row] = qe;
#endif
      }
#ifdef OQR_EXP_TRSM_PTR
      qp += qstep;
#endif
    }
    follow = false;
  }
}

// ---- K3, warp-pair form (experiment build OQR_EXP_TRSM_PAIR; measured slower) ----------------
// The same right-looking substitution (the same pieces of the same sums) with the per-tile
// accumulators of one 8-row block split over a PAIR of warps:
// warp v of the pair owns the tiles jt with jt % 2 == v (half the registers: twice the warps per
// SM to hide the diagonal solves' latency).  Tile t's owner solves it, publishes its DMMA
// A-fragments (2 doubles per lane) in a shared-memory slot and arrives on the pair's mbarrier for
// t's parity; the partner waits, applies q_t to ITS next tile t+1 at once with DFMA (the only work
// on the critical path, kept off the tensor pipe whose queue holds the other warps' bulk DMMAs),
// solves t+1 and publishes it, and only then applies q_t to its later tiles (deferred, DMMA)
// together with q_{t+1} -- so each warp's bulk DMMA updates overlap the partner's solve.
// Slots are reused every second tile of a parity: the owner of t+2 waits for q_{t+1}, which its
// partner publishes only after reading slot t.
constexpr int TP_GROUPS = 8;  // warp pairs per CTA (16 warps)
#ifndef OQR_EXP_TP_PD
#define OQR_EXP_TP_PD 4
#endif
constexpr int TP_PD = OQR_EXP_TP_PD;  // Z prefetch distance in own tiles

__device__ __forceinline__ uint32_t tp_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tp_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tp_smem(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tp_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tp_smem(bar)) : "memory");
}
__device__ __forceinline__ void tp_mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(tp_smem(bar)), "r"(parity)
        : "memory");
  }
}

template <int NT>
constexpr size_t trsm_pair_smem_bytes() {
  return trsm_smem_doubles<NT>(true) * sizeof(double) + (size_t)TP_GROUPS * 2 * 64 * sizeof(double) +
         (size_t)TP_GROUPS * 2 * sizeof(uint64_t);
}

template <int NT>
__global__ void __launch_bounds__(TP_GROUPS * 64, 1)
trsm_pair_kernel(int64_t m, int n, const double* Z, int64_t ldz,  // Z may alias Q (in place)
                 const double* __restrict__ R, int64_t ldr, double* Q, int64_t ldq, const int* info) {
  if (info != nullptr && *info != 0) return;
  constexpr int H = (NT + 1) / 2;  // tiles per warp (upper bound)
  extern __shared__ __align__(16) double rsm[];
  double* const Rt_base = rsm;
  double* const Ri_base = rsm + (size_t)NT * (NT - 1) / 2 * 64;
  double* const Rd_base = Ri_base + (size_t)NT * 8;
  double* const slots = Rd_base + (size_t)NT * 64;                       // [TP_GROUPS][2][2][32]
  uint64_t* const bars = reinterpret_cast<uint64_t*>(slots + TP_GROUPS * 2 * 64);  // [TP_GROUPS][2]
  {
    constexpr int TOT = NT * (NT - 1) / 2 * 64;
    for (int e0 = threadIdx.x; e0 < TOT; e0 += 8 * TP_GROUPS * 64) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * TP_GROUPS * 64;
        v[u] = 0.0;
        if (e < TOT) {
          const int t = e >> 6;
          int jt = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)t)) * 0.5f);
          while (jt * (jt - 1) / 2 > t) --jt;
          while ((jt + 1) * jt / 2 <= t) ++jt;
          const int kt = t - jt * (jt - 1) / 2, ln = e & 31, h = (e >> 5) & 1;
          const int k = kt * 8 + 4 * h + (ln & 3), col = jt * 8 + (ln >> 2);
          if (col < n) v[u] = R[(int64_t)col * ldr + k];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * TP_GROUPS * 64;
        if (e < TOT) Rt_base[e] = v[u];
      }
    }
    for (int e = threadIdx.x; e < NT * 64; e += blockDim.x) {
      const int jt = e >> 6, c = (e >> 3) & 7, c2 = e & 7;
      const int r = jt * 8 + c, col = jt * 8 + c2;
      double v = 0.0;
      if (c <= c2) v = (col < n) ? R[(int64_t)col * ldr + r] : (c == c2 ? 1.0 : 0.0);
      Rd_base[e] = v;
    }
    for (int e = threadIdx.x; e < NT * 8; e += blockDim.x)
      Ri_base[e] = (e < n) ? 1.0 / R[(int64_t)e * ldr + e] : 1.0;
    if (threadIdx.x < TP_GROUPS * 2) tp_mbar_init(&bars[threadIdx.x], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp >> 1, v = warp & 1;
  const int q4 = lane & 3, gbase = lane & ~3;
  double* const myslot = slots + grp * 2 * 64;
  uint64_t* const mybars = bars + grp * 2;
  uint32_t wph = 0;  // phase of the partner's barriers this warp waits on (one completion per wait)
#pragma unroll 1
  for (int64_t r0 = ((int64_t)blockIdx.x * TP_GROUPS + grp) * 8; r0 < m; r0 += (int64_t)gridDim.x * TP_GROUPS * 8) {
    const int64_t row = r0 + (lane >> 2);
    const bool row_ok = row < m;
    uint32_t Rt = (uint32_t)__cvta_generic_to_shared(Rt_base);
    uint32_t Rd = (uint32_t)__cvta_generic_to_shared(Rd_base);
    uint32_t Ri = (uint32_t)__cvta_generic_to_shared(Ri_base);
    int64_t ldz_l = ldz, ldq_l = ldq;
    int n_l = n;
    asm volatile("" : "+r"(Rt), "+r"(Rd), "+r"(Ri), "+l"(ldz_l), "+l"(ldq_l), "+r"(n_l));
    double S[H][2];
#pragma unroll
    for (int h = 0; h < H; ++h) S[h][0] = S[h][1] = 0.0;
    // Z of this warp's own tiles, prefetched TP_PD own tiles ahead (a global load's latency spans
    // several tile solves: ncu showed the subtraction z - S waiting on it with one tile ahead)
    double zq[TP_PD][2];
#pragma unroll
    for (int d = 0; d < TP_PD; ++d)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tt = v + 2 * d, col = tt * 8 + 2 * q4 + e;
        zq[d][e] = (row_ok && tt < NT && col < n_l) ? Z[(int64_t)col * ldz_l + row] : 0.0;
      }
    double d0 = 0.0, d1 = 0.0;  // deferred fragments of the partner's last tile
    int dt = -1;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      if ((t & 1) == v) {
        // ---- own tile t: S[t/2] holds every q_k R[k, t], k < t
        const int h = t >> 1;
        const double zc0 = zq[h % TP_PD][0], zc1 = zq[h % TP_PD][1];
        if (t + 2 * TP_PD < NT) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = (t + 2 * TP_PD) * 8 + 2 * q4 + e;
            zq[h % TP_PD][e] = (row_ok && col < n_l) ? Z[(int64_t)col * ldz_l + row] : 0.0;
          }
        }
        double t0 = zc0 - S[t >> 1][0];
        double t1 = zc1 - S[t >> 1][1];
        double tt[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          tt[2 * q] = __shfl_sync(0xffffffffu, t0, gbase | q);
          tt[2 * q + 1] = __shfl_sync(0xffffffffu, t1, gbase | q);
        }
        double qv[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int dc = t * 8 + c;
          qv[c] = tt[c] * lds_f64(Ri + 8u * dc);
#pragma unroll
          for (int c2 = c + 1; c2 < 8; ++c2) tt[c2] = fma(-qv[c], lds_f64(Rd + 8u * ((t * 8 + c) * 8 + c2)), tt[c2]);
        }
        const double a0 = sel4(q4, qv[0], qv[1], qv[2], qv[3]);
        const double a1 = sel4(q4, qv[4], qv[5], qv[6], qv[7]);
        if (t + 1 < NT) {  // publish the solved 8 x 8 tile, row-major, for the partner
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double qe = sel4(q4, qv[e], qv[2 + e], qv[4 + e], qv[6 + e]);
            myslot[(t & 1) * 64 + (lane >> 2) * 8 + 2 * q4 + e] = qe;
          }
          __syncwarp();
          if (lane == 0) tp_mbar_arrive(&mybars[t & 1]);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = t * 8 + 2 * q4 + e;
          const double qe = sel4(q4, qv[e], qv[2 + e], qv[4 + e], qv[6 + e]);
  #ifdef OQR_EXP_TRSM_NOSTG  // timing-only diagnostic build: no Q stores except a never-true one
        if (row_ok && col < n_l && qe == 1.2345e300) Q[(int64_t)col * ldq_l + row] = qe;
#else
        if (row_ok && col < n_l) Q[(int64_t)col * ldq_l + row] = qe;
#endif
        }
        // ---- bulk: the deferred q_{t-1} (partner's) and then q_t on this warp's tiles > t, in k
        // order (first halves, then second halves, per k: the same order as the one-warp kernel)
        if (dt >= 0) {
#pragma unroll
          for (int j2 = t + 2; j2 < NT; j2 += 2)
            dmma_f(S[j2 >> 1], d0, lds_f64(Rt + 8u * ((j2 * (j2 - 1) / 2 + (t - 1)) * 64 + lane)));
#pragma unroll
          for (int j2 = t + 2; j2 < NT; j2 += 2)
            dmma_f(S[j2 >> 1], d1, lds_f64(Rt + 8u * ((j2 * (j2 - 1) / 2 + (t - 1)) * 64 + 32 + lane)));
        }
#pragma unroll
        for (int j2 = t + 2; j2 < NT; j2 += 2)
          dmma_f(S[j2 >> 1], a0, lds_f64(Rt + 8u * ((j2 * (j2 - 1) / 2 + t) * 64 + lane)));
#pragma unroll
        for (int j2 = t + 2; j2 < NT; j2 += 2)
          dmma_f(S[j2 >> 1], a1, lds_f64(Rt + 8u * ((j2 * (j2 - 1) / 2 + t) * 64 + 32 + lane)));
        dt = -1;
      } else {
        // ---- partner's tile t: wait for q_t (published only when a tile follows), apply it to
        // this warp's next tile t+1 at once, the rest deferred
        if (t + 1 < NT) {
          tp_mbar_wait(&mybars[t & 1], wph);  // the partner's parity: one completion per its tile
          wph ^= 1u;
          double qr[8];                        // row lane/4 of q_t
#pragma unroll
          for (int k = 0; k < 8; ++k) qr[k] = myslot[(t & 1) * 64 + (lane >> 2) * 8 + k];
          d0 = (q4 == 0) ? qr[0] : (q4 == 1) ? qr[1] : (q4 == 2) ? qr[2] : qr[3];
          d1 = (q4 == 0) ? qr[4] : (q4 == 1) ? qr[5] : (q4 == 2) ? qr[6] : qr[7];
          // the critical update S[t+1] += q_t R[t, t+1] on the FP64 FMA pipe, not behind the
          // queued bulk DMMAs of the tensor pipe: this lane's C entries (row lane/4, columns
          // 2 q4 + e) read R[t*8 + k, (t+1)*8 + 2 q4 + e] from the B-fragment tile (t+1, t)
          const uint32_t rtile = Rt + 8u * (((t + 1) * t / 2 + t) * 64);
#ifdef OQR_EXP_TP_DMMA_CRIT  // experiment build: the critical update on the tensor pipe too
          dmma_f(S[(t + 1) >> 1], d0, lds_f64(rtile + 8u * lane));
          dmma_f(S[(t + 1) >> 1], d1, lds_f64(rtile + 8u * (32 + lane)));
#else
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int k = 0; k < 8; ++k)
              S[(t + 1) >> 1][e] = fma(qr[k], lds_f64(rtile + 8u * ((k >> 2) * 32 + (k & 3) + 4 * (2 * q4 + e))),
                                       S[(t + 1) >> 1][e]);
#endif
          dt = t;
        }
      }
    }
  }
}

// ---- K3, column-panel form (experiment build OQR_EXP_TRSM_PANEL; measured slower) -----------
// The same substitution, with the per-tile accumulators of a warp's 8-row block limited to one
// panel of PW column tiles: for panel P (tiles t0 .. t0+PW-1) the contributions of the tiles
// already solved, S[j] = sum_{kt < t0} q_kt R[kt, j], are accumulated LEFT-looking (the q_kt
// A-fragments re-read from Q, which this warp wrote, through L1/L2) -- long independent DMMA
// streams, PW accumulators -- and the panel itself is solved right-looking as before.  Each
// accumulator receives its terms in the same order as in trsm_dmma_kernel (k ascending, first
// half before second half), so the result is bitwise that kernel's.  PW accumulators instead of
// NT free registers for more warps per SM (latency hiding) and the panel's Z is prefetched under
// the left-looking stream.
constexpr int KP_PW = 8;      // tiles per panel
constexpr int KP_MAXW = 16;   // warps per CTA at most (register budget: 65536 / (16 * 32) = 128)

template <int NT>
__global__ void __launch_bounds__(KP_MAXW * 32, 1)
trsm_panel_kernel(int64_t m, int n, const double* Z, int64_t ldz,  // Z may alias Q (in place)
                  const double* __restrict__ R, int64_t ldr, double* Q, int64_t ldq, const int* info) {
  if (info != nullptr && *info != 0) return;
  extern __shared__ __align__(16) double rsm[];
  double* const Rt_base = rsm;
  double* const Ri_base = rsm + (size_t)NT * (NT - 1) / 2 * 64;
  double* const Rd_base = Ri_base + (size_t)NT * 8;
  {
    constexpr int TOT = NT * (NT - 1) / 2 * 64;
    for (int e0 = threadIdx.x; e0 < TOT; e0 += 8 * blockDim.x) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        v[u] = 0.0;
        if (e < TOT) {
          const int t = e >> 6;
          int jt = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)t)) * 0.5f);
          while (jt * (jt - 1) / 2 > t) --jt;
          while ((jt + 1) * jt / 2 <= t) ++jt;
          const int kt = t - jt * (jt - 1) / 2, ln = e & 31, h = (e >> 5) & 1;
          const int k = kt * 8 + 4 * h + (ln & 3), col = jt * 8 + (ln >> 2);
          if (col < n) v[u] = R[(int64_t)col * ldr + k];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e < TOT) Rt_base[e] = v[u];
      }
    }
    for (int e = threadIdx.x; e < NT * 64; e += blockDim.x) {
      const int jt = e >> 6, c = (e >> 3) & 7, c2 = e & 7;
      const int r = jt * 8 + c, col = jt * 8 + c2;
      double v = 0.0;
      if (c <= c2) v = (col < n) ? R[(int64_t)col * ldr + r] : (c == c2 ? 1.0 : 0.0);
      Rd_base[e] = v;
    }
    for (int e = threadIdx.x; e < NT * 8; e += blockDim.x)
      Ri_base[e] = (e < n) ? 1.0 / R[(int64_t)e * ldr + e] : 1.0;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int q4 = lane & 3, gbase = lane & ~3;
#pragma unroll 1
  for (int64_t r0 = ((int64_t)blockIdx.x * nw + warp) * 8; r0 < m; r0 += (int64_t)gridDim.x * nw * 8) {
    const int64_t row = r0 + (lane >> 2);
    const bool row_ok = row < m;
    uint32_t Rt = (uint32_t)__cvta_generic_to_shared(Rt_base);
    uint32_t Rd = (uint32_t)__cvta_generic_to_shared(Rd_base);
    uint32_t Ri = (uint32_t)__cvta_generic_to_shared(Ri_base);
    int64_t ldz_l = ldz, ldq_l = ldq;
    int n_l = n;
    asm volatile("" : "+r"(Rt), "+r"(Rd), "+r"(Ri), "+l"(ldz_l), "+l"(ldq_l), "+r"(n_l));
#pragma unroll 1
    for (int t0 = 0; t0 < NT; t0 += KP_PW) {
      constexpr int PWC = KP_PW;
      // this panel's Z (PW tiles, two values per lane each), in flight under the left-looking stream
      double zq[PWC][2];
#pragma unroll
      for (int j = 0; j < PWC; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = (t0 + j) * 8 + 2 * q4 + e;
          zq[j][e] = (t0 + j < NT && row_ok && col < n_l) ? Z[(int64_t)col * ldz_l + row] : 0.0;
        }
      double S[PWC][2];
#pragma unroll
      for (int j = 0; j < PWC; ++j) S[j][0] = S[j][1] = 0.0;
      // left-looking: q_kt (kt < t0) from Q -- written by this warp in earlier panels (ordered by
      // the __syncwarp below) -- onto every tile of the panel
      if (t0 > 0) {
        __syncwarp();
        const int64_t qrow = r0 + (lane >> 2);
        const bool qok = qrow < m;
#pragma unroll 2
        for (int kt = 0; kt < t0; ++kt) {
          {
            const double a0 = qok ? Q[(int64_t)(kt * 8 + q4) * ldq_l + qrow] : 0.0;
            const double a1 = qok ? Q[(int64_t)(kt * 8 + 4 + q4) * ldq_l + qrow] : 0.0;
#pragma unroll
            for (int j = 0; j < PWC; ++j)
              if (t0 + j < NT)
                dmma_f(S[j], a0, lds_f64(Rt + 8u * (((t0 + j) * (t0 + j - 1) / 2 + kt) * 64 + lane)));
#pragma unroll
            for (int j = 0; j < PWC; ++j)
              if (t0 + j < NT)
                dmma_f(S[j], a1, lds_f64(Rt + 8u * (((t0 + j) * (t0 + j - 1) / 2 + kt) * 64 + 32 + lane)));
          }
        }
      }
      // right-looking inside the panel
#pragma unroll
      for (int j = 0; j < PWC; ++j) {
        const int jt = t0 + j;
        if (jt < NT) {
          double tt[8];
          {
            const double t0v = zq[j][0] - S[j][0], t1v = zq[j][1] - S[j][1];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              tt[2 * q] = __shfl_sync(0xffffffffu, t0v, gbase | q);
              tt[2 * q + 1] = __shfl_sync(0xffffffffu, t1v, gbase | q);
            }
          }
          double qv[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            qv[c] = tt[c] * lds_f64(Ri + 8u * (jt * 8 + c));
#pragma unroll
            for (int c2 = c + 1; c2 < 8; ++c2) tt[c2] = fma(-qv[c], lds_f64(Rd + 8u * ((jt * 8 + c) * 8 + c2)), tt[c2]);
          }
          const double a0 = sel4(q4, qv[0], qv[1], qv[2], qv[3]);
          const double a1 = sel4(q4, qv[4], qv[5], qv[6], qv[7]);
#pragma unroll
          for (int j2 = j + 1; j2 < PWC; ++j2)
            if (t0 + j2 < NT)
              dmma_f(S[j2], a0, lds_f64(Rt + 8u * (((t0 + j2) * (t0 + j2 - 1) / 2 + jt) * 64 + lane)));
#pragma unroll
          for (int j2 = j + 1; j2 < PWC; ++j2)
            if (t0 + j2 < NT)
              dmma_f(S[j2], a1, lds_f64(Rt + 8u * (((t0 + j2) * (t0 + j2 - 1) / 2 + jt) * 64 + 32 + lane)));
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = jt * 8 + 2 * q4 + e;
            const double qe = sel4(q4, qv[e], qv[2 + e], qv[4 + e], qv[6 + e]);
    #ifdef OQR_EXP_TRSM_NOSTG  // timing-only diagnostic build: no Q stores except a never-true one
        if (row_ok && col < n_l && qe == 1.2345e300) Q[(int64_t)col * ldq_l + row] = qe;
#else
        if (row_ok && col < n_l) Q[(int64_t)col * ldq_l + row] = qe;
#endif
          }
        }
      }
    }
  }
}

static int trsm_num_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

template <int NT>
static cudaError_t trsm_nt(int64_t m, int n, const double* Z, int64_t ldz, const double* R, int64_t ldr,
                           double* Q, int64_t ldq, const int* info, cudaStream_t s, const double* img,
                           const int* prog) {
#ifdef OQR_EXP_TRSM_PANEL  // experiment build only: the column-panel kernel (measured slower)
  if constexpr (NT > KP_PW) {
    constexpr bool smem_rd = true;
    constexpr size_t bytes = trsm_smem_doubles<NT>(smem_rd) * sizeof(double);
    if constexpr (bytes <= (size_t)SMEM_MAX) {
      cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(trsm_panel_kernel<NT>), (int)bytes);
      if (e != cudaSuccess) return e;
      // warps per CTA (<= KP_MAXW): the fewest passes over the 8-row blocks, then the fewest warps
      const int sms = trsm_num_sms();
      const int64_t rb = cdiv(m, 8);
      const int64_t per = cdiv(rb, sms);
      int best_w = KP_MAXW;
      int64_t best = INT64_MAX;
      for (int w = 8; w <= KP_MAXW; ++w) {
        const int64_t cost = cdiv(per, w) * w;
        if (cost < best) { best = cost; best_w = w; }
      }
      int64_t g = cdiv(rb, best_w);
      if (g > sms) g = sms;
      timing_begin(s, OQR_TIMING_K3);
      trsm_panel_kernel<NT><<<(unsigned)g, best_w * 32, bytes, s>>>(m, n, Z, ldz, R, ldr, Q, ldq, info);
      e = cudaGetLastError();
      timing_end(s);
      return e;
    }
  }
#endif
#ifdef OQR_EXP_TRSM_PAIR  // experiment build only: the warp-pair kernel (measured slower)
  if constexpr (NT >= 2 && trsm_pair_smem_bytes<NT>() <= (size_t)SMEM_MAX) {
    constexpr size_t bytes = trsm_pair_smem_bytes<NT>();
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(trsm_pair_kernel<NT>), (int)bytes);
    if (e != cudaSuccess) return e;
    int64_t g = cdiv(m, TP_GROUPS * 8);
    const int sms = trsm_num_sms();
    if (g > sms) g = sms;
    timing_begin(s, OQR_TIMING_K3);
    trsm_pair_kernel<NT><<<(unsigned)g, TP_GROUPS * 64, bytes, s>>>(m, n, Z, ldz, R, ldr, Q, ldq, info);
    e = cudaGetLastError();
    timing_end(s);
    return e;
  }
#endif
  constexpr bool smem_rd = trsm_smem_doubles<NT>(true) * sizeof(double) <= (size_t)SMEM_MAX;
  constexpr size_t bytes = trsm_smem_doubles<NT>(smem_rd) * sizeof(double);
  static_assert(bytes <= (size_t)SMEM_MAX, "R fragments must fit in shared memory");
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(trsm_dmma_kernel<NT, smem_rd>), (int)bytes);
  if (e != cudaSuccess) return e;
  constexpr int THREADS = trsm_threads(NT);
  int64_t g = cdiv(m, (THREADS / 32) * 8);  // 8 rows per warp per pass
  const int sms = trsm_num_sms();
  if (g > sms) g = sms;          // persistent: R is staged once per CTA
  if (prog != nullptr) {
    // overlapped with the K2 launched just before on `s` (launch_potrf with the same prog): a
    // programmatic dependent launch, one SM left to K2 when the two cannot share one
    if constexpr (!smem_rd) return cudaErrorInvalidValue;
    if (g >= sms && sms > 1) g = sms - 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, trsm_dmma_kernel<NT, smem_rd>, m, n, Z, ldz, R, ldr, Q, ldq, info, img, prog);
  }
  timing_begin(s, OQR_TIMING_K3);
  trsm_dmma_kernel<NT, smem_rd><<<(unsigned)g, THREADS, bytes, s>>>(m, n, Z, ldz, R, ldr, Q, ldq, info, img, nullptr);
  e = cudaGetLastError();
  timing_end(s);
  return e;
}

#define OQR_TRSM_CASES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) \
  X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30)

bool trsm_overlap_ok(int n) { return trsm_img_has_rd((int)cdiv(n, 8)); }

cudaError_t launch_trsm(int64_t m, int n, const double* Z, int64_t ldz, const double* R, int64_t ldr,
                        double* Q, int64_t ldq, const int* info, cudaStream_t s, const double* img,
                        const int* prog) {
  cudaError_t e;
  switch ((int)cdiv(n, 8)) {
#define OQR_CASE(NT) \
  case NT: e = trsm_nt<NT>(m, n, Z, ldz, R, ldr, Q, ldq, info, s, img, prog); break;
    OQR_TRSM_CASES(OQR_CASE)
#undef OQR_CASE
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K5 --------------------
// R = R2 R1 for upper triangular n x n ("R = US"; normal2: R = R2 R1):
// R[k, l] = sum_{p=k}^{l} R2[k, p] R1[p, l] (p ascending); strictly lower part zero.
__global__ void trmm_kernel(int n, const double* __restrict__ R2, const double* __restrict__ R1,
                            double* __restrict__ R, const int* info) {
  if (info != nullptr && *info != 0) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int l = e / n, k = e - l * n;
    double s = 0.0;
    if (k <= l)
      for (int p = k; p <= l; ++p) s += R2[(int64_t)p * n + k] * R1[(int64_t)l * n + p];
    R[e] = s;
  }
}

cudaError_t launch_trmm(int n, const double* R2, const double* R1, double* R, const int* info,
                        cudaStream_t s) {
  const int total = n * n;
  trmm_kernel<<<(unsigned)cdiv(total, 256), 256, 0, s>>>(n, R2, R1, R, info);
  note_launch();
  return cudaGetLastError();
}

}  // namespace oqr
