// oqr_hhqr.cu -- K6: Householder QR of Z (the paper's stable Euclidean pre-step of PRE-CHOLQR).
//
// Algorithm 2 line 1: [Y, S] = qr(Z) with "a stable Euclidean QR
// factorization (such as Householder QR)"; Theorem 3
// assumes exactly this pre-step.  Output: Y (m x n, ld m) with orthonormal columns and S (n x n,
// ld n) upper triangular with positive diagonal (the problem statement's convention,
// PAPER.md:44-51), Z = Y S.
//
// Householder convention (LAPACK dlarfg): for column j with alpha = x_j and tail = sum_{i>j} x_i^2,
//   tail == 0: tau = 0 (H = I), beta = alpha;
//   else       beta = -sign(alpha) sqrt(alpha^2 + tail), tau = (beta - alpha) / beta,
//              v_j = 1, v_i = x_i / (alpha - beta);  H_j = I - tau v v^T;  R_jj = beta.
// Signs: S = D R and Y = Q[:, :n] D with D = diag(sign R_jj) (exact), Y formed as
// H_0 ... H_{n-1} (I[:, :n] D).
//
// B200 design: one persistent cooperative kernel, one CTA per SM, each CTA owning a contiguous
// block of rows (the whole m x n working matrix stays L2-resident: 64 MB at m = 40000, n = 200).
// Columns are processed in panels of HNB = 16:
//   * panel factorization, one grid-wide exchange per column: each CTA reduces over its rows (kept
//     in shared memory) the partial sums of tail = sum x_i^2 AND d_l = sum x_i X_il for the panel's
//     later columns in one pass -- w_l = v^T X_l = X_jl + d_l / (alpha - beta) needs only the
//     scalars, so the norm and the reflector application share one reduction -- publishes them
//     with a per-CTA release flag, and every CTA sums the CTAs' partials (each read as soon as its
//     flag is up, no separate barrier) in the same fixed order (bitwise-identical scalars
//     everywhere, deterministic); one pass over its rows then applies H_j and accumulates the next
//     column's partials;
//   * blocked trailing update with the compact WY form (Schreiber-Van Loan):
//     Q_p = H_j0 ... H_j0+15 = I - V T V^T, C <- Q_p^T C = C - V T^T (V^T C): the partial
//     V^T [V C] of every CTA is reduce-scattered across the CTAs (two grid barriers), T is built
//     from V^T V and the taus (dlarft recurrence), and each CTA updates its rows;
//   * Y = Q_0 ... Q_{P-1} (I[:, :n] D) by the same blocked application, last panel first, to the
//     trailing block of Y only (dorgqr's structure).
// Summation order differs from the CPU checker's unblocked LAPACK-style loops; the result is
// the same Householder QR up to rounding, and parity is gated on the backward-stability
// properties Theorem 3 needs (tests/test_gpu_hhqr.py).
#include <algorithm>

#include "oqr_internal.cuh"

namespace oqr {

constexpr int HNB = 16;        // panel width
constexpr int HTH = 256;       // threads per CTA
constexpr int HWARPS = HTH / 32;
constexpr int HROWS = 256;     // target rows per CTA

#ifdef OQR_EXP_HH_PROF  // experiment build only (tools/exp): phase timestamps of CTA 0
__device__ unsigned long long g_hh_prof[16384];
__device__ int g_hh_prof_n;
#define HH_MARK(tag)                                                                  \
  do {                                                                                \
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_hh_prof_n < 8190) {                  \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_hh_prof[g_hh_prof_n++] = ((unsigned long long)(tag) << 56) | (t_ & ((1ull << 56) - 1)); \
    }                                                                                 \
  } while (0)
#else
#define HH_MARK(tag) \
  do {               \
  } while (0)
#endif

struct HhArgs {
  int64_t m;
  int n;
  const double* Z;
  int64_t ldz;
  double* X;        // m x n working matrix (ld m): R on/above, reflectors below the diagonal
  double* Y;        // m x n output (ld m)
  double* S;        // n x n output (ld n)
  double* part;     // [2][g][HNB + 1] per-column partial sums
  double* rowpub;   // [2][HNB] the pivot row of the current column (its owner publishes it)
  double* wpart;    // [g][HNB * (HNB + n)] per-CTA partials of V^T [V C]
  double* wfin;     // [HNB * (HNB + n)] reduced V^T [V C]
  unsigned* bar;    // grid barrier arrival counter (zeroed before the launch)
  unsigned* flags;  // [g] per-CTA column counters: CTA c has published column t's partials (zeroed)
  int rows_per;
  int g;
  int lookahead;    // 1: a second panel buffer in shared memory -> deferred trailing updates
};

// Grid-wide barrier among the g co-resident CTAs (cooperative launch): monotonic arrival counter.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& epoch, unsigned g) {
  __syncthreads();
  epoch += 1;
  if (threadIdx.x == 0) {
    // the CTA barrier above orders every thread's writes before this release (cumulative), and
    // the acquire below orders the CTA barrier after it -- no separate fences needed
    const unsigned target = epoch * g;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
// first local row of a CTA (rows [r0, r0 + rows)) at global row >= i0
__device__ __forceinline__ int first_row(int64_t i0, int64_t r0, int rows) { return (int)imax(0, imin(rows, i0 - r0)); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int HGU = 5;  // <= 32 * HGU CTAs: a lane's loads over the CTAs are unrolled

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr int HFS = 32;  // flag stride (unsigned): one 128-byte line per CTA's flag, no polling hot spot

// Wait until every CTA's flag shows column `step` published: warp 0, lanes over the CTAs, each
// polling round one batch of independent acquire loads (one round trip when the flags are up).
__device__ __forceinline__ void wait_flags(const unsigned* flags, unsigned step, int g, int lane) {
  bool ok;
  do {
    unsigned f[HGU];
#pragma unroll
    for (int t = 0; t < HGU; ++t) {
      const int c = lane + 32 * t;
      f[t] = (c < g) ? ld_acquire(flags + (int64_t)c * HFS) : step;
    }
    ok = true;
#pragma unroll
    for (int t = 0; t < HGU; ++t) ok = ok && f[t] >= step;
  } while (!__all_sync(0xffffffffu, ok));
}

// Sum over c = 0..g-1 of x[c * stride + k] (one warp; lanes over c, loads in one batch, fixed
// shuffle tree).
__device__ __forceinline__ double warp_sum_parts(const double* x, int g, int stride, int k, int lane) {
  double v[HGU];
#pragma unroll
  for (int t = 0; t < HGU; ++t) {
    const int c = lane + 32 * t;
    v[t] = (c < g) ? __ldcg(x + (int64_t)c * stride + k) : 0.0;
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < HGU; ++t) s += v[t];
  return warp_sum(s);
}

// Transposing butterfly: v[0..63] summed over the 32 lanes in 62 shuffles (instead of 64 x 5);
// afterwards lane L holds the totals of indices 2L and 2L + 1 in v[0], v[1].  Fixed order.
__device__ __forceinline__ void warp_reduce64(double (&v)[64], int lane) {
#define OQR_HH_STEP(H, O)                                                 \
  _Pragma("unroll") for (int i = 0; i < (H); ++i) {                       \
    const bool up = (lane & (O)) != 0;                                    \
    const double send = up ? v[i] : v[i + (H)];                           \
    const double keep = up ? v[i + (H)] : v[i];                           \
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, (O));                \
  }
  OQR_HH_STEP(32, 16)
  OQR_HH_STEP(16, 8)
  OQR_HH_STEP(8, 4)
  OQR_HH_STEP(4, 2)
  OQR_HH_STEP(2, 1)
#undef OQR_HH_STEP
}

constexpr int HCG = 4;  // columns per warp task in the panel products (4 x HNB = 64 accumulators)
constexpr int HRU = 4;  // row iterations per batch (loads in flight per lane: HRU * HCG)

// V^T [V C] partials of this CTA (local rows [lo, rows); V = Vs, HNB columns, zero beyond the
// panel), written to out: entry (a, col) at a * ncw + col, for a < nbp; col < nvv: (V^T V)[a][col],
// else (V^T C)[a][col - nvv] with C column cbase + col - nvv of (Cm, ldc) (row r0 + il).
// Warp per 4-column task, lanes over rows, 16 loads in flight per lane, transposing reduction.
__device__ void vtc_partials(const double* Vs, int RP, int lo, int rows, int nbp, int nvv, int ncw, const double* Cm,
                             int64_t ldc, int64_t r0, int cbase, double* out, int lane, int wid) {
  for (int col0 = wid * HCG; col0 < ncw; col0 += HWARPS * HCG) {
    double v[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = 0.0;
    const double* src[HCG];
    bool fromv[HCG], valid[HCG];
#pragma unroll
    for (int q = 0; q < HCG; ++q) {
      const int col = col0 + q;
      valid[q] = col < ncw;
      fromv[q] = col < nvv;
      src[q] = fromv[q] ? Vs + col * RP : Cm + (int64_t)(cbase + col - nvv) * ldc + r0;
    }
    for (int il0 = lo + lane; il0 < rows; il0 += 32 * HRU) {
      double cv[HRU][HCG];
#pragma unroll
      for (int u = 0; u < HRU; ++u)
#pragma unroll
        for (int q = 0; q < HCG; ++q) {
          const int il = il0 + 32 * u;
          cv[u][q] = (valid[q] && il < rows) ? (fromv[q] ? src[q][il] : __ldcg(src[q] + il)) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < HRU; ++u) {
        const int il = il0 + 32 * u;
        if (il < rows) {
#pragma unroll
          for (int aa = 0; aa < HNB; ++aa) {
            const double va = Vs[aa * RP + il];
#pragma unroll
            for (int q = 0; q < HCG; ++q) v[q * HNB + aa] = fma(va, cv[u][q], v[q * HNB + aa]);
          }
        }
      }
    }
    warp_reduce64(v, lane);
    const int q = lane >> 3, a0 = (2 * lane) & (HNB - 1), col = col0 + q;
    if (col < ncw) {
      if (a0 < nbp) __stcg(out + a0 * ncw + col, v[0]);
      if (a0 + 1 < nbp) __stcg(out + (a0 + 1) * ncw + col, v[1]);
    }
  }
}

// D[i, cbase + l] = C[i, cbase + l] - sum_a V[i][a] M[a][l] for local rows [lo, rows), l < ncols;
// M in shared memory (row a at Ms + a * ldm).  C read from (Cs, ldcs), written to (Cd, ldcd)
// (may be the same).  Warp per 4-column task, lanes over rows.
__device__ void panel_apply(const double* Vs, int RP, int lo, int rows, const double* Ms, int ldm, int ncols,
                            const double* Cs, int64_t ldcs, double* Cd, int64_t ldcd, int64_t r0, int cbase,
                            int lane, int wid, int nwarps = HWARPS) {
  for (int col0 = wid * HCG; col0 < ncols; col0 += nwarps * HCG) {
    double mm[HNB][HCG];
#pragma unroll
    for (int aa = 0; aa < HNB; ++aa)
#pragma unroll
      for (int q = 0; q < HCG; ++q) mm[aa][q] = (col0 + q < ncols) ? Ms[aa * ldm + col0 + q] : 0.0;
    for (int il0 = lo + lane; il0 < rows; il0 += 32 * HRU) {
      double cv[HRU][HCG];
#pragma unroll
      for (int u = 0; u < HRU; ++u)
#pragma unroll
        for (int q = 0; q < HCG; ++q) {
          const int il = il0 + 32 * u;
          cv[u][q] = (col0 + q < ncols && il < rows) ? Cs[(int64_t)(cbase + col0 + q) * ldcs + r0 + il] : 0.0;
        }
#pragma unroll
      for (int u = 0; u < HRU; ++u) {
        const int il = il0 + 32 * u;
        if (il < rows) {
          double sacc[HCG];
#pragma unroll
          for (int q = 0; q < HCG; ++q) sacc[q] = 0.0;
#pragma unroll
          for (int aa = 0; aa < HNB; ++aa) {
            const double va = Vs[aa * RP + il];
#pragma unroll
            for (int q = 0; q < HCG; ++q) sacc[q] = fma(va, mm[aa][q], sacc[q]);
          }
#pragma unroll
          for (int q = 0; q < HCG; ++q)
            if (col0 + q < ncols) Cd[(int64_t)(cbase + col0 + q) * ldcd + r0 + il] = cv[u][q] - sacc[q];
        }
      }
    }
  }
}

// Reduce-scatter of the CTAs' partials (fixed order over c), then everyone loads the result.
// This CTA sums its share of the E entries: 8 slices of the CTAs per entry, each slice's loads
// in flight together, the 8 slice sums added in slice order.
__device__ void reduce_partials(const HhArgs& a, int E, int c, double* Ws, double* scr, unsigned& epoch) {
  grid_barrier(a.bar, epoch, a.g);
  const int stride = HNB * (HNB + a.n);
  const int e0 = (int)((int64_t)E * c / a.g), e1 = (int)((int64_t)E * (c + 1) / a.g);
  const int tid = threadIdx.x, sl = tid & 7;
  const int c0 = a.g * sl / 8, c1 = a.g * (sl + 1) / 8;
  for (int eb = e0; eb < e1; eb += HTH / 8) {
    const int e = eb + (tid >> 3);
    double s = 0.0;
    if (e < e1) {
      double v[HGU * 4];
#pragma unroll
      for (int t = 0; t < HGU * 4; ++t) v[t] = (c0 + t < c1) ? __ldcg(a.wpart + (int64_t)(c0 + t) * stride + e) : 0.0;
#pragma unroll
      for (int t = 0; t < HGU * 4; ++t) s += v[t];
    }
    scr[tid] = s;
    __syncthreads();
    if (tid < HTH / 8 && eb + tid < e1) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) t += scr[tid * 8 + q];
      __stcg(a.wfin + eb + tid, t);
    }
    __syncthreads();
  }
  grid_barrier(a.bar, epoch, a.g);
  for (int e = threadIdx.x; e < E; e += HTH) Ws[e] = __ldcg(a.wfin + e);
  __syncthreads();
}

// v[0..15] summed over the 32 lanes in 16 shuffles; afterwards lanes 2k and 2k+1 hold the total of
// index k in v[0].  Fixed order.
__device__ __forceinline__ void warp_reduce16(double (&v)[HNB], int lane) {
#pragma unroll
  for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const bool up = (lane & o) != 0;
      const double send = up ? v[i] : v[i + h];
      const double keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
}

__global__ void __launch_bounds__(HTH, 1) hhqr_kernel(HhArgs a) {
  extern __shared__ double sm[];
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t m = a.m;
  const int n = a.n, RP = a.rows_per;
  const int P = (n + HNB - 1) / HNB;
  const int64_t r0 = (int64_t)c * RP;
  const int rows = (int)imax(0, imin(m, r0 + RP) - r0);
  double* Xs = sm;                          // [HNB][RP]: panel column a, local row il
  double* Ws = Xs + HNB * RP;               // [HNB][HNB + n]
  double* Ms = Ws + HNB * (HNB + n);        // [HNB][n]
  double* Ts = Ms + HNB * n;                // [P][HNB][HNB]: T of panel p, row a, column b
  double* taus = Ts + P * HNB * HNB;        // [n]
  double* betas = taus + n;                 // [n]
  double* red = betas + n;                  // [HNB]
  double* rowv = red + HNB;                 // [HNB]
  double* wscr = rowv + HNB;                // [HTH]: per-warp column partials / reduce-scatter slices
  double* Vp = wscr + HTH;                  // [HNB][RP] (look-ahead only): the previous panel's V
  unsigned epoch = 0, cstep = 0;
  int colbuf = 0;
  // Look-ahead: the trailing update of panel p is applied at once only to panel p+1's columns; the
  // rest is deferred and done, one chunk per column step of panel p+1, by warps 1..7 while warp 0
  // publishes and waits for the CTAs' flags (the exchange latency hides it).  Per column the same
  // arithmetic as the undeferred update.
  bool pending = false;
  int dcols = 0, dcb = 0, dlo = 0, dch = 0, dnt = 0;
  const double* dsrc = nullptr;
  int64_t dld = 0;
  HH_MARK(1);

  // ---------------------------------------------------------------- factorization ----
  // Panel 0 is read from Z directly and its trailing update writes X, so Z is never copied.
  for (int p = 0; p < P; ++p) {
    const int j0 = p * HNB, nbp = (int)imin(HNB, n - j0);
    const double* Xsrc = p == 0 ? a.Z : a.X;
    const int64_t ldsrc = p == 0 ? a.ldz : m;
    for (int il = tid; il < rows; il += HTH) {
      double x[HNB];
#pragma unroll
      for (int aa = 0; aa < HNB; ++aa) x[aa] = aa < nbp ? __ldcg(Xsrc + (int64_t)(j0 + aa) * ldsrc + r0 + il) : 0.0;
#pragma unroll
      for (int aa = 0; aa < HNB; ++aa) Xs[aa * RP + il] = x[aa];
    }
    __syncthreads();
    HH_MARK(2);
    // partial sums of the panel's first column over this CTA's rows i > j0:
    // acc[0] = sum x_i^2, acc[k] = sum x_i X_{i, k}; later columns get theirs in the fused pass
    double acc[HNB];
#pragma unroll
    for (int k = 0; k < HNB; ++k) acc[k] = 0.0;
    for (int il = first_row(j0 + 1, r0, rows) + tid; il < rows; il += HTH) {
      const double x = Xs[il];
      acc[0] = fma(x, x, acc[0]);
#pragma unroll
      for (int k = 1; k < HNB; ++k) acc[k] = fma(x, Xs[k * RP + il], acc[k]);
    }
    for (int jj = 0; jj < nbp; ++jj) {
      const int j = j0 + jj;
      const int nk = nbp - jj;  // tail + d_l for l = jj+1..nbp-1
      ++cstep;
      warp_reduce16(acc, lane);
      if ((lane & 1) == 0) wscr[wid * HNB + (lane >> 1)] = acc[0];
      __syncthreads();
      double* part = a.part + (int64_t)colbuf * a.g * (HNB + 1);
      double* rowpub = a.rowpub + colbuf * HNB;
      const bool owner = (j >= r0 && j < r0 + rows);
      if (wid == 0) {
        // warp 0 publishes: lane k < nk sums the 8 warps' k-th partial; the owner of row j also
        // publishes that row; then lane 0's release store (cumulative over the warp's writes,
        // ordered by __syncwarp) raises this CTA's flag -- no fence, no extra CTA barrier
        if (lane < nk) {
          double s = 0.0;
#pragma unroll
          for (int w = 0; w < HWARPS; ++w) s += wscr[w * HNB + lane];
          __stcg(part + c * (HNB + 1) + lane, s);
          if (owner) __stcg(rowpub + lane, Xs[(jj + lane) * RP + (j - r0)]);
        }
        __syncwarp();
        if (lane == 0)
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.flags + (int64_t)c * HFS), "r"(cstep) : "memory");
        HH_MARK(3);
        wait_flags(a.flags, cstep, a.g, lane);
      } else if (pending) {
        const int d0 = jj * dch, d1 = (int)imin(dcols, d0 + dch);
        if (d1 > d0)
          panel_apply(Vp, RP, dlo, rows, Ms + (HNB + d0), dnt, d1 - d0, dsrc, dld, a.X, m, r0, dcb + d0, lane, wid - 1,
                      HWARPS - 1);
      }
      __syncthreads();
      for (int k = wid; k < nk; k += HWARPS) {
        const double s = warp_sum_parts(part, a.g, HNB + 1, k, lane);
        if (lane == 0) red[k] = s;
      }
      if (tid >= 32 * (HWARPS - 1) && tid - 32 * (HWARPS - 1) < nk)
        rowv[tid - 32 * (HWARPS - 1)] = __ldcg(rowpub + tid - 32 * (HWARPS - 1));
      colbuf ^= 1;
      __syncthreads();
      HH_MARK(4);
      const double alpha = rowv[0], tail = red[0];
      double beta = alpha, tau = 0.0, scal = 0.0;
      if (tail != 0.0) {
        const double nrm = sqrt(alpha * alpha + tail);
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      if (tid == 0) {
        taus[j] = tau;
        betas[j] = beta;
      }
      double w[HNB];  // w_k = v^T X_{jj+k} = X_{j, jj+k} + scal * d_k
#pragma unroll
      for (int k = 1; k < HNB; ++k) w[k] = (k < nk) ? rowv[k] + scal * red[k] : 0.0;
      // one pass over this CTA's rows i > j: apply H_j to the panel's later columns and, in the
      // same pass, accumulate the next column's partial sums (rows i > j + 1) -- a row is updated
      // and then read by the same thread, so no barrier is needed in between
#pragma unroll
      for (int k = 0; k < HNB; ++k) acc[k] = 0.0;
      const int lo = first_row(j + 1, r0, rows);
      const bool upd = tail != 0.0;
      for (int il = lo + tid; il < rows; il += HTH) {
        double x1 = nk > 1 ? Xs[(jj + 1) * RP + il] : 0.0;
        if (upd) {
          const double v = Xs[jj * RP + il] * scal;
          Xs[jj * RP + il] = v;
          const double tv = tau * v;
          x1 -= tv * w[1];
#pragma unroll
          for (int k = 1; k < HNB; ++k)
            if (k < nk) Xs[(jj + k) * RP + il] -= tv * w[k];
        }
        if (nk > 1 && r0 + il > j + 1) {
          acc[0] = fma(x1, x1, acc[0]);
#pragma unroll
          for (int k = 1; k < HNB; ++k)
            if (k + 1 < nk) acc[k] = fma(x1, Xs[(jj + 1 + k) * RP + il], acc[k]);
        }
      }
      if (owner && tid == 0 && upd) {
        const int il = (int)(j - r0);
#pragma unroll
        for (int k = 1; k < HNB; ++k)
          if (k < nk) Xs[(jj + k) * RP + il] -= tau * w[k];
        Xs[jj * RP + il] = beta;
      }
      HH_MARK(5);
    }
    __syncthreads();
    if (pending) {  // chunks the column steps did not cover (a panel narrower than HNB)
      const int d0 = nbp * dch;
      if (d0 < dcols)
        panel_apply(Vp, RP, dlo, rows, Ms + (HNB + d0), dnt, dcols - d0, dsrc, dld, a.X, m, r0, dcb + d0, lane, wid);
      pending = false;
      __syncthreads();
    }
    // panel done: write back, turn the panel into V (zeros above, ones on the diagonal, zero
    // columns beyond the panel)
    for (int aa = 0; aa < nbp; ++aa)
      for (int il = tid; il < rows; il += HTH) {
        const int64_t i = r0 + il;
        const double x = Xs[aa * RP + il];
        a.X[(int64_t)(j0 + aa) * m + i] = x;
        Xs[aa * RP + il] = (i < j0 + aa) ? 0.0 : (i == j0 + aa ? 1.0 : x);
      }
    __syncthreads();
    const int nt = n - j0 - nbp;
    const int ncw = nbp + nt;
    const int lo = first_row(j0, r0, rows);
    vtc_partials(Xs, RP, lo, rows, nbp, nbp, ncw, Xsrc, ldsrc, r0, j0 + nbp, a.wpart + (int64_t)c * HNB * (HNB + n),
                 lane, wid);
    HH_MARK(6);
    reduce_partials(a, nbp * ncw, c, Ws, wscr, epoch);
    HH_MARK(7);
    // T (dlarft, forward columnwise): T_bb = tau_b, T[0:b, b] = -tau_b T[0:b, 0:b] (V^T V)[0:b, b]
    double* T = Ts + p * HNB * HNB;
    if (wid == 0) {
      for (int b = 0; b < HNB; ++b) {
        double t = 0.0;
        if (b < nbp && lane < b) {
          const double tb = taus[j0 + b];
          double s = 0.0;
          for (int k = lane; k < b; ++k) s = fma(T[lane * HNB + k], Ws[k * ncw + b], s);
          t = -tb * s;
        }
        __syncwarp();
        if (lane < HNB) {
          if (lane < b) T[lane * HNB + b] = (b < nbp) ? t : 0.0;
          else if (lane == b) T[b * HNB + b] = (b < nbp) ? taus[j0 + b] : 0.0;
          else T[lane * HNB + b] = 0.0;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (nt > 0) {
      // M = T^T W_C: M[a][l] = sum_{b <= a} T[b][a] W[b][nbp + l]; rows a >= nbp are zero
      for (int e = tid; e < HNB * nt; e += HTH) {
        const int aa = e / nt, l = e - aa * nt;
        double s = 0.0;
        if (aa < nbp)
          for (int b = 0; b <= aa; ++b) s = fma(T[b * HNB + aa], Ws[b * ncw + nbp + l], s);
        Ms[aa * nt + l] = s;
      }
      __syncthreads();
      // X[i, j0 + nbp + l] = C[i, l] - sum_a V[i][a] M[a][l] for this CTA's rows i >= j0
      if (a.lookahead && nt > HNB) {
        // now: the next panel's columns; the rest during the next panel's column steps
        panel_apply(Xs, RP, lo, rows, Ms, nt, HNB, Xsrc, ldsrc, a.X, m, r0, j0 + nbp, lane, wid);
        for (int e = tid; e < HNB * RP; e += HTH) Vp[e] = Xs[e];
        pending = true;
        dcols = nt - HNB;
        dcb = j0 + nbp + HNB;
        dlo = lo;
        dnt = nt;
        dsrc = Xsrc;
        dld = ldsrc;
        const int nnext = (int)imin(HNB, n - (j0 + nbp));
        dch = (dcols + nnext - 1) / nnext;
      } else {
        panel_apply(Xs, RP, lo, rows, Ms, nt, nt, Xsrc, ldsrc, a.X, m, r0, j0 + nbp, lane, wid);
      }
      __syncthreads();
    }
    HH_MARK(9);
  }

  // ---------------------------------------------------------------- S and Y ----
  for (int il = tid; il < rows; il += HTH) {
    const int64_t i = r0 + il;
    if (i < n) {
      const double sg = betas[i] < 0.0 ? -1.0 : 1.0;
      for (int l = 0; l < n; ++l) a.S[(int64_t)l * n + i] = (l >= i) ? sg * a.X[(int64_t)l * m + i] : 0.0;
    }
  }
  // Y = I[:, :n] D on this CTA's rows (only rows < n carry a nonzero)
  for (int64_t e = tid; e < (int64_t)rows * n; e += HTH) {
    const int l = (int)(e / rows), il = (int)(e - (int64_t)l * rows);
    const int64_t i = r0 + il;
    a.Y[(int64_t)l * m + i] = (i == l) ? (betas[l] < 0.0 ? -1.0 : 1.0) : 0.0;
  }
  __syncthreads();
  for (int p = P - 1; p >= 0; --p) {
    const int j0 = p * HNB, nbp = (int)imin(HNB, n - j0);
    const int nc = n - j0;
    for (int il = tid; il < rows; il += HTH) {
      const int64_t i = r0 + il;
      double x[HNB];
#pragma unroll
      for (int aa = 0; aa < HNB; ++aa)
        x[aa] = (aa >= nbp || i < j0 + aa) ? 0.0 : (i == j0 + aa ? 1.0 : __ldcg(a.X + (int64_t)(j0 + aa) * m + i));
#pragma unroll
      for (int aa = 0; aa < HNB; ++aa) Xs[aa * RP + il] = x[aa];
    }
    __syncthreads();
    const int lo = first_row(j0, r0, rows);
    // W = V^T Y[:, j0:n] (T is kept from the factorization: no V^T V needed)
    vtc_partials(Xs, RP, lo, rows, nbp, 0, nc, a.Y, m, r0, j0, a.wpart + (int64_t)c * HNB * (HNB + n), lane, wid);
    HH_MARK(10);
    reduce_partials(a, nbp * nc, c, Ws, wscr, epoch);
    HH_MARK(11);
    // M = T W: M[a][l] = sum_{b >= a} T[a][b] W[b][l]; rows a >= nbp are zero
    const double* T = Ts + p * HNB * HNB;
    for (int e = tid; e < HNB * nc; e += HTH) {
      const int aa = e / nc, l = e - aa * nc;
      double s = 0.0;
      if (aa < nbp)
        for (int b = aa; b < nbp; ++b) s = fma(T[aa * HNB + b], Ws[b * nc + l], s);
      Ms[aa * nc + l] = s;
    }
    __syncthreads();
    panel_apply(Xs, RP, lo, rows, Ms, nc, nc, a.Y, m, a.Y, m, r0, j0, lane, wid);
    __syncthreads();
    HH_MARK(12);
  }
  HH_MARK(13);
}

// ---------------------------------------------------------------- host side ----
struct HhPlan {
  int g = 0, rows_per = 0, lookahead = 0;
  size_t smem = 0;
};

static int sm_count() {
  static int cnt[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cnt[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cnt[dev] = v > 0 ? v : 148;
  }
  return cnt[dev];
}

static HhPlan hh_plan(int64_t m, int n) {
  HhPlan pl;
  const int64_t gmax = sm_count();
  // <= 32 * HGU CTAs (the flag polls and partial-sum loads are unrolled)
  int64_t g = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(gmax, 32 * HGU), cdiv(m, HROWS)));
  const int64_t rp = cdiv(m, g);
  g = cdiv(m, rp);
  pl.g = (int)g;
  pl.rows_per = (int)rp;
  const int P = (n + HNB - 1) / HNB;
  pl.smem = sizeof(double) * ((size_t)HNB * rp + (size_t)HNB * (HNB + n) + (size_t)HNB * n +
                              (size_t)P * HNB * HNB + 2 * (size_t)n + 2 * HNB + HTH);
  const size_t la = sizeof(double) * (size_t)HNB * rp;  // the look-ahead panel buffer
#ifndef OQR_EXP_HH_NOLOOKAHEAD
  if (pl.smem + la <= (size_t)SMEM_MAX) {
    pl.smem += la;
    pl.lookahead = 1;
  }
#endif
  return pl;
}

size_t hh_scratch_doubles(int64_t m, int n) {
  const HhPlan pl = hh_plan(m, n);
  return 2 * (size_t)pl.g * (HNB + 1) + 2 * HNB + (size_t)pl.g * HNB * (HNB + n) + (size_t)HNB * (HNB + n) + 2 +
         ((size_t)(pl.g + 1) * HFS + 1) / 2;  // barrier counter line and the per-CTA column flag lines
}

bool hh_supported(int64_t m, int n) { return hh_plan(m, n).smem <= (size_t)SMEM_MAX; }

cudaError_t launch_hhqr(int64_t m, int n, const double* Z, int64_t ldz, double* X, double* Y, double* S,
                        double* scratch, cudaStream_t s) {
  const HhPlan pl = hh_plan(m, n);
  if (pl.smem > (size_t)SMEM_MAX) return cudaErrorInvalidValue;
  cudaError_t e = ensure_smem_attr((const void*)hhqr_kernel, (int)pl.smem);
  if (e != cudaSuccess) return e;
  HhArgs a;
  a.m = m;
  a.n = n;
  a.Z = Z;
  a.ldz = ldz;
  a.X = X;
  a.Y = Y;
  a.S = S;
  a.part = scratch;
  a.rowpub = a.part + 2 * (size_t)pl.g * (HNB + 1);
  a.wpart = a.rowpub + 2 * HNB;
  a.wfin = a.wpart + (size_t)pl.g * HNB * (HNB + n);
  a.bar = reinterpret_cast<unsigned*>(a.wfin + (size_t)HNB * (HNB + n));
  a.flags = a.bar + HFS;
  a.rows_per = pl.rows_per;
  a.g = pl.g;
  a.lookahead = pl.lookahead;
  e = cudaMemsetAsync(a.bar, 0, sizeof(unsigned) * (HFS + (size_t)pl.g * HFS), s);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)pl.g);
  cfg.blockDim = dim3(HTH);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: the grid barrier is safe
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  timing_begin(s, OQR_TIMING_K6);
  e = cudaLaunchKernelEx(&cfg, hhqr_kernel, a);
  timing_end(s);
  note_launch();
  return e;
}

}  // namespace oqr

#ifdef OQR_EXP_HH_PROF
extern "C" int oqr_exp_hh_prof(unsigned long long* out, int cap) {
  int n = 0;
  cudaMemcpyFromSymbol(&n, oqr::g_hh_prof_n, sizeof(int));
  if (n > cap) n = cap;
  cudaMemcpyFromSymbol(out, oqr::g_hh_prof, sizeof(unsigned long long) * n);
  int z = 0;
  cudaMemcpyToSymbol(oqr::g_hh_prof_n, &z, sizeof(int));
  return n;
}
#endif
