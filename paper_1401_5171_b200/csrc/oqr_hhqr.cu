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
//   * panel factorization, one grid barrier per column: each CTA reduces over its rows (kept in
//     shared memory) the partial sums of tail = sum x_i^2 AND d_l = sum x_i X_il for the panel's
//     later columns in one pass -- w_l = v^T X_l = X_jl + d_l / (alpha - beta) needs only the
//     scalars, so the norm and the reflector application share one reduction -- publishes them,
//     and after the barrier every CTA sums the CTAs' partials in the same fixed order
//     (bitwise-identical scalars everywhere, deterministic) and updates its rows;
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
  int rows_per;
  int g;
};

// Grid-wide barrier among the g co-resident CTAs (cooperative launch): monotonic arrival counter.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& epoch, unsigned g) {
  __syncthreads();
  epoch += 1;
  if (threadIdx.x == 0) {
    const unsigned target = epoch * g;
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    __threadfence();
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

// Sum of x[c * stride + k] over c = 0..g-1 by one warp (lanes over c, fixed shuffle tree).
__device__ __forceinline__ double warp_sum_parts(const double* x, int g, int stride, int k, int lane) {
  double s = 0.0;
  for (int c = lane; c < g; c += 32) s += __ldcg(x + (int64_t)c * stride + k);
  return warp_sum(s);
}

// V^T [V C] partials of this CTA (rows [lo, rows) of its block; V has nbp columns), written to
// wpart[c]: entry (a, col) at a * ncw + col; col < nvv: (V^T V)[a][col], else (V^T C)[a][col - nvv]
// with C column cbase + col - nvv of `Cm` (ld m).  Warp per output column, lanes over rows.
__device__ void vtc_partials(const double* Vs, int RP, int lo, int rows, int nbp, int nvv, int ncw, const double* Cm,
                             int64_t m, int64_t r0, int cbase, double* out, int lane, int wid) {
  for (int col = wid; col < ncw; col += HWARPS) {
    double acc[HNB];
#pragma unroll
    for (int a = 0; a < HNB; ++a) acc[a] = 0.0;
    const double* cg = (col < nvv) ? nullptr : Cm + (int64_t)(cbase + col - nvv) * m + r0;
    for (int il = lo + lane; il < rows; il += 32) {
      const double cv = cg ? cg[il] : Vs[col * RP + il];
#pragma unroll
      for (int a = 0; a < HNB; ++a)
        if (a < nbp) acc[a] = fma(Vs[a * RP + il], cv, acc[a]);
    }
#pragma unroll
    for (int a = 0; a < HNB; ++a) {
      if (a < nbp) {
        const double s = warp_sum(acc[a]);
        if (lane == 0) __stcg(out + a * ncw + col, s);
      }
    }
  }
}

// Reduce-scatter of the CTAs' partials (fixed order over c), then everyone loads the result.
__device__ void reduce_partials(const HhArgs& a, int E, int c, double* Ws, unsigned& epoch) {
  grid_barrier(a.bar, epoch, a.g);
  const int stride = HNB * (HNB + a.n);
  const int e0 = (int)((int64_t)E * c / a.g), e1 = (int)((int64_t)E * (c + 1) / a.g);
  for (int e = e0 + threadIdx.x; e < e1; e += HTH) {
    double s = 0.0;
    for (int cc = 0; cc < a.g; ++cc) s += __ldcg(a.wpart + (int64_t)cc * stride + e);
    __stcg(a.wfin + e, s);
  }
  grid_barrier(a.bar, epoch, a.g);
  for (int e = threadIdx.x; e < E; e += HTH) Ws[e] = __ldcg(a.wfin + e);
  __syncthreads();
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
  double* red = betas + n;                  // [HNB + 1]
  double* rowv = red + HNB + 1;             // [HNB]
  double* wscr = rowv + HNB;                // [HWARPS][HNB + 1]
  unsigned epoch = 0;
  int colbuf = 0;

  // working copy of this CTA's rows of Z
  for (int l = 0; l < n; ++l)
    for (int il = tid; il < rows; il += HTH) a.X[(int64_t)l * m + r0 + il] = a.Z[(int64_t)l * a.ldz + r0 + il];
  __syncthreads();

  // ---------------------------------------------------------------- factorization ----
  for (int p = 0; p < P; ++p) {
    const int j0 = p * HNB, nbp = (int)imin(HNB, n - j0);
    for (int aa = 0; aa < nbp; ++aa)
      for (int il = tid; il < rows; il += HTH) Xs[aa * RP + il] = a.X[(int64_t)(j0 + aa) * m + r0 + il];
    __syncthreads();
    for (int jj = 0; jj < nbp; ++jj) {
      const int j = j0 + jj;
      const int nk = nbp - jj;  // tail + d_l for l = jj+1..nbp-1
      // partial sums over this CTA's rows i > j
      double acc[HNB];
#pragma unroll
      for (int k = 0; k < HNB; ++k) acc[k] = 0.0;
      const int lo = first_row(j + 1, r0, rows);
      for (int il = lo + tid; il < rows; il += HTH) {
        const double x = Xs[jj * RP + il];
        acc[0] = fma(x, x, acc[0]);
#pragma unroll
        for (int k = 1; k < HNB; ++k)
          if (k < nk) acc[k] = fma(x, Xs[(jj + k) * RP + il], acc[k]);
      }
#pragma unroll
      for (int k = 0; k < HNB; ++k) {
        if (k < nk) {
          const double s = warp_sum(acc[k]);
          if (lane == 0) wscr[wid * (HNB + 1) + k] = s;
        }
      }
      __syncthreads();
      double* part = a.part + (int64_t)colbuf * a.g * (HNB + 1);
      double* rowpub = a.rowpub + colbuf * HNB;
      if (tid < nk) {
        double s = 0.0;
        for (int w = 0; w < HWARPS; ++w) s += wscr[w * (HNB + 1) + tid];
        __stcg(part + c * (HNB + 1) + tid, s);
      }
      const bool owner = (j >= r0 && j < r0 + rows);
      if (owner && tid < nk) __stcg(rowpub + tid, Xs[(jj + tid) * RP + (j - r0)]);
      grid_barrier(a.bar, epoch, a.g);
      for (int k = wid; k < nk; k += HWARPS) {
        const double s = warp_sum_parts(part, a.g, HNB + 1, k, lane);
        if (lane == 0) red[k] = s;
      }
      if (tid < nk) rowv[tid] = __ldcg(rowpub + tid);
      colbuf ^= 1;
      __syncthreads();
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
      if (tail != 0.0) {
        double w[HNB];  // w_k = v^T X_{jj+k} = X_{j, jj+k} + scal * d_k
#pragma unroll
        for (int k = 1; k < HNB; ++k) w[k] = (k < nk) ? rowv[k] + scal * red[k] : 0.0;
        for (int il = lo + tid; il < rows; il += HTH) {
          const double v = Xs[jj * RP + il] * scal;
          Xs[jj * RP + il] = v;
          const double tv = tau * v;
#pragma unroll
          for (int k = 1; k < HNB; ++k)
            if (k < nk) Xs[(jj + k) * RP + il] -= tv * w[k];
        }
        if (owner && tid == 0) {
          const int il = (int)(j - r0);
#pragma unroll
          for (int k = 1; k < HNB; ++k)
            if (k < nk) Xs[(jj + k) * RP + il] -= tau * w[k];
          Xs[jj * RP + il] = beta;
        }
      }
      __syncthreads();
    }
    // panel done: write back, turn the panel into V (zeros above, ones on the diagonal)
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
    vtc_partials(Xs, RP, lo, rows, nbp, nbp, ncw, a.X, m, r0, j0 + nbp, a.wpart + (int64_t)c * HNB * (HNB + n), lane, wid);
    reduce_partials(a, nbp * ncw, c, Ws, epoch);
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
      // M = T^T W_C: M[a][l] = sum_{b <= a} T[b][a] W[b][nbp + l]
      for (int e = tid; e < nbp * nt; e += HTH) {
        const int aa = e / nt, l = e - aa * nt;
        double s = 0.0;
        for (int b = 0; b <= aa; ++b) s = fma(T[b * HNB + aa], Ws[b * ncw + nbp + l], s);
        Ms[aa * nt + l] = s;
      }
      __syncthreads();
      // C[i, l] -= sum_a V[i][a] M[a][l] for this CTA's rows i >= j0
      for (int l = 0; l < nt; ++l) {
        double* cg = a.X + (int64_t)(j0 + nbp + l) * m + r0;
        for (int il = lo + tid; il < rows; il += HTH) {
          double s = 0.0;
#pragma unroll
          for (int aa = 0; aa < HNB; ++aa)
            if (aa < nbp) s = fma(Xs[aa * RP + il], Ms[aa * nt + l], s);
          cg[il] -= s;
        }
      }
      __syncthreads();
    }
  }

  // ---------------------------------------------------------------- S and Y ----
  for (int il = tid; il < rows; il += HTH) {
    const int64_t i = r0 + il;
    if (i < n) {
      const double sg = betas[i] < 0.0 ? -1.0 : 1.0;
      for (int l = 0; l < n; ++l) a.S[(int64_t)l * n + i] = (l >= i) ? sg * a.X[(int64_t)l * m + i] : 0.0;
    }
  }
  for (int l = 0; l < n; ++l)
    for (int il = tid; il < rows; il += HTH) {
      const int64_t i = r0 + il;
      a.Y[(int64_t)l * m + i] = (i == l) ? (betas[l] < 0.0 ? -1.0 : 1.0) : 0.0;
    }
  __syncthreads();
  for (int p = P - 1; p >= 0; --p) {
    const int j0 = p * HNB, nbp = (int)imin(HNB, n - j0);
    const int nc = n - j0;
    for (int aa = 0; aa < nbp; ++aa)
      for (int il = tid; il < rows; il += HTH) {
        const int64_t i = r0 + il;
        Xs[aa * RP + il] = (i < j0 + aa) ? 0.0 : (i == j0 + aa ? 1.0 : a.X[(int64_t)(j0 + aa) * m + i]);
      }
    __syncthreads();
    const int lo = first_row(j0, r0, rows);
    // W = V^T Y[:, j0:n] (T is kept from the factorization: no V^T V needed)
    vtc_partials(Xs, RP, lo, rows, nbp, 0, nc, a.Y, m, r0, j0, a.wpart + (int64_t)c * HNB * (HNB + n), lane, wid);
    reduce_partials(a, nbp * nc, c, Ws, epoch);
    // M = T W: M[a][l] = sum_{b >= a} T[a][b] W[b][l]
    const double* T = Ts + p * HNB * HNB;
    for (int e = tid; e < nbp * nc; e += HTH) {
      const int aa = e / nc, l = e - aa * nc;
      double s = 0.0;
      for (int b = aa; b < nbp; ++b) s = fma(T[aa * HNB + b], Ws[b * nc + l], s);
      Ms[aa * nc + l] = s;
    }
    __syncthreads();
    for (int l = 0; l < nc; ++l) {
      double* yg = a.Y + (int64_t)(j0 + l) * m + r0;
      for (int il = lo + tid; il < rows; il += HTH) {
        double s = 0.0;
#pragma unroll
        for (int aa = 0; aa < HNB; ++aa)
          if (aa < nbp) s = fma(Xs[aa * RP + il], Ms[aa * nc + l], s);
        yg[il] -= s;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- host side ----
struct HhPlan {
  int g = 0, rows_per = 0;
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
  int64_t g = std::max<int64_t>(1, std::min<int64_t>(gmax, cdiv(m, HROWS)));
  const int64_t rp = cdiv(m, g);
  g = cdiv(m, rp);
  pl.g = (int)g;
  pl.rows_per = (int)rp;
  const int P = (n + HNB - 1) / HNB;
  pl.smem = sizeof(double) * ((size_t)HNB * rp + (size_t)HNB * (HNB + n) + (size_t)HNB * n +
                              (size_t)P * HNB * HNB + 2 * (size_t)n + (HNB + 1) + HNB + HWARPS * (HNB + 1));
  return pl;
}

size_t hh_scratch_doubles(int64_t m, int n) {
  const HhPlan pl = hh_plan(m, n);
  return 2 * (size_t)pl.g * (HNB + 1) + 2 * HNB + (size_t)pl.g * HNB * (HNB + n) + (size_t)HNB * (HNB + n) + 2;
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
  a.rows_per = pl.rows_per;
  a.g = pl.g;
  e = cudaMemsetAsync(a.bar, 0, sizeof(unsigned), s);
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
