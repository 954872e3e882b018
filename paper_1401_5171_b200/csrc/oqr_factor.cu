// oqr_factor.cu -- K2 single-CTA Cholesky, K3 row-wise triangular solve, K5 triangular product.
#include "oqr_internal.cuh"

namespace oqr {

// ------------------------------------------------------------------ K2 --------------------
// R = chol(G), upper, R^T R = G: Algorithm 1 line 3, backward error
// eq:normal:chol.  One CTA; the upper triangle of G lives packed in shared
// memory (column-major packed index l(l+1)/2 + k, k <= l; n = 240 -> 231,360 B).  Right-looking:
// at step j the pivot d = a_jj is tested with the LAPACK rule (breakdown iff !(d > 0), which
// also catches NaN; reading R4), row j is scaled by 1/sqrt(d) (true division), and the
// trailing upper triangle is updated a_kl -= r_jk r_jl.  Only the upper triangle is read.
__device__ __forceinline__ int pk(int k, int l) { return l * (l + 1) / 2 + k; }

__global__ void __launch_bounds__(1024, 1)
potrf_kernel(int n, const double* __restrict__ G, int64_t ldg, double* __restrict__ R, int64_t ldr,
             int* info, int info_off) {
  extern __shared__ double S[];
  if (info_off > 0 && *info != 0) return;  // an earlier stage already broke down
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int l = ty; l < n; l += 32)
    for (int k = tx; k <= l; k += 32) S[pk(k, l)] = G[(int64_t)l * ldg + k];
  __syncthreads();
  int brk = 0;
  for (int j = 0; j < n; ++j) {
    const double d = S[pk(j, j)];
    if (!(d > 0.0)) {  // uniform: every thread read the same value after the last barrier
      brk = j + 1;
      break;
    }
    const double rjj = sqrt(d);
    __syncthreads();  // all reads of a_jj done before it is overwritten
    for (int l = j + 1 + threadIdx.x; l < n; l += blockDim.x) S[pk(j, l)] = S[pk(j, l)] / rjj;
    if (threadIdx.x == 0) S[pk(j, j)] = rjj;
    __syncthreads();
    for (int l = j + 1 + ty; l < n; l += 32) {
      const double rjl = S[pk(j, l)];
      for (int k = j + 1 + tx; k <= l; k += 32) S[pk(k, l)] -= S[pk(j, k)] * rjl;
    }
    __syncthreads();
  }
  if (brk) {
    if (threadIdx.x == 0) *info = info_off + brk;
    return;
  }
  for (int l = ty; l < n; l += 32)
    for (int k = tx; k < n; k += 32) R[(int64_t)l * ldr + k] = (k <= l) ? S[pk(k, l)] : 0.0;
  if (threadIdx.x == 0 && info_off == 0) *info = 0;
}

cudaError_t launch_potrf(int n, const double* G, int64_t ldg, double* R, int64_t ldr, int* info,
                         int info_off, cudaStream_t s) {
  const size_t bytes = (size_t)n * (n + 1) / 2 * sizeof(double);
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  potrf_kernel<<<1, 1024, bytes, s>>>(n, G, ldg, R, ldr, info, info_off);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K3 --------------------
// Q = Z R^{-1}: Algorithm 1 line 4 as the row-wise substitution whose backward
// error is stated at PAPER.md:197-198:  q_ij = (z_ij - sum_{k<j} q_ik r_kj) / r_jj.
// One thread per row (coalesced: consecutive threads = consecutive rows of column-major Z/Q).
// Columns are processed in blocks of NB: the NB partial sums stay in registers while k runs
// 0..j-1 in ascending order, so each q_ij is the true substitution value (no explicit R^{-1}).
// The thread's finished q_i,0..j-1 are kept in shared memory (column-major, conflict-free),
// the current R column block is staged in shared memory and read as a broadcast.
constexpr int TRSM_NB = 8;

__global__ void trsm_kernel(int64_t m, int n, const double* Z, int64_t ldz,  // Z may alias Q
                            const double* __restrict__ R, int64_t ldr, double* Q, int64_t ldq,
                            const int* info) {
  if (info != nullptr && *info != 0) return;
  extern __shared__ double sm[];
  const int T = blockDim.x, tid = threadIdx.x;
  double* Qs = sm;                       // [n][T]
  double* Rb = sm + (size_t)n * T;       // [(n + NB)][NB]
  const int64_t i = blockIdx.x * (int64_t)T + tid;
  const bool valid = i < m;
  for (int jb = 0; jb < n; jb += TRSM_NB) {
    __syncthreads();
    const int rows = jb + TRSM_NB;
    for (int e = tid; e < rows * TRSM_NB; e += T) {
      const int k = e / TRSM_NB, c = e - k * TRSM_NB;
      Rb[e] = (jb + c < n && k < n) ? R[(int64_t)(jb + c) * ldr + k] : 0.0;
    }
    __syncthreads();
    double s[TRSM_NB];
#pragma unroll
    for (int c = 0; c < TRSM_NB; ++c) s[c] = (valid && jb + c < n) ? Z[(int64_t)(jb + c) * ldz + i] : 0.0;
    for (int k = 0; k < jb; ++k) {
      const double qk = Qs[(size_t)k * T + tid];
      const double* rk = Rb + k * TRSM_NB;
#pragma unroll
      for (int c = 0; c < TRSM_NB; ++c) s[c] -= qk * rk[c];
    }
#pragma unroll
    for (int c = 0; c < TRSM_NB; ++c) {
      if (jb + c < n) {
        const double q = s[c] / Rb[(jb + c) * TRSM_NB + c];
        Qs[(size_t)(jb + c) * T + tid] = q;
#pragma unroll
        for (int c2 = c + 1; c2 < TRSM_NB; ++c2) s[c2] -= q * Rb[(jb + c) * TRSM_NB + c2];
        if (valid) Q[(int64_t)(jb + c) * ldq + i] = q;
      }
    }
  }
}

cudaError_t launch_trsm(int64_t m, int n, const double* Z, int64_t ldz, const double* R, int64_t ldr,
                        double* Q, int64_t ldq, const int* info, cudaStream_t s) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const size_t rb = (size_t)(n + TRSM_NB) * TRSM_NB * sizeof(double);
  int T = 128;
  while (T > 32 && (size_t)n * T * sizeof(double) + rb > (size_t)SMEM_MAX) T >>= 1;
  const size_t bytes = (size_t)n * T * sizeof(double) + rb;
  trsm_kernel<<<(unsigned)cdiv(m, T), T, bytes, s>>>(m, n, Z, ldz, R, ldr, Q, ldq, info);
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
