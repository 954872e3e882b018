// oqr_gram.cu -- K1 fused A-Gram, K4 Euclidean Gram, K1r deterministic slot reduction,
// and the Z packing pre-pass.  sm_100a, FP64 tensor path (mma.sync m8n8k4 -> SASS DMMA).
//
// K1 computes Algorithm 1 lines 1-2 (s2 "Stability Analysis of CHOLQR"):
//     B = A Z;  C = Z^T B,
// as  G = sum_I Z_I^T W_I  with  W_I = A_{I,:} Z  (I = panels of BM rows), never storing B.
// By bilinearity any split of the k-range of W_I is allowed, so each CTA takes an equal,
// contiguous range of (panel, k-block) units; at the end of each run on one panel it
// contracts the partial W_I it holds with Z_I^T into its private slot.  The slots are then
// summed in a fixed order (K1r), so G is bitwise reproducible for a given grid size.
//
// FP64 has no tcgen05 kind on sm_100a (ptxas rejects .kind::f64); the FP64 tensor pipe is
// reached through warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Operands are staged in
// shared memory by the bulk-copy engine (cp.async.bulk -> SASS UBLKCP) through an mbarrier
// ring fed by one producer warp; 8 consumer warps each own 8 rows of W_I in registers.
#include "oqr_internal.cuh"

namespace oqr {

// ------------------------------------------------------------------ PTX wrappers ---------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 1-D bulk copy global -> shared, completion signalled on an mbarrier (complete_tx).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// D = A * B + D on the FP64 tensor pipe.  A: 8x4 row (lane: row lane/4, col lane%4),
// B: 4x8 col (lane: row lane%4, col lane/4), D: 8x8 (lane: row lane/4, cols 2*(lane%4)+{0,1}).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------------ Z packing -------------
__global__ void pack_z_kernel(int64_t m, int n, int NP, const double* __restrict__ Z, int64_t ldz,
                              double* __restrict__ Zp, int64_t total) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int kk = (int)(e % ZS);
    const int64_t bl = e / ZS;
    const int l = (int)(bl % NP);
    const int64_t b = bl / NP;
    const int64_t row = b * BK + kk;
    double v = 0.0;
    if (kk < BK && row < m && l < n) v = Z[(int64_t)l * ldz + row];
    Zp[e] = v;
  }
}

cudaError_t launch_pack_z(int64_t m, int n, const double* Z, int64_t ldz, double* Zp, cudaStream_t s) {
  const int NP = 8 * (int)cdiv(n, 8);
  const int64_t total = zp_doubles(m, NP);
  int64_t blocks = cdiv(total, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  pack_z_kernel<<<(unsigned)blocks, 256, 0, s>>>(m, n, NP, Z, ldz, Zp, total);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ contraction -----------
// Slot += Z_I^T W for the 64-row panel starting at row0, where consumer warp `warp` holds
// W[row0 + warp*8 + lane/4, lt*8 + 2*(lane%4) + e] in acc[lt][e] (DMMA accumulator layout).
// Each warp contracts its own 8 rows on the tensor pipe; the 8 warp partials of each chunk of
// LG output tiles are summed through shared memory in warp order 0..7 (fixed order), and the
// sum is added to the CTA-private slot (written on the CTA's first segment).
template <int NT>
__device__ __forceinline__ void contract_panel(double (&acc)[NT][2], int64_t row0,
                                               const double* __restrict__ Zp, double* red,
                                               double* __restrict__ slot, bool first, int warp,
                                               int lane, int ctid) {
  constexpr int NP = NT * 8;
  // 1. Re-distribute W from accumulator layout to B-operand layout (rows = i, cols = l):
  //    wb[lt][h] = W[warp*8 + 4h + lane%4, lt*8 + lane/4].
  double wb[NT][2];
  const int e_sel = (lane >> 2) & 1;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int src = 16 * h + 4 * (lane & 3) + (lane >> 3);
#pragma unroll
    for (int lt = 0; lt < NT; ++lt) {
      const double v0 = __shfl_sync(0xffffffffu, acc[lt][0], src);
      const double v1 = __shfl_sync(0xffffffffu, acc[lt][1], src);
      wb[lt][h] = e_sel ? v1 : v0;
    }
  }
  // 2. A-operand rows = k, cols = i: Z[row0 + warp*8 + 4h + lane%4, kt*8 + lane/4].
  const int64_t r0 = row0 + warp * 8 + (lane & 3);
  const int64_t r1 = r0 + 4;
  const double* z0 = Zp + ((r0 / BK) * NP + (lane >> 2)) * ZS + (r0 % BK);
  const double* z1 = Zp + ((r1 / BK) * NP + (lane >> 2)) * ZS + (r1 % BK);
  constexpr int NG = (NT + LG - 1) / LG;
#pragma unroll 1
  for (int kt = 0; kt < NT; ++kt) {
    const double za0 = z0[kt * 8 * ZS];
    const double za1 = z1[kt * 8 * ZS];
#pragma unroll
    for (int lg = 0; lg < NG; ++lg) {
#pragma unroll
      for (int j = 0; j < LG; ++j) {
        const int lt = lg * LG + j;
        if (lt < NT) {
          double o[2] = {0.0, 0.0};
          dmma(o, za0, wb[lt][0]);
          dmma(o, za1, wb[lt][1]);
          *reinterpret_cast<double2*>(red + (warp * LG + j) * 64 + lane * 2) = make_double2(o[0], o[1]);
        }
      }
      // this thread's output entry of the chunk (LG*64 == NCW*32: exactly one per thread);
      // its previous slot value is fetched before the barrier so the L2 latency overlaps it
      static_assert(LG * 64 == NCW * 32, "one chunk entry per consumer thread");
      const int v = ctid;
      const int j = v >> 6;
      const int lt = lg * LG + j;
      const int t = (v & 63) >> 1, e = v & 1;
      double* p = slot + (int64_t)(lt * 8 + 2 * (t & 3) + e) * NP + kt * 8 + (t >> 2);
      const double prev = (!first && lt < NT) ? *p : 0.0;
      named_bar_sync(1, NCW * 32);
      if (lt < NT) {
        double s = red[j * 64 + (v & 63)];
#pragma unroll
        for (int w = 1; w < NCW; ++w) s += red[(w * LG + j) * 64 + (v & 63)];
        *p = first ? s : (prev + s);
      }
      named_bar_sync(1, NCW * 32);
    }
  }
}

// ------------------------------------------------------------------ K1 --------------------
// Fill ring slot `s` with unit u = (panel I, k-block kb): BK columns of A (rows I*BM..+BM, one
// 512 B bulk copy per column into a padded smem column) and the packed Z block kb (one bulk
// copy).  Executed by all 32 lanes of warp 0.
// Ragged tiles (last panel / last k-block when m is not a multiple of BM / BK): only the valid
// rows and columns are copied; the rest of the slot keeps finite stale data (the ring is zeroed
// at kernel start), which only ever meets the zero rows of the packed Z (rows >= m), so it adds
// exactly 0.  Bulk copies move multiples of 16 B, so an odd count of valid rows copies one row
// fewer and the last row is loaded with plain loads.  When A's columns are not 16-byte aligned
// (odd lda or an 8-byte aligned A) every tile is loaded with plain loads (correct, slow).
template <int NT>
__device__ __forceinline__ void issue_stage(int64_t u, int64_t KB, int64_t m, const double* __restrict__ A,
                                            int64_t lda, const double* __restrict__ Zp, double* As,
                                            uint64_t* bar, int lane, uint64_t pol_a, uint64_t pol_z,
                                            bool bulk_ok) {
  constexpr int NP = NT * 8;
  constexpr uint32_t zbytes = NP * ZS * 8;
  const int64_t I = u / KB, kb = u - I * KB;
  const int64_t row0 = I * BM, col0 = kb * BK;
  double* Zs = As + BK * AS;
  const double* zsrc = Zp + kb * (int64_t)(NP * ZS);
  const int rows = (int)(m - row0 < BM ? m - row0 : BM);
  const int cols = (int)(m - col0 < BK ? m - col0 : BK);
  if (bulk_ok) {
    const int rows_bulk = rows & ~1;
    if (rows_bulk != rows && lane < cols)  // odd valid-row count: last row by plain loads
      As[lane * AS + rows - 1] = A[(col0 + lane) * lda + row0 + rows - 1];
    fence_proxy_async_smem();  // order these generic writes before later bulk writes to the slot
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(bar, zbytes + (uint32_t)(cols * rows_bulk * 8));
    __syncwarp();
    if (lane < cols && rows_bulk > 0)
      bulk_g2s(As + lane * AS, A + (col0 + lane) * lda + row0, rows_bulk * 8, bar, pol_a);
    else if (lane == BK)
      bulk_g2s(Zs, zsrc, zbytes, bar, pol_z);
  } else {
    for (int e = lane; e < BK * BM; e += 32) {
      const int k = e / BM, r = e - k * BM;
      double v = 0.0;
      if (r < rows && k < cols) v = A[(col0 + k) * lda + row0 + r];
      As[k * AS + r] = v;
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive_expect_tx(bar, zbytes);
      bulk_g2s(Zs, zsrc, zbytes, bar, pol_z);
    }
  }
  __syncwarp();
}

// 8 warps, one CTA per SM (2 warps per SM sub-partition => up to 255 registers per thread).
// Every warp owns 8 rows of W_I (all NP columns) in DMMA accumulators.  Warp 0 fills the ring
// initially; afterwards whichever warp releases slot s last refills it with the unit `stages`
// ahead, so `stages - 1` stages of compute cover the copy latency.
template <int NT>
__global__ void __launch_bounds__(NCW * 32, 1)
gram_fused_kernel(int64_t m, const double* __restrict__ A, int64_t lda, const double* __restrict__ Zp,
                  double* __restrict__ P, int64_t KB, int64_t U, int stages, bool bulk_ok) {
  constexpr int NP = NT * 8;
  constexpr int STAGE = BK * AS + NP * ZS;  // doubles per pipeline stage
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  unsigned* relcnt = reinterpret_cast<unsigned*>(empty + 8);  // 8 release counters (32 B)
  double* red = reinterpret_cast<double*>(smem + 192);
  double* ring = red + NCW * LG * 64;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = gridDim.x, c = blockIdx.x;
  const int64_t u0 = U * c / g, u1 = U * (c + 1) / g;

  // zero the ring once: slots of ragged tiles keep finite data outside their valid region
  for (int e = threadIdx.x; e < stages * STAGE; e += blockDim.x) ring[e] = 0.0;
  fence_proxy_async_smem();  // generic zero-fill before the async-proxy (bulk) writes
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
      relcnt[s] = 0u;
    }
    mbar_fence_init();
  }
  __syncthreads();

  const uint64_t pol_a = policy_evict_first();  // A is streamed exactly once
  const uint64_t pol_z = policy_evict_last();   // Zp is re-read by every panel
  if (warp == 0) {
    for (int s = 0; s < stages && u0 + s < u1; ++s)
      issue_stage<NT>(u0 + s, KB, m, A, lda, Zp, ring + s * STAGE, &full[s], lane, pol_a, pol_z, bulk_ok);
  }

  double* slot = P + c * (int64_t)NP * NP;
  double acc[NT][2];
#pragma unroll
  for (int lt = 0; lt < NT; ++lt) acc[lt][0] = acc[lt][1] = 0.0;
  bool first = true;
  int s = 0;
  uint32_t ph = 0;
  const int a_off = (lane & 3) * AS + warp * 8 + (lane >> 2);
  const int b_off = (lane >> 2) * ZS + (lane & 3);
  for (int64_t u = u0; u < u1; ++u) {
    mbar_wait(&full[s], ph);
    const double* As = ring + s * STAGE;
    const double* Zs = As + BK * AS;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const double a = As[kk * 4 * AS + a_off];
#pragma unroll
      for (int lt = 0; lt < NT; ++lt) {
        const double b = Zs[lt * 8 * ZS + kk * 4 + b_off];
        dmma(acc[lt], a, b);
      }
    }
    __syncwarp();
    // release the slot; the LAST warp to release it refills it at once (no warp is paced by
    // another's compute).  The arrival counter only elects that warp; the empty mbarrier's
    // acquire then orders all eight warps' reads of the slot before the new bulk writes.
    int last = 0;
    if (lane == 0) {
      mbar_arrive(&empty[s]);
      last = (atomicAdd(&relcnt[s], 1u) % NCW) == NCW - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last && u + stages < u1) {
      mbar_wait(&empty[s], ph);
      issue_stage<NT>(u + stages, KB, m, A, lda, Zp, ring + s * STAGE, &full[s], lane, pol_a, pol_z, bulk_ok);
    }
    if (++s == stages) {
      s = 0;
      ph ^= 1;
    }
    const int64_t I = u / KB;
    if (u + 1 == u1 || (u + 1) / KB != I) {
      contract_panel<NT>(acc, I * BM, Zp, red, slot, first, warp, lane, threadIdx.x);
      first = false;
#pragma unroll
      for (int lt = 0; lt < NT; ++lt) acc[lt][0] = acc[lt][1] = 0.0;
    }
  }
}

// ------------------------------------------------------------------ K4 --------------------
// G_E = Z^T Z = sum_I Z_I^T Z_I (PRE-CHOLQR pre-step as Cholesky-QR, reading R2).  Each CTA
// takes a contiguous range of 64-row panels; W is Z_I itself, loaded in accumulator layout.
template <int NT>
__global__ void __launch_bounds__(NCW * 32, 1)
gram_euclid_kernel(const double* __restrict__ Zp, int64_t npanels, double* __restrict__ P) {
  constexpr int NP = NT * 8;
  __shared__ __align__(16) double red[NCW * LG * 64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = gridDim.x, c = blockIdx.x;
  const int64_t p0 = npanels * c / g, p1 = npanels * (c + 1) / g;
  double* slot = P + c * (int64_t)NP * NP;
  bool first = true;
  for (int64_t I = p0; I < p1; ++I) {
    const int64_t r = I * BM + warp * 8 + (lane >> 2);
    const double* zr = Zp + ((r / BK) * NP + 2 * (lane & 3)) * ZS + (r % BK);
    double acc[NT][2];
#pragma unroll
    for (int lt = 0; lt < NT; ++lt) {
      acc[lt][0] = zr[(lt * 8) * ZS];
      acc[lt][1] = zr[(lt * 8 + 1) * ZS];
    }
    contract_panel<NT>(acc, I * BM, Zp, red, slot, first, warp, lane, threadIdx.x);
    first = false;
  }
}

// ------------------------------------------------------------------ K1r -------------------
// G[k, l] = sum_{c=0}^{g-1} P[c][l*NP + k], c ascending (fixed order => reproducible bits).
__global__ void gram_reduce_kernel(int n, int NP, int g, const double* __restrict__ P,
                                   double* __restrict__ G, int64_t ldg) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  const int l = (int)(idx / n), k = (int)(idx - (int64_t)l * n);
  const double* p = P + (int64_t)l * NP + k;
  const int64_t stride = (int64_t)NP * NP;
  double s = p[0];
  for (int c = 1; c < g; ++c) s += p[c * stride];
  G[(int64_t)l * ldg + k] = s;
}

cudaError_t launch_gram_reduce(int n, int g, const double* P, double* G, int64_t ldg, cudaStream_t s) {
  const int NP = 8 * (int)cdiv(n, 8);
  const int64_t total = (int64_t)n * n;
  gram_reduce_kernel<<<(unsigned)cdiv(total, 128), 128, 0, s>>>(n, NP, g, P, G, ldg);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ dispatch --------------
static int num_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

int gram_grid(int64_t /*m*/) { return num_sms(); }

size_t slots_doubles(int n, int g) {
  const size_t NP = 8 * (size_t)cdiv(n, 8);
  return (size_t)g * NP * NP;
}

static int fused_stages(int NT, size_t* bytes) {
  const size_t stage = (size_t)(BK * AS + NT * 8 * ZS) * 8;
  const size_t fixed = 192 + (size_t)NCW * LG * 64 * 8;
  int st = (int)((SMEM_MAX - fixed) / stage);
  if (st > 8) st = 8;
  *bytes = fixed + st * stage;
  return st;
}

template <int NT>
static cudaError_t gram_fused_nt(int64_t m, const double* A, int64_t lda, const double* Zp, double* P,
                                 int* g_out, cudaStream_t s) {
  size_t bytes;
  const int stages = fused_stages(NT, &bytes);
  static bool attr_done = false;  // per instantiation
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(gram_fused_kernel<NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int64_t KB = cdiv(m, BK), U = cdiv(m, BM) * KB;
  int64_t g = num_sms();
  if (g > U) g = U;
  *g_out = (int)g;
  timing_begin(s);
  const bool bulk_ok = (lda % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0);
  gram_fused_kernel<NT><<<(unsigned)g, NCW * 32, bytes, s>>>(m, A, lda, Zp, P, KB, U, stages, bulk_ok);
  note_launch();
  cudaError_t e = cudaGetLastError();
  timing_end(s);
  return e;
}

template <int NT>
static cudaError_t gram_euclid_nt(int64_t m, const double* Zp, double* P, int* g_out, cudaStream_t s) {
  const int64_t np = cdiv(m, BM);
  int64_t g = num_sms();
  if (g > np) g = np;
  *g_out = (int)g;
  gram_euclid_kernel<NT><<<(unsigned)g, NCW * 32, 0, s>>>(Zp, np, P);
  note_launch();
  return cudaGetLastError();
}

#define OQR_NT_CASES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) \
  X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30)

cudaError_t launch_gram_fused(int64_t m, int n, const double* A, int64_t lda, const double* Zp,
                              double* P, int* g_out, cudaStream_t s) {
  switch ((int)cdiv(n, 8)) {
#define OQR_CASE(NT) \
  case NT: return gram_fused_nt<NT>(m, A, lda, Zp, P, g_out, s);
    OQR_NT_CASES(OQR_CASE)
#undef OQR_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gram_euclid(int64_t m, int n, const double* Zp, double* P, int* g_out, cudaStream_t s) {
  switch ((int)cdiv(n, 8)) {
#define OQR_CASE(NT) \
  case NT: return gram_euclid_nt<NT>(m, Zp, P, g_out, s);
    OQR_NT_CASES(OQR_CASE)
#undef OQR_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace oqr
