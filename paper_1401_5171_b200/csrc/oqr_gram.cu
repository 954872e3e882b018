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
// shared memory through an mbarrier ring: the A tile (64 rows x KS = 32 or 64 columns) by ONE
// tensor TMA request over a 4-D view of A that lands it bank-conflict-free (SASS UTMALDG;
// out-of-bounds rows/columns are zero-filled by the hardware; see ALAY_*), the packed Z block by
// one 1-D bulk copy (SASS UBLKCP).  16 warps per CTA (8 row groups x 2 column halves) keep W_I
// in DMMA accumulators.  Also here: K4' (packed tall-skinny Grams, full and upper-triangle),
// the tiled packing kernel and K1r.
#include <cuda.h>  // CUtensorMap and its enums (the encode entry point is fetched at run time)

#include <cstdlib>
#include <cstring>

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
// 2-D tensor TMA global -> shared (box of the tensor map at coordinates {c0, c1}).
__device__ __forceinline__ void tma_g2s_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                           uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_g2s_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                           uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_g2s_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                           uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// D = A * B + D on the FP64 tensor pipe.  A: 8x4 row (lane: row lane/4, col lane%4),
// B: 4x8 col (lane: row lane%4, col lane/4), D: 8x8 (lane: row lane/4, cols 2*(lane%4)+{0,1}).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
#ifdef OQR_EXP_NODMMA  // experiment build only (tools/exp): keeps the operand loads, drops DMMA
  d[0] += a;
  d[1] += b;
  return;
#endif
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// D = A * B + D when `on` (warp-uniform), as ONE predicated instruction -- no branch around the
// mma.sync (a branch costs a WARPSYNC and keeps the compiler from hoisting the operand loads).
__device__ __forceinline__ void dmma_if(double (&d)[2], double a, double b, bool on) {
#ifdef OQR_EXP_NODMMA
  if (on) {
    d[0] += a;
    d[1] += b;
  }
  return;
#endif
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@p mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n\t}"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b), "r"((int)on));
}

// ------------------------------------------------------------------ Z packing -------------
// Zp[((b*NT + lt)*4 + kk)*32 + ln] = Z[b*BK + kk*4 + ln%4, lt*8 + ln/4] (zero outside Z).
// Packing through shared memory: a CTA stages a 64-row x 32-column tile of Z (plus one halo row
// above and below for the stencil) with coalesced column reads, then writes the tile's 4 x 4
// fragment groups of Zp (and W = T Z) as contiguous 1 KiB runs.  TRI: also W, w_il =
// e_{i-1} z_{i-1,l} + d_i z_il + e_i z_{i+1,l} (fma order as the per-element kernel).
#ifndef OQR_EXP_PT_C
#define OQR_EXP_PT_C 32
#endif
constexpr int PT_R = 64, PT_C = OQR_EXP_PT_C;
template <bool TRI>
__global__ void __launch_bounds__(256)
pack_tile_kernel(int64_t m, int n, int NT, const double* __restrict__ Z, int64_t ldz, double* __restrict__ Zp,
                 double* __restrict__ Wp, const double* __restrict__ d, const double* __restrict__ e, double scale,
                 int64_t nrt) {
  __shared__ double zs[PT_C][PT_R + 3];
  __shared__ double ds[PT_R], es[PT_R + 1];
  const int nct = (NT * 8 + PT_C - 1) / PT_C;
  for (int64_t tile = blockIdx.x; tile < nrt * nct; tile += gridDim.x) {
    const int64_t rt = tile / nct;
    const int ct = (int)(tile - rt * nct);
    const int64_t r0 = rt * PT_R;
    const int c0 = ct * PT_C;
    __syncthreads();  // previous tile's readers are done
    {  // all of this thread's loads in flight before the first shared-memory store
      constexpr int NQ = (PT_C * (PT_R + 2) + 255) / 256;
      double v[NQ];
#pragma unroll
      for (int u = 0; u < NQ; ++u) {
        const int q = threadIdx.x + u * 256;
        const int c = q / (PT_R + 2), rr = q - c * (PT_R + 2);
        const int64_t row = r0 + rr - 1;
        const int col = c0 + c;
        v[u] = (q < PT_C * (PT_R + 2) && row >= 0 && row < m && col < n) ? Z[(int64_t)col * ldz + row] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < NQ; ++u) {
        const int q = threadIdx.x + u * 256;
        if (q < PT_C * (PT_R + 2)) zs[q / (PT_R + 2)][q % (PT_R + 2)] = v[u];
      }
    }
    if (TRI) {
      for (int q = threadIdx.x; q < PT_R + 1; q += blockDim.x) {
        const int64_t row = r0 + q - 1;  // es[q] = e_{r0+q-1} (the coupling of rows r0+q-1, r0+q)
        es[q] = (row >= 0 && row < m - 1) ? e[row] : 0.0;
        if (q < PT_R) ds[q] = (r0 + q < m) ? d[r0 + q] : 0.0;
      }
    }
    __syncthreads();
    // 4 row blocks x 4 column tiles, 128 doubles each: o -> (block, tile, kk, lane)
    for (int o = threadIdx.x; o < (PT_R / BK) * (PT_C / 8) * 4 * FRAG; o += blockDim.x) {
      const int grp = o >> 7, w = o & 127;
      const int bl = grp / (PT_C / 8), tl = grp % (PT_C / 8);
      const int kk = w >> 5, ln = w & 31;
      const int r = bl * BK + kk * 4 + (ln & 3);  // tile-local row
      const int c = tl * 8 + (ln >> 2);           // tile-local column
      const int64_t b = r0 / BK + bl;
      const int lt = c0 / 8 + tl;
      if (lt >= NT) continue;
      const int64_t dst = ((b * NT + lt) * 4 + kk) * FRAG + ln;
      const double zv = zs[c][r + 1];
      if (TRI) {
        double wv = es[r] * zs[c][r];
        wv = fma(ds[r], zv, wv);
        wv = fma(es[r + 1], zs[c][r + 2], wv);
        Zp[dst] = zv;
        Wp[dst] = (r0 + r < m) ? wv : 0.0;
      } else {
        Zp[dst] = scale * zv;
      }
    }
  }
}

cudaError_t launch_pack_z(int64_t m, int n, const double* Z, int64_t ldz, double* Zp, cudaStream_t s, double scale) {
  const int NT = (int)cdiv(n, 8);
  const int64_t nrt = cdiv(zp_blocks(m) * BK, PT_R);  // Zp is padded to whole 64-row panels
  int64_t grid = nrt * cdiv(NT * 8, PT_C);
  if (grid > 148 * 8) grid = 148 * 8;
  pack_tile_kernel<false><<<(unsigned)grid, 256, 0, s>>>(m, n, NT, Z, ldz, Zp, nullptr, nullptr, nullptr, scale, nrt);
  note_launch();
  return cudaGetLastError();
}

// Zp and W = T Z for T = tridiag(e, d, e) (NEXT-N3) in one pass over Z, both written straight into
// the packed fragment order (the A and B operands of the packed Gram kernel): pack_tile_kernel<true>.
cudaError_t launch_pack_zw_tridiag(int64_t m, int n, const double* d, const double* e, const double* Z, int64_t ldz,
                                   double* Zp, double* Wp, cudaStream_t s) {
  const int NT = (int)cdiv(n, 8);
  const int64_t nrt = cdiv(zp_blocks(m) * BK, PT_R);
  int64_t grid = nrt * cdiv(NT * 8, PT_C);
  if (grid > 148 * 8) grid = 148 * 8;
  pack_tile_kernel<true><<<(unsigned)grid, 256, 0, s>>>(m, n, NT, Z, ldz, Zp, Wp, d, e, 1.0, nrt);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ contraction -----------
// Slot += Z_I^T W for the 64-row panel starting at row0.  Warp (rg, ch) holds, in DMMA
// accumulator layout, W[row0 + rg*8 + lane/4, (ch*NTW + t)*8 + 2*(lane%4) + e] in acc[t][e]
// for its NTW local n-tiles t.  Each warp contracts its own 8 rows on the tensor pipe; the 8
// row-group partials of every output entry are summed through shared memory in row-group order
// 0..7 (fixed order => reproducible bits), and the sum is added to the CTA-private slot (written
// on the CTA's first segment).  One chunk = output tile-row kt x LG local tiles of both halves
// = NCH*LG*64 = 512 entries, one per thread.
template <int NT>
__device__ __forceinline__ void contract_panel(double (&acc)[(NT + 1) / 2][2], int64_t row0,
                                               const double* __restrict__ Zp, double* red,
                                               double* __restrict__ slot, bool first, int rg, int ch,
                                               int lane, int ctid) {
  constexpr int NP = NT * 8;
  constexpr int NTW = (NT + 1) / 2;
  static_assert(NCH * LG * 64 <= NCW * 32, "at most one chunk entry per thread");
#ifdef OQR_EXP_NOCONTRACT  // experiment build only (tools/exp): measures the contraction's share
  {
    double t = 0.0;  // consume every accumulator (else ptxas drops the DMMAs)
#pragma unroll
    for (int i = 0; i < NTW; ++i) t += acc[i][0] + acc[i][1];
    slot[ctid] = first ? t : slot[ctid] + t;
    return;
  }
#endif
  // 1. Re-distribute W from accumulator layout to B-operand layout (rows = i, cols = l):
  //    wb[t][h] = W[rg*8 + 4h + lane%4, (ch*NTW + t)*8 + lane/4].
  double wb[NTW][2];
  const int e_sel = (lane >> 2) & 1;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int src = 16 * h + 4 * (lane & 3) + (lane >> 3);
#pragma unroll
    for (int t = 0; t < NTW; ++t) {
      const double v0 = __shfl_sync(0xffffffffu, acc[t][0], src);
      const double v1 = __shfl_sync(0xffffffffu, acc[t][1], src);
      wb[t][h] = e_sel ? v1 : v0;
    }
  }
  // 2. A operand (rows = k, cols = i): Z[row0 + rg*8 + 4h + lane%4, kt*8 + lane/4], which in the
  //    fragment-ordered Zp is lane `lane` of fragment (block r/BK, n-tile kt, k-step (r%BK)/4).
  const int64_t r0 = row0 + rg * 8, r1 = r0 + 4;
  const double* z0 = Zp + (((r0 / BK) * NT) * 4 + (r0 % BK) / 4) * FRAG + lane;
  const double* z1 = Zp + (((r1 / BK) * NT) * 4 + (r1 % BK) / 4) * FRAG + lane;
  constexpr int NG = (NTW + LG - 1) / LG;
  // this thread's entry of every chunk
  const bool has_entry = ctid < NCH * LG * 64;
  const int vch = ctid / (LG * 64), vj = (ctid >> 6) % LG, v64 = ctid & 63;
  const int vt = v64 >> 1, ve = v64 & 1;
  // this thread's slot entry of chunk (kt, lg): p_lg + 8 kt.  Its previous value and the next
  // tile-row's Z fragments are loaded one kt ahead (L2 latency off the per-chunk critical path).
  double* pbase = slot + (int64_t)(2 * (vt & 3) + ve) * NP + (vt >> 2);
  double pc[NG], pn[NG];
#pragma unroll
  for (int lg = 0; lg < NG; ++lg) {
    const int tl = lg * LG + vj, lt = vch * NTW + tl;
    const bool valid = has_entry && tl < NTW && lt < NT;
    pc[lg] = (!first && valid) ? pbase[(int64_t)lt * 8 * NP] : 0.0;
  }
  double za0 = z0[0], za1 = z1[0];
#pragma unroll 1
  for (int kt = 0; kt < NT; ++kt) {
    const bool more = kt + 1 < NT;
    const double zn0 = more ? z0[(kt + 1) * 4 * FRAG] : 0.0;
    const double zn1 = more ? z1[(kt + 1) * 4 * FRAG] : 0.0;
#pragma unroll
    for (int lg = 0; lg < NG; ++lg) {
      const int tl = lg * LG + vj, lt = vch * NTW + tl;
      const bool valid = has_entry && tl < NTW && lt < NT;
      pn[lg] = (!first && valid && more) ? pbase[(int64_t)lt * 8 * NP + (kt + 1) * 8] : 0.0;
    }
#pragma unroll
    for (int lg = 0; lg < NG; ++lg) {
#pragma unroll
      for (int j = 0; j < LG; ++j) {
        const int t = lg * LG + j;
        if (t < NTW && ch * NTW + t < NT) {
          double o[2] = {0.0, 0.0};
          dmma(o, za0, wb[t][0]);
          dmma(o, za1, wb[t][1]);
          *reinterpret_cast<double2*>(red + ((ch * NRG + rg) * LG + j) * 64 + lane * 2) =
              make_double2(o[0], o[1]);
        }
      }
      const int tl = lg * LG + vj;
      const int lt = vch * NTW + tl;
      const bool valid = has_entry && tl < NTW && lt < NT;
      __syncthreads();
      if (valid) {
        const double* rr = red + (vch * NRG * LG + vj) * 64 + v64;
        double s = rr[0];
#pragma unroll
        for (int g = 1; g < NRG; ++g) s += rr[g * LG * 64];
        pbase[(int64_t)lt * 8 * NP + kt * 8] = first ? s : (pc[lg] + s);
      }
      __syncthreads();
    }
#pragma unroll
    for (int lg = 0; lg < NG; ++lg) pc[lg] = pn[lg];
    za0 = zn0;
    za1 = zn1;
  }
}

// ------------------------------------------------------------------ K1 --------------------
// Unit schedule.  Dense: every panel I has KB k-blocks.  SYM (NEXT-N4, symmetric A): panel I only
// has the k-blocks of the block-lower triangle including its own 64 x 64 diagonal panel,
// nk(I) = min(KB, 4 (I + 1)), so the units before panel I number 2 I (I + 1) (only the last
// panel can be clipped).
// Stage width KS (columns of A per stage): every stage costs a fixed hand-off (barrier wait,
// release, refill election), so wide stages pay -- 64 columns for n <= 64 (there K1 is HBM- or
// hand-off-bound: 32 columns is 1.3x slower at n = 8..32), 32 above (16 is 2.5% slower at
// n = 200 and 8% for the symmetric schedule, although a 32-wide ring holds only 2-3 stages
// at n >= 200: tools/time_k1.py sweeps).  The packed Z layout keeps 16-row blocks
// (BK); a KS-wide stage moves KS/16 of them.  OQR_EXP_KS_* override the thresholds (experiments).
#ifndef OQR_EXP_KS_NT64
#define OQR_EXP_KS_NT64 8
#endif
#ifndef OQR_EXP_KS_NT32
#define OQR_EXP_KS_NT32 30
#endif
#ifndef OQR_EXP_PF32
#define OQR_EXP_PF32 22
#endif
__host__ __device__ constexpr int stage_k(int NT) {
  return NT <= OQR_EXP_KS_NT64 ? 64 : (NT <= OQR_EXP_KS_NT32 ? 32 : 16);
}

template <bool SYM, int KS>
__host__ __device__ __forceinline__ int unit_nk(int I, int KB) {
  return SYM ? min(KB, (I + 1) * (BM / KS)) : KB;
}
// Balanced split of the unit range over the CTAs: a panel costs its units plus one contraction
// (~panel_w units of time), so the split equalises W(u) = u + panel_w * (panels started before
// u) instead of u alone -- the symmetric schedule has panels of 4 .. KB units.  The contraction
// is ~NT times costlier than one unit relative to the unit's NT-proportional work, so
// panel_w = PANEL_W_PER_NT * NT (calibrated on B200 with tools/time_k1.py and -DOQR_EXP_PANEL_W builds).
constexpr double PANEL_W_PER_NT = 2.0;

// SYM: panel I has R (I + 1) units (R = BM / KS), so the units before panel I number R I (I+1)/2.
template <bool SYM, int KS>
__host__ __device__ __forceinline__ int unit_panels_before(int u, int KB) {  // panels starting at < u
  if (u <= 0) return 0;
  if (!SYM) return (u + KB - 1) / KB;
  constexpr long long R = BM / KS;
  int i = (int)((sqrt(8.0 * (double)u / (double)R + 1.0) - 1.0) * 0.5);
  while (R * (i + 1) * (i + 2) / 2 < (long long)u) ++i;     // largest i with start(i) < u
  while (i > 0 && R * i * (i + 1) / 2 >= (long long)u) --i;
  return i + 1;
}

template <bool SYM, int KS>
__device__ __forceinline__ int unit_split(int c, int g, int U, int KB, int npanels, double panel_w) {
  if (c <= 0) return 0;
  if (c >= g) return U;
  const double target = ((double)U + panel_w * npanels) * c / g;
  int lo = 0, hi = U;  // smallest u with W(u) >= target
  while (lo < hi) {
    const int mid = lo + (hi - lo) / 2;
    if ((double)mid + panel_w * unit_panels_before<SYM, KS>(mid, KB) >= target) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

template <bool SYM, int KS>
__host__ __device__ __forceinline__ void unit_locate(int u, int KB, int* I, int* kb) {
  if (!SYM) {
    *I = u / KB;
    *kb = u - *I * KB;
    return;
  }
  constexpr long long R = BM / KS;
  int i = (int)((sqrt(8.0 * (double)u / (double)R + 1.0) - 1.0) * 0.5);
  while (R * (i + 1) * (i + 2) / 2 <= (long long)u) ++i;
  while (i > 0 && R * i * (i + 1) / 2 > (long long)u) --i;
  *I = i;
  *kb = (int)(u - R * i * (i + 1) / 2);
}

// Shared-memory layouts of the 64 x KS A tile.  A warp's k-step reads rows rg*8 + 0..7 of four
// columns, each half warp rows 0..3 or 4..7 of them.
//  ALAY_R4  [row/4][col][row%4] (4-D tensor map): a half warp reads 16 consecutive doubles --
//           conflict-free; TMA moves 32-byte lines.  The default (rows % 8 == 0).
//  ALAY_R8  [row/8][col][row%8] (3-D map): 2-way bank conflict, 64-byte TMA lines.  n <= 8
//           only, where K1 is HBM-bound and the line rate of the 32-byte layout, not shared
//           memory, would limit it (tools/time_k1.py: 1.88 vs 2.15 ms at m = 40000, n = 8).
//  ALAY_COL column-major 64 x KS (2-D map), 4-way conflict; rows % 8 != 0 only.
constexpr int ALAY_COL = 0, ALAY_R8 = 1, ALAY_R4 = 2;

// Fill a ring slot with unit (panel I, k-block kb): the A tile A[I*BM.., kb*KS..] (64 x KS,
// column-major in smem) and the KS/16 packed Z blocks of the k-block (NT KiB each).  Executed by warp 0's lanes.
// With a tensor map (A 16-byte aligned, lda even) both are single async requests and ragged
// tiles need nothing special: TMA zero-fills rows/columns >= m.  Otherwise the A tile is loaded
// with plain loads and zero fill (correct, slow).
template <int NT, bool SYM, int KS>
__device__ __forceinline__ void issue_stage(int I, int kb, int64_t m, int64_t mr, const CUtensorMap* tmap,
                                            const double* __restrict__ A, int64_t lda,
                                            const double* __restrict__ Zp, const double* __restrict__ Zh,
                                            double* As, uint64_t* bar, int lane, uint64_t pol_a, uint64_t pol_z,
                                            bool tma_ok, int alay) {
  constexpr int ZB = KS / BK;                     // packed Z blocks per stage
  constexpr uint32_t zbytes = ZB * NT * 4 * FRAG * 8;
  constexpr uint32_t abytes = BM * KS * 8;
  const int64_t row0 = (int64_t)I * BM, col0 = (int64_t)kb * KS;
  double* Zs = As + BM * KS;
  // SYM: the diagonal panel's k-blocks (kb >= I BM/KS) use Z / 2 (exact): T = S + D/2, G = T + T^T
  const double* zsrc = ((SYM && kb >= I * (BM / KS)) ? Zh : Zp) + kb * (int64_t)(ZB * NT * 4 * FRAG);
#ifdef OQR_EXP_NOLOAD  // experiment build only (tools/exp): no copies, barrier still completes
  if (lane == 0) mbar_arrive(bar);
  __syncwarp();
  return;
#endif
  if (tma_ok) {
    if (lane == 0) {
      mbar_arrive_expect_tx(bar, abytes + zbytes);
      if (alay == ALAY_R4) tma_g2s_4d(As, tmap, 0, (int)col0, 0, (int)(row0 >> 3), bar, pol_a);
      else if (alay == ALAY_R8) tma_g2s_3d(As, tmap, 0, (int)col0, (int)(row0 >> 3), bar, pol_a);
      else tma_g2s_2d(As, tmap, (int)row0, (int)col0, bar, pol_a);
      bulk_g2s(Zs, zsrc, zbytes, bar, pol_z);
    }
  } else {
    for (int e = lane; e < KS * BM; e += 32) {
      const int k = e / BM, r = e - k * BM;
      double v = 0.0;
      if (row0 + r < mr && col0 + k < m) v = A[(col0 + k) * lda + row0 + r];
      As[alay == ALAY_R4 ? (((r >> 2) * KS + k) << 2) + (r & 3)
                         : (alay == ALAY_R8 ? (((r >> 3) * KS + k) << 3) + (r & 7) : e)] = v;
    }
    fence_proxy_async_smem();  // generic writes before later async-proxy writes to the slot
    __syncwarp();
    if (lane == 0) {
      mbar_arrive_expect_tx(bar, zbytes);
      bulk_g2s(Zs, zsrc, zbytes, bar, pol_z);
    }
  }
  __syncwarp();
}

// The DMMA loop of one warp over its unit range.  NTL (compile time) = this warp's n-tiles:
// NTW for the first column half, NT - NTW for the second (one less when NT is odd), so no
// DMMA is predicated.  Unit bookkeeping is incremental int32 (no division in the loop):
// (I, kb) is the unit being consumed, (Ii, kbi) the unit `stages` ahead that a refill loads.
template <int NT, int NTL, bool SYM, int KS>
__device__ __forceinline__ void consume_units(const CUtensorMap* tmap, int64_t m, int64_t mr,
                                              const double* __restrict__ A, int64_t lda,
                                              const double* __restrict__ Zp, const double* __restrict__ Zc,
                                              const double* __restrict__ Zh, double* slot,
                                              double* red, double* ring, uint64_t* full, uint64_t* empty,
                                              unsigned* relcnt, int KB, int u0, int u1, int stages,
                                              bool tma_ok, int alay, bool accum, int rg, int ch, int lane,
                                              uint64_t pol_a, uint64_t pol_z) {
  constexpr int NTW = (NT + 1) / 2;
  constexpr int ZB = KS / BK;
  constexpr int STAGE = BM * KS + ZB * NT * 4 * FRAG;
  static_assert(NTL <= NTW, "tile split");
  double acc[NTW][2];
#pragma unroll
  for (int t = 0; t < NTW; ++t) acc[t][0] = acc[t][1] = 0.0;
  bool first = !accum;  // accum: the slot already holds an earlier launch's partial (column chunks)
  int s = 0;
  uint32_t ph = 0;
  int I, kb;
  unit_locate<SYM, KS>(u0, KB, &I, &kb);
  int nk = unit_nk<SYM, KS>(I, KB);
  int ui = u0 + stages;  // next unit to be loaded into the slot being released
  int Ii, kbi;
  unit_locate<SYM, KS>(ui, KB, &Ii, &kbi);
  int nki = unit_nk<SYM, KS>(Ii, KB);
  // A fragment: A[row0 + rg*8 + lane/4, col0 + kk*4 + lane%4] (tile layouts: see ALAY_*)
  const int a_off = alay == ALAY_R4   ? (((2 * rg + (lane >> 4)) * KS + (lane & 3)) << 2) + ((lane >> 2) & 3)
                    : alay == ALAY_R8 ? ((rg * KS + (lane & 3)) << 3) + (lane >> 2)
                                      : (lane & 3) * BM + rg * 8 + (lane >> 2);
  const int a_step = alay == ALAY_R4 ? 16 : (alay == ALAY_R8 ? 32 : 4 * BM);  // doubles per k-step
  // B fragment (block zb, lt, kk): 32 consecutive doubles of the packed blocks
  const int b_off = BM * KS + ch * NTW * 4 * FRAG + lane;
  unsigned pend = 0u;  // lane 0: the previous release's counter value (elects the refiller)
  bool pvalid = false;
  int ps = 0, pIi = 0, pkbi = 0;
  uint32_t pph = 0;
  for (int u = u0; u < u1; ++u) {
    mbar_wait(&full[s], ph);
    const double* As = ring + s * STAGE;
    const double* Zs = As + b_off;
    double a_cur = As[a_off];
    double b_cur[NTL > 0 ? NTL : 1];
#pragma unroll
    for (int t = 0; t < NTL; ++t) b_cur[t] = Zs[t * 4 * FRAG];
    // the next k-step's fragments are prefetched while this one's DMMAs run -- except for
    // NT > 22 (KS = 32; 25 for KS = 16), where the second fragment set does not fit in 128
    // registers next to the accumulators (spills)
    constexpr bool PREFETCH = NT <= (KS == 16 ? 25 : OQR_EXP_PF32);
#pragma unroll
    for (int kk = 0; kk < KS / 4; ++kk) {
      double a_nxt = 0.0, b_nxt[NTL > 0 ? NTL : 1];
      if (!PREFETCH && kk > 0) {
        a_cur = As[kk * a_step + a_off];
#pragma unroll
        for (int t = 0; t < NTL; ++t) b_cur[t] = Zs[(((kk >> 2) * NT + t) * 4 + (kk & 3)) * FRAG];
      }
      if (PREFETCH && kk + 1 < KS / 4) {
        const int k1 = kk + 1, zb = k1 >> 2, k4 = k1 & 3;
        a_nxt = As[k1 * a_step + a_off];
#pragma unroll
        for (int t = 0; t < NTL; ++t) b_nxt[t] = Zs[((zb * NT + t) * 4 + k4) * FRAG];
      }
#pragma unroll
      for (int t = 0; t < NTL; ++t) dmma(acc[t], a_cur, b_cur[t]);
      if (PREFETCH && kk + 1 < KS / 4) {
        a_cur = a_nxt;
#pragma unroll
        for (int t = 0; t < NTL; ++t) b_cur[t] = b_nxt[t];
      }
    }
    // Release the slot; the LAST warp to release it refills it (no warp is paced by another's
    // compute).  The arrival counter only elects that warp; the empty mbarrier's acquire then
    // orders all warps' reads of the slot before the new async writes.  The election result is
    // read one unit later (after this warp's next DMMAs are issued), so the counter's round
    // trip is off the per-unit critical path; the refill lands stages - 2 units ahead.  Only for
    // NT <= 16 (short stages, where that round trip matters): the five extra live registers
    // would make the NT > 22 instantiations spill.
#ifndef OQR_EXP_DEFER_NT
#define OQR_EXP_DEFER_NT 16
#endif
    constexpr bool DEFER = NT <= OQR_EXP_DEFER_NT;
    if (!DEFER) {
      __syncwarp();
      unsigned cnt = 0u;
      if (lane == 0) {
        mbar_arrive(&empty[s]);
        cnt = atomicAdd(&relcnt[s], 1u);
      }
      cnt = __shfl_sync(0xffffffffu, cnt, 0);
      if ((cnt % NCW) == NCW - 1 && ui < u1) {
        mbar_wait(&empty[s], ph);
        issue_stage<NT, SYM, KS>(Ii, kbi, m, mr, tmap, A, lda, Zp, Zh, ring + s * STAGE, &full[s], lane, pol_a,
                                 pol_z, tma_ok, alay);
      }
    } else {
      const unsigned prev = __shfl_sync(0xffffffffu, pend, 0);
      if (pvalid && (prev % NCW) == NCW - 1) {
        mbar_wait(&empty[ps], pph);
        issue_stage<NT, SYM, KS>(pIi, pkbi, m, mr, tmap, A, lda, Zp, Zh, ring + ps * STAGE, &full[ps], lane, pol_a,
                                 pol_z, tma_ok, alay);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty[s]);
        pend = atomicAdd(&relcnt[s], 1u);
      }
      pvalid = ui < u1;
      ps = s;
      pph = ph;
      pIi = Ii;
      pkbi = kbi;
    }
    ++ui;
    if (++kbi == nki) {
      kbi = 0;
      ++Ii;
      nki = unit_nk<SYM, KS>(Ii, KB);
    }
    if (++s == stages) {
      s = 0;
      ph ^= 1;
    }
    const bool panel_end = (++kb == nk);
    if (panel_end || u + 1 == u1) {
      contract_panel<NT>(acc, (int64_t)I * BM, Zc, red, slot, first, rg, ch, lane, threadIdx.x);
      first = false;
#pragma unroll
      for (int t = 0; t < NTW; ++t) acc[t][0] = acc[t][1] = 0.0;
    }
    if (panel_end) {
      kb = 0;
      ++I;
      nk = unit_nk<SYM, KS>(I, KB);
    }
  }
}

// 16 warps, one CTA per SM (4 warps per SM sub-partition, <= 128 registers per thread).
// Warp (rg = warp % 8, ch = warp / 8) owns rows rg*8..rg*8+7 of W_I and n-tiles ch*NTW..; the
// operand fragments of k-step kk+1 are loaded while the DMMAs of k-step kk run.  Warp 0 fills
// the ring initially; afterwards whichever warp releases slot s last refills it with the unit
// `stages` ahead, so `stages - 1` stages of compute cover the copy latency.
template <int NT, bool SYM>
__global__ void __launch_bounds__(NCW * 32, 1)
gram_fused_kernel(const __grid_constant__ CUtensorMap tmap, int64_t m, int64_t mr, const double* __restrict__ A,
                  int64_t lda, const double* __restrict__ Zp, const double* __restrict__ Zc,
                  const double* __restrict__ Zh, double* __restrict__ P, int KB, int U, int stages, bool tma_ok, int alay,
                  double panel_w, bool accum) {
  constexpr int NP = NT * 8;
  constexpr int NTW = (NT + 1) / 2;
  constexpr int KS = stage_k(NT);
  constexpr int STAGE = BM * KS + (KS / BK) * NT * 4 * FRAG;  // doubles per pipeline stage
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  unsigned* relcnt = reinterpret_cast<unsigned*>(empty + 8);  // 8 release counters (32 B)
  double* red = reinterpret_cast<double*>(smem + 256);
  double* ring = red + NCH * NRG * LG * 64;  // 128-byte aligned (TMA destination)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rg = warp % NRG, ch = warp / NRG;
  const int g = gridDim.x, c = blockIdx.x;
  const int npanels = (int)cdiv(mr, BM);
  const int u0 = unit_split<SYM, KS>(c, g, U, KB, npanels, panel_w);
  const int u1 = unit_split<SYM, KS>(c + 1, g, U, KB, npanels, panel_w);
  if (u0 >= u1) {  // the weighted split can leave a CTA without units: its slot is zero
    double* slot = P + c * (int64_t)NP * NP;
    if (!accum)
      for (int e = threadIdx.x; e < NP * NP; e += blockDim.x) slot[e] = 0.0;
    return;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
      relcnt[s] = 0u;
    }
    mbar_fence_init();
    if (tma_ok) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  __syncthreads();

  const uint64_t pol_a = policy_evict_first();  // A is streamed exactly once
  const uint64_t pol_z = policy_evict_last();   // Zp is re-read by every panel
  if (warp == 0) {
    for (int s = 0; s < stages && u0 + s < u1; ++s) {
      int I, kb;
      unit_locate<SYM, KS>(u0 + s, KB, &I, &kb);
      issue_stage<NT, SYM, KS>(I, kb, m, mr, &tmap, A, lda, Zp, Zh, ring + s * STAGE, &full[s], lane, pol_a, pol_z,
                               tma_ok, alay);
    }
  }
  double* slot = P + c * (int64_t)NP * NP;
  if (ch == 0)
    consume_units<NT, NTW, SYM, KS>(&tmap, m, mr, A, lda, Zp, Zc, Zh, slot, red, ring, full, empty, relcnt, KB, u0,
                                u1, stages, tma_ok, alay, accum, rg, ch, lane, pol_a, pol_z);
  else
    consume_units<NT, NT - NTW, SYM, KS>(&tmap, m, mr, A, lda, Zp, Zc, Zh, slot, red, ring, full, empty, relcnt, KB,
                                     u0, u1, stages, tma_ok, alay, accum, rg, ch, lane, pol_a, pol_z);
}


// ------------------------------------------------------------------ K1r -------------------
// G[k, l] = sum_{c=0}^{g-1} P[c][l*NP + k], c ascending (fixed order => reproducible bits).
// sym (NEXT-N4): G = T + T^T with T = sum_c P[c], i.e. G[k,l] = T[k,l] + T[l,k] (bitwise symmetric).
__global__ void gram_reduce_kernel(int n, int NP, int g, const double* __restrict__ P,
                                   double* __restrict__ G, int64_t ldg, bool mirror) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int k, l;
  if (mirror) {  // one thread per upper entry k <= l (packed column order: coalesced slot reads)
    if (idx >= (int64_t)n * (n + 1) / 2) return;
    l = (int)((sqrt(8.0 * (double)idx + 1.0) - 1.0) * 0.5);
    while ((int64_t)l * (l + 1) / 2 > idx) --l;
    while ((int64_t)(l + 1) * (l + 2) / 2 <= idx) ++l;
    k = (int)(idx - (int64_t)l * (l + 1) / 2);
  } else {
    if (idx >= (int64_t)n * n) return;
    l = (int)(idx / n);
    k = (int)(idx - (int64_t)l * n);
  }
  const int64_t stride = (int64_t)NP * NP;
  const double* p = P + (int64_t)l * NP + k;
  // c ascending; loads issued eight at a time, added in order (the same bits as a plain loop)
  double s = p[0];
  int c = 1;
  for (; c + 8 <= g; c += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = p[(int64_t)(c + u) * stride];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; c < g; ++c) s += p[(int64_t)c * stride];
  G[(int64_t)l * ldg + k] = s;
  if (mirror && k != l) G[(int64_t)k * ldg + l] = s;
}

// sym (NEXT-N4): G holds T = sum_c P[c]; G[k,l] = G[l,k] = T[k,l] + T[l,k] for k <= l (the
// operand order of both entries is the upper one: bitwise symmetric).  One thread per pair.
__global__ void gram_symmetrize_kernel(int n, double* __restrict__ G, int64_t ldg) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * (n + 1) / 2) return;
  int l = (int)((sqrt(8.0 * (double)idx + 1.0) - 1.0) * 0.5);
  while ((int64_t)l * (l + 1) / 2 > idx) --l;
  while ((int64_t)(l + 1) * (l + 2) / 2 <= idx) ++l;
  const int k = (int)(idx - (int64_t)l * (l + 1) / 2);
  const double v = G[(int64_t)l * ldg + k] + G[(int64_t)k * ldg + l];
  G[(int64_t)l * ldg + k] = v;
  G[(int64_t)k * ldg + l] = v;
}

cudaError_t launch_gram_reduce(int n, int g, const double* P, double* G, int64_t ldg, cudaStream_t s, bool sym,
                               bool mirror) {
  const int NP = 8 * (int)cdiv(n, 8);
  const int64_t total = mirror ? (int64_t)n * (n + 1) / 2 : (int64_t)n * n;
  gram_reduce_kernel<<<(unsigned)cdiv(total, 128), 128, 0, s>>>(n, NP, g, P, G, ldg, mirror);
  note_launch();
  if (sym) {
    const int64_t pairs = (int64_t)n * (n + 1) / 2;
    gram_symmetrize_kernel<<<(unsigned)cdiv(pairs, 128), 128, 0, s>>>(n, G, ldg);
    note_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_sum_partials(int n, int count, const double* P, double* G, int64_t ldg, cudaStream_t s) {
  const int64_t total = (int64_t)n * n;
  gram_reduce_kernel<<<(unsigned)cdiv(total, 128), 128, 0, s>>>(n, n, count, P, G, ldg, false);
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
  const int KS = stage_k(NT);
  const size_t stage = (size_t)(BM * KS + (KS / BK) * NT * 4 * FRAG) * 8;
  const size_t fixed = 256 + (size_t)NCH * NRG * LG * 64 * 8;
  int st = (int)((SMEM_MAX - fixed) / stage);
  if (st > 8) st = 8;
  *bytes = fixed + st * stage;
  return st;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link needed).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// A (or a row block of it) as a 2-D FP64 tensor {rows mr (contiguous), cols m (stride lda)},
// box {BM, KS}, no swizzle,
// out-of-bounds elements zero-filled.
// The A tensor map for tile layout alay (ALAY_*): ALAY_R4 is the 4-D view (row % 4, col,
// (row / 4) % 2, row / 8) of the same matrix, strides {8 B, lda * 8 B, 32 B, 64 B} (not
// increasing -- the encoder accepts that, tools/tma3d_probe.cu), box (4, ks, 2, 8); ALAY_R8 the
// 3-D view (row % 8, col, row / 8), box (8, ks, 8); ALAY_COL the plain 2-D view, box (64, ks).
static bool make_tmap_a(CUtensorMap* map, const double* A, int64_t mr, int64_t m, int64_t lda, int ks, int alay) {
  if ((reinterpret_cast<uintptr_t>(A) & 15) != 0 || (lda & 1) != 0 || m > (int64_t)INT32_MAX) return false;
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  if (alay == ALAY_R8) {
    const cuuint64_t dims[3] = {8, (cuuint64_t)m, (cuuint64_t)(mr / 8)};
    const cuuint64_t strides[2] = {(cuuint64_t)lda * sizeof(double), 8 * sizeof(double)};
    const cuuint32_t box[3] = {8, (cuuint32_t)ks, (cuuint32_t)(BM / 8)};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(A), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  if (alay == ALAY_R4) {
    const cuuint64_t dims[4] = {4, (cuuint64_t)m, 2, (cuuint64_t)(mr / 8)};
    const cuuint64_t strides[3] = {(cuuint64_t)lda * sizeof(double), 4 * sizeof(double), 8 * sizeof(double)};
    const cuuint32_t box[4] = {4, (cuuint32_t)ks, 2, (cuuint32_t)(BM / 8)};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(A), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)mr, (cuuint64_t)m};
  const cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)BM, (cuuint32_t)ks};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NT, bool SYM>
static cudaError_t gram_fused_nt(int64_t m, int64_t mr, const double* A, int64_t lda, const double* Zp,
                                 const double* Zc, const double* Zh, double* P, int* g_out, cudaStream_t s,
                                 bool accum) {
  size_t bytes;
  const int stages = fused_stages(NT, &bytes);
  {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(gram_fused_kernel<NT, SYM>), (int)bytes);
    if (e != cudaSuccess) return e;
  }
  constexpr int KS = stage_k(NT);
  const int64_t KB = cdiv(m, KS), NPAN = cdiv(mr, BM);
  // U < 2^31 for every m that fits in HBM.  SYM: R P (P - 1)/2 units before the last panel.
  const int64_t R = BM / KS;
  const int64_t U = SYM ? R * (NPAN - 1) * NPAN / 2 + unit_nk<true, KS>((int)(NPAN - 1), (int)KB) : NPAN * KB;
  if (U > (int64_t)INT32_MAX - 64) return cudaErrorInvalidValue;
  int64_t g = num_sms();
  if (g > U) g = U;
  *g_out = (int)g;
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  const int alay = (mr % 8) != 0 ? ALAY_COL : (NT == 1 ? ALAY_R8 : ALAY_R4);
  const bool tma_ok = make_tmap_a(&tmap, A, mr, m, lda, KS, alay);
  timing_begin(s, OQR_TIMING_K1);
  // panel weight in units: a unit carries KS/16 times the work of a 16-wide unit.  (Experiment
  // builds may override the weight at compile time, -DOQR_EXP_PANEL_W=<w>: it changes the unit
  // split and so the summation order; the product build has no run-time knob, so results are
  // bitwise reproducible for a given (m, n, SM count) as include/oqr.h states.)
#ifdef OQR_EXP_PANEL_W
  const double panel_w = OQR_EXP_PANEL_W;
#else
  const double panel_w = PANEL_W_PER_NT * NT * (16.0 / KS);
#endif
  gram_fused_kernel<NT, SYM><<<(unsigned)g, NCW * 32, bytes, s>>>(tmap, m, mr, A, lda, Zp, Zc, Zh, P, (int)KB,
                                                                  (int)U, stages, tma_ok, alay, panel_w, accum);
  note_launch();
  cudaError_t e = cudaGetLastError();
  timing_end(s);
  return e;
}

// ------------------------------------------------------------------ K4 family -------------
// Upper triangle of a tall-skinny Gram that is symmetric in exact arithmetic, G = sum_b X_b^T Y_b
// over 16-row blocks b: the Euclidean Gram Z^T Z of the PRE-CHOLQR pre-step (north_star (4),
// reading R2; X = Y = Z) and the tridiagonal Gram Z^T (T Z) (NEXT-N3; Y = T Z).  K2 reads only the
// upper triangle; the reduction mirrors it (launch_gram_reduce(..., mirror = true)).  Three
// operand sources, one DMMA schedule:
//   UPK_EUCLID  (K4e) Z read ONCE from the caller's column-major array: one 2-D tensor-TMA request
//               per block lands the 20 x NP box of Z starting at row 16 b - 2 as [column][20 rows]
//               (the 20-double column stride makes every A- and B-fragment load conflict-free; an
//               even start row is what TMA requires, tools/tma_halo_probe.cu), rows outside
//               0..m-1 and columns >= n zero-filled.  No packed copy of Z through HBM.
//   UPK_TRI     (K4t) the same box; two producer warps form W = T Z for the block in B-fragment
//               order in a ring of W buffers (the packing kernel's arithmetic, PAPER.md:957-961
//               workload, reading R18) while the consumers run earlier blocks' DMMAs -- no packed Z
//               or T Z through HBM.
//   UPK_PACKED  (K4') Xp, Yp already packed in fragment order (the fallback when TMA cannot
//               describe Z: odd ldz or 8-byte alignment), one bulk copy each (one when X = Y).
// Schedule (round 2): tile rows are taken in PAIRS (2p, 2p+1); a unit is one tile column l >= 2p
// of a pair -- two 8x8 output tiles sharing the unit's B fragment (the lower tile (2p+1, 2p) is
// skipped).  Consumer warps own contiguous runs of at most C units (at most two pairs per warp)
// in DMMA accumulators, so per k-step a warp loads 2-4 A fragments and one B fragment per unit
// for up to 2 DMMAs each: about 0.6 fragment loads per DMMA instead of the one-row schedule's
// 1.08.  One producer lane refills the ring; stages and W buffers are handed over through mbarriers
// (full: TMA landed / W formed by every consumer; empty: every consumer warp done), no CTA barrier.
// Each warp runs a code path compiled for its exact unit count (no predicated-off DMMA: on the
// FP64 pipe a predicated-off DMMA still takes its issue slot).
// The per-tile k order (blocks ascending, k-steps ascending) is the same for every source: for a
// given K-slice split the three produce bitwise the same slots (tested).
enum { UPK_PACKED = 0, UPK_EUCLID = 1, UPK_TRI = 2 };
constexpr int TRB = 20;      // rows per Z box: 2 halo rows above, the block's 16, 2 halo rows below
constexpr int TRH = 2;       // halo rows above (the box starts at the even row 16 b - 2)
#ifndef OQR_EXP_UP_MAXC  // experiment builds only (tools/exp)
#define OQR_EXP_UP_MAXC 6
#endif
constexpr int UP_MAXC = OQR_EXP_UP_MAXC;  // units per consumer warp, at most (accumulators: 8 C registers)
constexpr int UP_MAXW = 24;  // consumer warps per CTA part, at most
__host__ __device__ constexpr int up_units(int NT) {  // sum over pairs p of (NT - 2p)
  return ((NT + 1) / 2) * NT - ((NT + 1) / 2) * ((NT + 1) / 2 - 1);
}
// CTA parts per K-slice: at most 96 units per part, so that ~12 consumer warps of <= 8 units hold
// the accumulators (8 registers per lane per unit) in ~128 registers per thread without spilling;
// n > 144 splits the tiles over two CTA parts on two SMs, n > 208 over three
#ifndef OQR_EXP_UP_PART_UNITS  // experiment builds only (tools/exp): units per CTA part, at most
#define OQR_EXP_UP_PART_UNITS 96
#endif
#ifndef OQR_EXP_UP_WARPS       // experiment builds only: consumer warps aimed at per part
#define OQR_EXP_UP_WARPS 16
#endif
#ifndef OQR_EXP_UP_TRI_WARPS   // experiment builds only: the same for UPK_TRI
#define OQR_EXP_UP_TRI_WARPS 11
#endif
__host__ __device__ constexpr int up_parts(int NT) {
  return (up_units(NT) + OQR_EXP_UP_PART_UNITS - 1) / OQR_EXP_UP_PART_UNITS;
}
__host__ __device__ constexpr int up_part_units(int NT) { return (up_units(NT) + up_parts(NT) - 1) / up_parts(NT); }
// units per warp: about 16 consumer warps per part (4 per SM sub-partition), 2..UP_MAXC units each;
// UPK_TRI: about 11 on three sub-partitions, up to 9 units each (its producers own the fourth)
__host__ __device__ constexpr int up_maxc(int MODE) { return MODE == UPK_TRI ? 9 : UP_MAXC; }
__host__ __device__ constexpr int up_target(int MODE) { return MODE == UPK_TRI ? OQR_EXP_UP_TRI_WARPS : OQR_EXP_UP_WARPS; }
__host__ __device__ constexpr int up_quota(int NT, int MODE) {
  return (up_part_units(NT) + up_target(MODE) - 1) / up_target(MODE) < 2
             ? 2
             : ((up_part_units(NT) + up_target(MODE) - 1) / up_target(MODE) > up_maxc(MODE)
                    ? up_maxc(MODE)
                    : (up_part_units(NT) + up_target(MODE) - 1) / up_target(MODE));
}
// consumer warps per part, at most: the split of build_upper_sched below, counted at compile time
// (runs of balanced length, a run cut short where it would reach a third pair)
__host__ __device__ constexpr int up_wcap(int NT, int MODE) {
  const int U = up_units(NT), parts = up_parts(NT), q = up_quota(NT, MODE);
  int best = 0;
  for (int part = 0; part < parts; ++part) {
    const int u0 = U * part / parts, u1 = U * (part + 1) / parts, nu = u1 - u0, w = (nu + q - 1) / q;
    int u = 0, p = 0, l = 0, nw = 0, cnt = 0, segs = 0, lastp = -1, quota = 0;
    for (p = 0, l = 0, u = 0; u < u1; ++u) {  // walk units in pair order: (p, l), l = 2p .. NT-1
      if (u >= u0) {
        if (nw == 0 || cnt == quota || (p != lastp && segs == 2)) {
          quota = nu / w + (nw < nu % w ? 1 : 0);
          quota = quota > q ? q : (quota < 1 ? 1 : quota);
          ++nw;
          cnt = segs = 0;
        }
        if (cnt == 0 || p != lastp) ++segs;
        ++cnt;
        lastp = p;
      }
      if (++l == NT) l = 2 * ++p;
    }
    best = nw > best ? nw : best;
  }
  return best;
}
// Warps of a CTA for nwc consumer warps.  UPK_TRI: the warps of sub-partition 0 (warp w runs on
// sub-partition w % 4) are the producers -- they form W = T Z and issue the TMA -- and the
// consumers run on sub-partitions 1-3 only: on sm_100a DFMA/DMUL and DMMA share a sub-partition's
// FP64 pipe, and producers sharing it with consumers were starved by their DMMAs (ncu "math pipe
// throttle" on the producer's DMUL, consumers waiting for W).  Other modes: warp 0 issues the TMA.
__host__ __device__ constexpr int up_total_warps(int nwc, int MODE) {
  return MODE == UPK_TRI ? nwc + (nwc + 2) / 3 : nwc + 1;
}

// Per CTA part, per consumer warp: pa, la, l1, pb, lb, len -- units t < l1 are (pair pa, column
// la + t), units l1 <= t < len are (pair pb, column lb + t - l1).
struct UpperSched {
  int nwc;  // consumer warps per CTA (the larger part; the other part's extra warps have len 0)
  unsigned char w[4][UP_MAXW][6];
};

// Units in pair order, split into `parts` contiguous halves; each half into w = ceil(units / q)
// runs of balanced length (floor or ceil of units / w), a run cut short where it would reach a
// third pair.
static bool build_upper_sched(int NT, int parts, int q, int wcap, UpperSched* S) {
  std::memset(S, 0, sizeof(*S));
  int up[256][2], U = 0;
  for (int p = 0; p < (NT + 1) / 2; ++p)
    for (int l = 2 * p; l < NT; ++l) {
      up[U][0] = p;
      up[U][1] = l;
      ++U;
    }
  for (int part = 0; part < parts; ++part) {
    const int u0 = U * part / parts, u1 = U * (part + 1) / parts, nu = u1 - u0;
    const int w = (nu + q - 1) / q;
    int nw = 0, cnt = 0, segs = 0, lastp = -1, quota = 0;
    unsigned char* cur = nullptr;
    for (int u = u0; u < u1; ++u) {
      const int p = up[u][0], l = up[u][1];
      if (cur == nullptr || cnt == quota || (p != lastp && segs == 2)) {
        if (nw == wcap || nw == UP_MAXW) return false;
        cur = S->w[part][nw];
        quota = nu / w + (nw < nu % w ? 1 : 0);
        if (quota > q) quota = q;
        if (quota < 1) quota = 1;
        ++nw;
        cnt = segs = 0;
      }
      if (cnt == 0 || p != lastp) {
        if (segs == 0) {
          cur[0] = (unsigned char)p; cur[1] = (unsigned char)l;
        }
        cur[3] = (unsigned char)p; cur[4] = (unsigned char)l;
        ++segs;
      }
      if (segs == 1) ++cur[2];
      ++cur[5];
      ++cnt;
      lastp = p;
    }
    if (nw > S->nwc) S->nwc = nw;
  }
  return true;
}

// registers per thread: warps are spread over the SM's four sub-partitions, each with a quarter
// of the register file (16384), so ceil(warps / 4) warps share one quarter
__host__ __device__ constexpr int up_maxreg(int NT, int MODE) {
  return (512 / ((up_total_warps(up_wcap(NT, MODE), MODE) + 3) / 4)) / 8 * 8 > 248
             ? 248
             : (512 / ((up_total_warps(up_wcap(NT, MODE), MODE) + 3) / 4)) / 8 * 8;
}

// One consumer warp's whole block loop, for a run of exactly LEN units (PRED: a run of `len` <= LEN
// units, the DMMAs of units t >= len predicated off -- only for runs cut short at a third pair).
// (Measured and not kept: the consumers forming W themselves, two blocks ahead, instead of two
// producer warps -- 0.30 vs 0.24 ms at m = 1e5, n = 200.)
struct UpShared {
  const double* ring;
  double* wbuf;
  const double* ds;
  const double* es;
  uint64_t* zfull;
  uint64_t* zempty;
  uint64_t* wfull;
  uint64_t* wempty;
  int stages, stage, nwb, nb, b0, nwc;
  int64_t m;
  bool same;
};


// W(b) = T Z for block i of the slice in B-fragment order, by producer warp pw of npw: k-steps
// kk = pw, pw + npw, .., its lane the row r = 4 kk + lane%4 of every n-tile (Zt[c * TRB + TRH + r] =
// Z[16 b + r, c], r = -2 .. 17); the three z of UPB n-tiles are loaded before any W is stored.
template <int NT>
__device__ __forceinline__ void up_form_w(const UpShared& S, int i, int pw, int npw, int lane) {
  constexpr int FB = NT * 4 * FRAG;
  const int s = i % S.stages, j = i % S.nwb;
  mbar_wait(&S.zfull[s], (i / S.stages) & 1);
  if (i >= S.nwb) mbar_wait(&S.wempty[j], ((i / S.nwb) - 1) & 1);
  const double* __restrict__ Zt = S.ring + s * S.stage;
  double* __restrict__ W = S.wbuf + j * FB;
  const int64_t r0 = (int64_t)(S.b0 + i) * BK;
#pragma unroll 1
  for (int kk = pw; kk < BK / 4; kk += npw) {
    const int r = kk * 4 + (lane & 3);
    const int il = i * BK + r;
    const bool in = r0 + r < S.m;
    const double em = S.es[il], dd = S.ds[il], ep = S.es[il + 1];
    const double* zc = Zt + (lane >> 2) * TRB + TRH + r;
    double* wp = W + kk * FRAG + lane;
    constexpr int UPB = 5;
#pragma unroll
    for (int l0 = 0; l0 < NT; l0 += UPB) {
      double zm[UPB], z0[UPB], zp[UPB];
#pragma unroll
      for (int k = 0; k < UPB; ++k)
        if (l0 + k < NT) {
          const double* z = zc + (l0 + k) * 8 * TRB;
          zm[k] = z[-1];
          z0[k] = z[0];
          zp[k] = z[1];
        }
#pragma unroll
      for (int k = 0; k < UPB; ++k)
        if (l0 + k < NT) {
          double wv = em * zm[k];     // e_{i-1} z_{i-1}
          wv = fma(dd, z0[k], wv);    // + d_i z_i
          wv = fma(ep, zp[k], wv);    // + e_i z_{i+1}
          wp[(l0 + k) * 4 * FRAG] = in ? wv : 0.0;
        }
    }
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&S.wfull[j]);
}

template <int NT, int MODE, int LEN, bool PRED>
__device__ __forceinline__ void up_consume(const UpShared& S, int cw, int lane, const unsigned char* tw,
                                        double* __restrict__ slot) {
  constexpr int NP = NT * 8;
  constexpr int FB = NT * 4 * FRAG;
  constexpr int LA = LEN > 0 ? LEN : 1;
  const int da = 2 * tw[0], la = tw[1], l1 = tw[2], db = 2 * tw[3], lb = tw[4], len = PRED ? tw[5] : LEN;
  const int da1 = da + 1 < NT ? da + 1 : NT - 1, db1 = db + 1 < NT ? db + 1 : NT - 1;
  // fragment offsets in the stage (k-step kk adds kk * AK / BKS):
  //   packed:  A tile row k: (k*4 + kk)*FRAG + lane          B tile column l: (l*4 + kk)*FRAG + lane
  //   Z box:   A tile row k: (k*8 + lane/4)*TRB + TRH + lane%4 + kk*4   (Z^T: lane row = Z column)
  //            B tile column l: the same with l (lane row lane%4 = Z row, col lane/4 = Z column)
  constexpr int AT = MODE == UPK_PACKED ? 4 * FRAG : 8 * TRB;  // per tile row of A
  constexpr int AK = MODE == UPK_PACKED ? FRAG : 4;             // per k-step of A
  constexpr int BT = MODE == UPK_EUCLID ? 8 * TRB : 4 * FRAG;   // per tile column of B
  constexpr int BKS = MODE == UPK_EUCLID ? 4 : FRAG;            // per k-step of B
  const int alane = MODE == UPK_PACKED ? lane : (lane >> 2) * TRB + TRH + (lane & 3);
  const int blane = MODE == UPK_EUCLID ? (lane >> 2) * TRB + TRH + (lane & 3) : lane;
  const int oa0 = da * AT + alane, oa1 = da1 * AT + alane, oc0 = db * AT + alane, oc1 = db1 * AT + alane;
  const int ob0 = la * BT + blane, ob1 = (lb - l1) * BT + blane;  // unit t: (t < l1 ? ob0 : ob1) + t*BT
  const int th0 = da - la, th1 = db - lb + l1;                   // second tile of unit t iff t > th
  double acc[LA][2][2];
#pragma unroll
  for (int t = 0; t < LA; ++t) acc[t][0][0] = acc[t][0][1] = acc[t][1][0] = acc[t][1][1] = 0.0;
  for (int i = 0; i < S.nb; ++i) {
    const int s = i % S.stages, j = MODE == UPK_TRI ? i % S.nwb : 0;
    mbar_wait(&S.zfull[s], (i / S.stages) & 1);
    if (MODE == UPK_TRI) mbar_wait(&S.wfull[j], (i / S.nwb) & 1);
    const double* As = S.ring + s * S.stage;
    const double* Bs = MODE == UPK_TRI ? S.wbuf + j * FB : (MODE == UPK_PACKED && !S.same ? As + FB : As);
#ifndef OQR_EXP_K4_NOCONSUME  // experiment build only: the consumers only hand the stages back
    if (LEN > 0) {
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        // every operand of the k-step first, then its DMMAs
        const double a0 = As[oa0 + kk * AK], a1 = As[oa1 + kk * AK];
        const double c0 = As[oc0 + kk * AK], c1 = As[oc1 + kk * AK];
        double bv[LA];
#pragma unroll
        for (int t = 0; t < LA; ++t)
          bv[t] = Bs[(!PRED || t < len ? (t < l1 ? ob0 : ob1) + t * BT : ob0) + kk * BKS];
#pragma unroll
        for (int t = 0; t < LA; ++t) {
          const bool s0 = t < l1;
          const bool on = !PRED || t < len;
          dmma_if(acc[t][0], s0 ? a0 : c0, bv[t], on);                          // tile (dr, l)
          dmma_if(acc[t][1], s0 ? a1 : c1, bv[t], on && t > (s0 ? th0 : th1));  // (dr + 1, l) iff l > dr
        }
      }
    }
#endif
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&S.zempty[s]);
      if (MODE == UPK_TRI) mbar_arrive(&S.wempty[j]);
    }
  }
  // C tile (k, l): rows k*8 + lane/4, cols l*8 + 2*(lane%4) + q
#pragma unroll
  for (int t = 0; t < LA; ++t) {
    if (t < len) {
      const bool s0 = t < l1;
      const int l = s0 ? la + t : lb + (t - l1);
      const int dr = s0 ? da : db;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && l <= dr) break;
#pragma unroll
        for (int q = 0; q < 2; ++q)
          slot[(int64_t)(l * 8 + 2 * (lane & 3) + q) * NP + (dr + h) * 8 + (lane >> 2)] = acc[t][h][q];
      }
    }
  }
}

template <int NT, int MODE>
__global__ void __maxnreg__(up_maxreg(NT, MODE))
gram_upper_kernel(const __grid_constant__ CUtensorMap zmap, const double* __restrict__ Xp,
                  const double* __restrict__ Yp, const double* __restrict__ d, const double* __restrict__ e,
                  int64_t m, int nblk, double* __restrict__ P, int stages, int nwb,
                  const __grid_constant__ UpperSched sched) {
  constexpr int NP = NT * 8;
  constexpr int C = up_quota(NT, MODE);
  constexpr int FB = NT * 4 * FRAG;  // doubles per packed block operand (and per W buffer)
  extern __shared__ __align__(1024) unsigned char smem[];
  UpShared S;
  S.same = MODE == UPK_PACKED && Xp == Yp;
  S.stage = MODE == UPK_PACKED ? (S.same ? FB : 2 * FB) : TRB * NP;
  S.zfull = reinterpret_cast<uint64_t*>(smem);
  S.zempty = S.zfull + 8;
  S.wfull = S.zempty + 8;
  S.wempty = S.wfull + 4;
  S.wbuf = reinterpret_cast<double*>(smem + 256);  // [nwb][FB] (UPK_TRI)
  double* ring = S.wbuf + (MODE == UPK_TRI ? nwb * FB : 0);
  S.ring = ring;
  S.stages = stages;
  S.nwb = nwb;
  S.m = m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  S.nwc = sched.nwc;
  const int slice = blockIdx.x, nslices = gridDim.x;
  const int b0 = (int)((int64_t)nblk * slice / nslices), b1 = (int)((int64_t)nblk * (slice + 1) / nslices);
  S.b0 = b0;
  S.nb = b1 - b0;
  const uint64_t pol = policy_evict_first();  // every operand is streamed once
  // UPK_TRI: the slice's diagonal and couplings, staged once: ds[i] = d_{16 b0 + i},
  // es[i] = e_{16 b0 + i - 1} (0 outside)
  double* ds = ring + stages * S.stage;
  double* es = ds + S.nb * BK;
  S.ds = ds;
  S.es = es;
  if (MODE == UPK_TRI) {
    const int64_t rs = (int64_t)b0 * BK;
    const int nr = S.nb * BK;
    for (int i = threadIdx.x; i <= nr; i += blockDim.x) {
      const int64_t row = rs + i;
      if (i < nr) ds[i] = row < m ? __ldg(d + row) : 0.0;
      es[i] = (row >= 1 && row - 1 < m - 1) ? __ldg(e + row - 1) : 0.0;
    }
  }
  auto issue = [&](int b, int s) {  // block b into ring stage s
    double* dst = ring + s * S.stage;
    if (MODE == UPK_PACKED) {
      const uint32_t fb = FB * 8;
      mbar_arrive_expect_tx(&S.zfull[s], S.same ? fb : 2 * fb);
      bulk_g2s(dst, Xp + (int64_t)b * FB, fb, &S.zfull[s], pol);
      if (!S.same) bulk_g2s(dst + FB, Yp + (int64_t)b * FB, fb, &S.zfull[s], pol);
    } else {
      mbar_arrive_expect_tx(&S.zfull[s], (uint32_t)(TRB * NP * 8));
      tma_g2s_2d(dst, &zmap, b * BK - TRH, 0, &S.zfull[s], pol);
    }
  };
  const int nwarps = blockDim.x >> 5;
  const int nprod = MODE == UPK_TRI ? (nwarps + 3) / 4 : 1;  // producer warps
  const int npw = nprod < BK / 4 ? nprod : BK / 4;           // ... that form W (one k-step or more each)
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&S.zfull[s], 1);
      mbar_init(&S.zempty[s], S.nwc);
    }
    for (int j = 0; j < nwb; ++j) {
      mbar_init(&S.wfull[j], npw);
      mbar_init(&S.wempty[j], S.nwc);
    }
    mbar_fence_init();
    for (int s = 0; s < stages && s < S.nb; ++s) issue(b0 + s, s);
  }
  __syncthreads();
  if (MODE == UPK_TRI ? (warp & 3) == 0 : warp == 0) {
    if constexpr (MODE != UPK_TRI) {  // producer: the ring refills (one elected lane)
      if (lane == 0)
        for (int i = stages; i < S.nb; ++i) {
          const int s = i % stages;
          mbar_wait(&S.zempty[s], ((i / stages) - 1) & 1);
          issue(b0 + i, s);
        }
    } else {  // the producers form W; warp 0's lane 0 also refills the ring one block behind
      const int pw = warp >> 2;
      if (pw >= npw) return;
      for (int i = 0; i < S.nb; ++i) {
        up_form_w<NT>(S, i, pw, npw, lane);
        if (warp == 0 && lane == 0 && i >= 1 && i - 1 + stages < S.nb) {
          const int ip = i - 1;
          mbar_wait(&S.zempty[ip % stages], (ip / stages) & 1);
          issue(b0 + ip + stages, ip % stages);
        }
      }
    }
    return;
  }
  const int cw = MODE == UPK_TRI ? warp - (warp >> 2) - 1 : warp - 1;
  const unsigned char* tw = sched.w[blockIdx.y][cw];
  double* slot = P + (int64_t)slice * NP * NP;
  const int len = tw[5];
  if (len == C)
    up_consume<NT, MODE, C, false>(S, cw, lane, tw, slot);
  else if (C > 1 && len == C - 1)
    up_consume<NT, MODE, (C > 1 ? C - 1 : 1), false>(S, cw, lane, tw, slot);
  else if (len == 0)
    up_consume<NT, MODE, 0, false>(S, cw, lane, tw, slot);
  else
    up_consume<NT, MODE, C, true>(S, cw, lane, tw, slot);
}

// The Z box map of K4e / K4t: the caller's column-major Z (m x n, ldz), box TRB rows x NP columns.
static bool make_tmap_z_box(CUtensorMap* map, const double* Z, int64_t m, int n, int64_t ldz, int NP) {
  if ((reinterpret_cast<uintptr_t>(Z) & 15) != 0 || (ldz & 1) != 0 || m > (int64_t)INT32_MAX) return false;
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)ldz * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)TRB, (cuuint32_t)NP};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(Z), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Launch the K4 family (MODE) for NT = ceil(n/8).  *done = false (nothing launched, no error) when
// the box modes cannot describe Z to TMA or the ring does not fit: the caller then packs.
template <int NT, int MODE>
static cudaError_t gram_upper_nt(int64_t m, int n, const double* Z, int64_t ldz, const double* Xp,
                                 const double* Yp, const double* d, const double* e, double* P, int* g_out,
                                 cudaStream_t s, bool* done) {
  *done = false;
  constexpr int NCP = up_parts(NT);
  UpperSched sched;
  if (!build_upper_sched(NT, NCP, up_quota(NT, MODE), up_wcap(NT, MODE), &sched)) return cudaErrorInvalidConfiguration;
  const int64_t nblk = zp_blocks(m);
  int64_t nsl = num_sms() / NCP;
  if (nsl > nblk) nsl = nblk;
  constexpr size_t fb = (size_t)NT * 4 * FRAG * 8;
  const size_t stage = MODE == UPK_PACKED ? (Xp == Yp ? fb : 2 * fb) : (size_t)TRB * NT * 8 * 8;
  const size_t de = MODE == UPK_TRI ? (size_t)(2 * (cdiv(nblk, nsl) * BK) + 1) * 8 : 0;
  int nwb = MODE == UPK_TRI ? 3 : 0;
  int stages = (int)((SMEM_MAX - 256 - nwb * fb - de) / stage);
  if (MODE == UPK_TRI && stages < 3) {
    nwb = 2;
    stages = (int)((SMEM_MAX - 256 - nwb * fb - de) / stage);
  }
  if (stages > 8) stages = 8;
#ifdef OQR_EXP_K4_STAGES  // experiment build only
  if (stages > OQR_EXP_K4_STAGES) stages = OQR_EXP_K4_STAGES;
#endif
  if (stages < 2) {
    if (MODE == UPK_PACKED) return cudaErrorInvalidConfiguration;
    return cudaSuccess;
  }
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  if (MODE != UPK_PACKED && !make_tmap_z_box(&tmap, Z, m, n, ldz, NT * 8)) return cudaSuccess;
  const size_t bytes = 256 + nwb * fb + de + stages * stage;
  cudaError_t err = ensure_smem_attr(reinterpret_cast<const void*>(gram_upper_kernel<NT, MODE>), (int)bytes);
  if (err != cudaSuccess) return err;
  *g_out = (int)nsl;
  timing_begin(s, OQR_TIMING_K4);
  gram_upper_kernel<NT, MODE><<<dim3((unsigned)nsl, NCP), 32 * up_total_warps(sched.nwc, MODE), bytes, s>>>(
      tmap, Xp, Yp, d, e, m, (int)nblk, P, stages, nwb, sched);
  note_launch();
  err = cudaGetLastError();
  timing_end(s);
  *done = true;
  return err;
}

#define OQR_NT_CASES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) \
  X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30)

cudaError_t launch_gram_fused(int64_t m, int64_t mr, int n, const double* A, int64_t lda, const double* Zp,
                              const double* Zc, const double* Zh, double* P, int* g_out, cudaStream_t s,
                              bool accum) {
  if (Zh != nullptr && mr != m) return cudaErrorInvalidValue;  // SYM is a whole-matrix schedule
  switch ((int)cdiv(n, 8)) {
#define OQR_CASE(NT)                                                                        \
  case NT:                                                                                  \
    return Zh ? gram_fused_nt<NT, true>(m, mr, A, lda, Zp, Zc, Zh, P, g_out, s, accum)       \
              : gram_fused_nt<NT, false>(m, mr, A, lda, Zp, Zc, nullptr, P, g_out, s, accum);
    OQR_NT_CASES(OQR_CASE)
#undef OQR_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gram_tridiag(int64_t m, int n, const double* d, const double* e, const double* Z, int64_t ldz,
                                double* P, int* g_out, cudaStream_t s, bool* done) {
  switch ((int)cdiv(n, 8)) {
#define OQR_CASE(NT) \
  case NT: return gram_upper_nt<NT, UPK_TRI>(m, n, Z, ldz, nullptr, nullptr, d, e, P, g_out, s, done);
    OQR_NT_CASES(OQR_CASE)
#undef OQR_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gram_euclid_box(int64_t m, int n, const double* Z, int64_t ldz, double* P, int* g_out,
                                   cudaStream_t s, bool* done) {
  switch ((int)cdiv(n, 8)) {
#define OQR_CASE(NT) \
  case NT: return gram_upper_nt<NT, UPK_EUCLID>(m, n, Z, ldz, nullptr, nullptr, nullptr, nullptr, P, g_out, s, done);
    OQR_NT_CASES(OQR_CASE)
#undef OQR_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gram_packed(int64_t m, int n, const double* Xp, const double* Yp, double* P, int* g_out,
                               cudaStream_t s) {
  bool done = false;
  switch ((int)cdiv(n, 8)) {
#define OQR_CASE(NT) \
  case NT: return gram_upper_nt<NT, UPK_PACKED>(m, n, nullptr, 0, Xp, Yp, nullptr, nullptr, P, g_out, s, &done);
    OQR_NT_CASES(OQR_CASE)
#undef OQR_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace oqr
