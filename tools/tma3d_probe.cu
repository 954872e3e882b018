// Probe (not product): can a tiled tensor map describe a column-major FP64 matrix as the 3-D
// view (r = row % 8, col, rg = row / 8) -- dim strides {8 B, lda*8 B, 64 B}, i.e. NOT in
// increasing order -- so that one TMA box (8, KS, 8) lands in shared memory as [rg][col][r]?
// And the 4-D view (row % 4, col, (row / 4) % 2, row / 8), box (4, KS, 2, 8) -> [row/4][col][row%4]
// (K1's ALAY_R4: each half warp's A-fragment load is 16 consecutive doubles).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tma3d tools/tma3d_probe.cu && /tmp/tma3d
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int KS = 32, RG = 8;

template <int RANK>
__global__ void probe(const __grid_constant__ CUtensorMap map, int col0, int rg0, double* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* buf = reinterpret_cast<double*>(smem + 1024);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar), d = (uint32_t)__cvta_generic_to_shared(buf);
  const uint32_t bytes = 8 * KS * RG * 8;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(bytes / 8); ++i) buf[i] = -777.0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    if (RANK == 3)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(d),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(col0), "r"(rg0), "r"(b)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
          "%5}], [%6];" ::"r"(d),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(col0), "r"(0), "r"(rg0), "r"(b)
          : "memory");
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(b)
          : "memory");
    }
    for (int i = 0; i < (int)(bytes / 8); ++i) out[i] = buf[i];
  }
}

int main() {
  const int64_t m = 1000, mr = 1000, lda = 1002;  // mr % 8 == 0
  std::vector<double> hA(lda * m);
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < lda; ++i) hA[j * lda + i] = (i < mr) ? (double)(j * 100000 + i) : -1.0;
  double *A, *out;
  cudaMalloc(&A, hA.size() * 8);
  cudaMalloc(&out, 8 * KS * RG * 8);
  cudaMemcpy(A, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn fn = reinterpret_cast<EncodeTiledFn>(p);
  int bad_total = 0;
  for (int rank = 3; rank <= 4; ++rank) {
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    CUresult r;
    if (rank == 3) {
      const cuuint64_t dims[3] = {8, (cuuint64_t)m, (cuuint64_t)(mr / 8)};
      const cuuint64_t strides[2] = {(cuuint64_t)lda * 8, 64};
      const cuuint32_t box[3] = {8, KS, RG};
      const cuuint32_t estr[3] = {1, 1, 1};
      r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      const cuuint64_t dims[4] = {4, (cuuint64_t)m, 2, (cuuint64_t)(mr / 8)};
      const cuuint64_t strides[3] = {(cuuint64_t)lda * 8, 32, 64};
      const cuuint32_t box[4] = {4, KS, 2, RG};
      const cuuint32_t estr[4] = {1, 1, 1, 1};
      r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, A, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    printf("encode %d-D (non-monotonic strides): %d\n", rank, (int)r);
    if (r != CUDA_SUCCESS) return 1;
    auto kern = rank == 3 ? probe<3> : probe<4>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 8 * KS * RG * 8);
    const int cases[3][2] = {{64, 16}, {(int)m - 5, 120}, {7, (int)(mr / 8) - 3}};
    for (auto& c : cases) {
      kern<<<1, 32, 1024 + 8 * KS * RG * 8>>>(map, c[0], c[1], out);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<double> h(8 * KS * RG);
      cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int g = 0; g < RG; ++g)
        for (int k = 0; k < KS; ++k)
          for (int i = 0; i < 8; ++i) {
            const int64_t col = c[0] + k, row = (int64_t)(c[1] + g) * 8 + i;
            const double want = (col < m && row < mr) ? hA[col * lda + row] : 0.0;
            const int at = rank == 3 ? (g * KS + k) * 8 + i : ((2 * g + i / 4) * KS + k) * 4 + i % 4;
            if (h[at] != want) ++bad;
          }
      printf("rank %d col0 %d rg0 %d: %s, %d mismatches of %d\n", rank, c[0], c[1], cudaGetErrorString(e), bad,
             8 * KS * RG);
      bad_total += bad;
    }
  }
  return bad_total != 0;
}
