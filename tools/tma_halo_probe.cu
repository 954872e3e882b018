// Probe (not product): the 2-D tensor-TMA box K4t uses for the fused tridiagonal Gram -- {TRB rows,
// NPB cols} of a column-major FP64 matrix -- at start rows -2, -1, 0, 15, 16, 1998 (halo above the
// first row, odd / even starts, a box reaching past the last row, one wholly past it) and a box
// wider than n.  Result (B200): even starts incl. -2 and wholly-out-of-bounds boxes work, an odd start
// row (a box start that is not 16-byte aligned) is an illegal instruction.
// Prints, per case, whether the copy completed without a CUDA error and whether every element is
// Z[r0 + i, j] or 0 outside the matrix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tmah tools/tma_halo_probe.cu && /tmp/tmah
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void probe(const __grid_constant__ CUtensorMap map, int r0, int nelem, double* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* buf = reinterpret_cast<double*>(smem + 1024);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar), d = (uint32_t)__cvta_generic_to_shared(buf);
  const uint32_t bytes = nelem * 8;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nelem; ++i) buf[i] = -777.0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(d), "l"(reinterpret_cast<uint64_t>(&map)), "r"(r0), "r"(0), "r"(b)
        : "memory");
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(b)
          : "memory");
    }
    for (int i = 0; i < nelem; ++i) out[i] = buf[i];
  }
}

int main() {
  const int64_t m = 2000, n = 30, ldz = 2000;
  const int TRB = 20, NPB = 32;
  std::vector<double> hZ(ldz * n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) hZ[j * ldz + i] = 1000.0 * j + i + 1;
  double *dZ, *dout;
  cudaMalloc(&dZ, hZ.size() * 8);
  cudaMalloc(&dout, TRB * NPB * 8);
  cudaMemcpy(dZ, hZ.data(), hZ.size() * 8, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn fn = reinterpret_cast<EncodeTiledFn>(p);
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)ldz * 8};
  const cuuint32_t box[2] = {(cuuint32_t)TRB, (cuuint32_t)NPB};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dZ, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode box {%d, %d} over {%ld, %ld}: %d\n", TRB, NPB, (long)m, (long)n, (int)cr);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int r0 : {0, 16, -2, 1998, 2014, 2016, 15}) {
    probe<<<1, 32, 64 * 1024>>>(map, r0, TRB * NPB, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("r0 = %5d: CUDA error %s -- stopping (the context is gone)\n", r0, cudaGetErrorString(e));
      return 1;
    }
    std::vector<double> o(TRB * NPB);
    cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < NPB; ++j)
      for (int i = 0; i < TRB; ++i) {
        const int64_t r = r0 + i;
        const double want = (r >= 0 && r < m && j < n) ? hZ[j * ldz + r] : 0.0;
        if (o[j * TRB + i] != want) ++bad;
      }
    printf("r0 = %5d: ok, %d mismatches of %d\n", r0, bad, TRB * NPB);
  }
  return 0;
}
