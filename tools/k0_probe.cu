// k0_probe.cu -- K0 peak microbenchmarks for the roofline denominators.
//
// MEASURED_PEAKS.json (driver-written) has HBM copy GB/s and bf16 GEMM TF/s but no FP64 entry,
// so the FP64 tensor (DMMA) and FP64 FMA (DFMA) peaks and a read-only HBM stream are measured
// here on the same B200 pool:
//   DMMA: mma.sync.m8n8k4.f64 with `chains` independent accumulators per warp, all SMs.
//   DFMA: fma.rn.f64 with independent chains.
//   HBM : read-only stream (double2 loads, sum kept live), 4 GiB buffer.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/k0_probe tools/k0_probe.cu
//   ./tools/k0_probe            (prints one line per measurement)
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_kernel(int iters, double* out) {
  double acc[CHAINS][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_kernel(int iters, double* out) {
  double acc[CHAINS];
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  std::printf("device %s sms %d clock %d kHz\n", prop.name, sms, clk);
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    dmma_kernel<8><<<sms, warps * 32>>>(iters, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_kernel<8><<<sms, warps * 32>>>(iters, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 512.0 * 8 * iters * warps * (double)sms;
    std::printf("DMMA m8n8k4 chains=8 warps/blk=%d : %.2f TFLOP/s (%.3f ms)\n", warps, fl / ms / 1e9, ms);
  }
  // sustained: back-to-back launches for >= 2 s (peaks at sustained clocks, >= 1 s)
  {
    const int nl = 80;  // ~26 ms each
    cudaEventRecord(e0);
    for (int r = 0; r < nl; ++r) dmma_kernel<8><<<sms, 16 * 32>>>(iters * 5, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("DMMA sustained (%d launches, %.2f s): %.2f TFLOP/s\n", nl, ms / 1e3,
                512.0 * 8 * iters * 5 * 16 * (double)sms * nl / ms / 1e9);
  }
  for (int warps : {8, 16, 32}) {
    dfma_kernel<8><<<sms, warps * 32>>>(iters, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_kernel<8><<<sms, warps * 32>>>(iters, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 8 * iters * warps * 32 * (double)sms;
    std::printf("DFMA chains=8 warps/blk=%d : %.2f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  const size_t bytes = (size_t)4 << 30;
  double2* buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 0, bytes));
  for (int bps : {2, 4, 8}) {
    read_kernel<<<sms * bps, 512>>>(buf, bytes / 16, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) read_kernel<<<sms * bps, 512>>>(buf, bytes / 16, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("HBM read blk/sm=%d: %.1f GB/s\n", bps, 5.0 * bytes / ms / 1e6);
  }
  cudaFree(buf);
  return 0;
}
