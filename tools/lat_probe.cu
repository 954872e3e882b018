// lat_probe.cu -- dependent-issue latencies on the FP64 pipe of one SM sub-partition (sm_100a),
// alone and while other warps of the SAME sub-partition stream independent DMMAs.  K2/K3 are
// bound by dependent FP64 chains (pivot chain, row substitution) that share the sub-partition's
// FP64 pipe with the DMMA trailing updates of other warps; this probe gives the
// per-step cost of such a chain in both situations.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
//   ./tools/lat_probe
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

constexpr int N = 2048;  // dependent steps timed

// MODE 0: DFMA chain; 1: DMUL -> DFMA alternating (the substitution step); 2: dependent DMMA
// (same accumulator); 3: DMMA whose result feeds the next DMMA's A operand; 4: SHFL chain;
// 5: DFMA chain with 2 independent DMMAs of the SAME warp between consecutive steps.
// Warp 0 runs the chain.  Warps w with (w % 4) == smsp_of_bg and w > 0 stream independent
// DMMAs (8 accumulators) until warp 0 raises `done`; `bg` = how many such warps are active.
template <int MODE>
__global__ void probe(int bg, int same_smsp, long long* cycles, double* sink, volatile int* done) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp == 0) {
    double x = 1.0 + lane * 1e-9, y = 1.0000001, z = 1e-9;
    double acc[2] = {x, x}, o1[2] = {0, 0}, o2[2] = {0, 0};
    // let the background warps get going
    for (volatile int spin = 0; spin < 2000; ++spin) {}
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
      if (MODE == 0) x = fma(x, y, z);
      if (MODE == 1) { x = x * y; asm volatile("" : "+d"(x)); x = fma(-x, z, y); }
      if (MODE == 2) dmma(acc, y, z);
      if (MODE == 3) { double o[2] = {0, 0}; dmma(o, x, z); x = o[0] + 1.0; }
      if (MODE == 4) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
      if (MODE == 5) { x = fma(x, y, z); dmma(o1, y, z); dmma(o2, y, z); }
      if (MODE == 6) { double o[2] = {0, 0}; dmma(o, x, z); x = o[0]; }
    }
    long long t1 = clock64();
    if (lane == 0) { cycles[0] = t1 - t0; stop = 1; }
    sink[threadIdx.x] = x + acc[0] + acc[1] + o1[0] + o2[0];
  } else {
    const bool on_smsp = same_smsp ? (warp % 4 == 0) : (warp % 4 != 0);
    // the first `bg` eligible warps are active
    int idx = same_smsp ? warp / 4 - 1 : (warp - 1 - warp / 4);
    if (on_smsp && idx < bg) {
      double a[8][2];
#pragma unroll
      for (int c = 0; c < 8; ++c) a[c][0] = a[c][1] = c;
      const double p = 1.0 + lane * 1e-9, q = 1.0 - lane * 1e-9;
      while (!stop) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) dmma(a[c], p, q);
      }
      double s = 0;
#pragma unroll
      for (int c = 0; c < 8; ++c) s += a[c][0] + a[c][1];
      sink[threadIdx.x] = s;
    }
  }
}

template <int MODE>
int run(const char* name, long long* cyc, double* sink, int* done) {
  for (int same = 1; same >= 0; --same)
    for (int bg : {0, 1, 2, 3}) {
      if (!same && bg == 0) continue;
      probe<MODE><<<1, 16 * 32>>>(bg, same, cyc, sink, done);
      CK(cudaDeviceSynchronize());
      long long c;
      CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
      const int per = (MODE == 1) ? 2 : 1;
      std::printf("%-44s bg DMMA warps on %s sub-partition = %d : %7.1f cycles per dependent op\n", name,
                  same ? "the SAME " : "ANOTHER  ", bg, (double)c / N / per);
    }
  return 0;
}

int main() {
  long long* cyc;
  double* sink;
  int* done;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaMalloc(&sink, 8 * 1024));
  CK(cudaMalloc(&done, 4));
  if (run<0>("DFMA chain", cyc, sink, done)) return 1;
  if (run<1>("DMUL -> DFMA chain (per op)", cyc, sink, done)) return 1;
  if (run<2>("DMMA, same accumulator", cyc, sink, done)) return 1;
  if (run<6>("DMMA -> A operand of the next DMMA", cyc, sink, done)) return 1;
  if (run<3>("DMMA -> DADD -> A operand (per pair)", cyc, sink, done)) return 1;
  if (run<4>("SHFL chain", cyc, sink, done)) return 1;
  if (run<5>("DFMA step + 2 own independent DMMAs", cyc, sink, done)) return 1;
  return 0;
}
