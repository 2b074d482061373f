// Do the FP64 tensor pipe (DMMA m8n8k4) and the FP64 vector pipe (DFMA)
// run concurrently on B200? Three launches at full occupancy:
//   dmma   every warp issues DMMA chains
//   dfma   every warp issues DFMA chains
//   mixed  each warp interleaves both (the same per-warp counts as above)
// If `mixed` takes about max(dmma, dfma) the pipes are independent and a
// Gram kernel can split its tiles between them; if it takes the sum they
// share the FP64 datapath.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_dfma_probe profiles/dmma_dfma_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kAcc = 4;  // independent DMMA accumulators per warp
constexpr int kDf = 8;   // independent DFMA chains per thread

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int NM, int NF>
__global__ void __launch_bounds__(256) probe(long long iters, double* sink) {
  double acc[kAcc][2];
  double f[kDf];
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 0.999999, c = 1e-12;
#pragma unroll
  for (int i = 0; i < kAcc; ++i) acc[i][0] = acc[i][1] = 0;
#pragma unroll
  for (int i = 0; i < kDf; ++i) f[i] = a + i;
  for (long long it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int m = 0; m < NM; ++m) dmma(acc[m % kAcc], a, b);
#pragma unroll
      for (int k = 0; k < NF; ++k) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[k % kDf]) : "d"(b), "d"(c));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kAcc; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < kDf; ++i) s += f[i];
  if (s == 1234.5) sink[0] = s;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, 8);
  const long long it = 20000;
  for (int ctas : {2, 4, 8}) {
    const int grid = sms * ctas;
    const double warps = grid * 8.0, lanes = grid * 256.0;
    // per iteration per warp: 4*NM DMMA (each 8*8*4*2 = 512 flops) and 4*NF DFMA per lane (2 flops)
    const float tm = timeit([&] { probe<8, 0><<<grid, 256>>>(it, sink); });
    const float tf = timeit([&] { probe<0, 16><<<grid, 256>>>(it, sink); });
    const float tx = timeit([&] { probe<8, 16><<<grid, 256>>>(it, sink); });
    const double fm = warps * it * 4 * 8 * 512.0, ff = lanes * it * 4 * 16 * 2.0;
    std::printf(
        "{\"ctas_per_sm\": %d, \"dmma_ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma_ms\": %.3f, \"dfma_tflops\": %.2f, "
        "\"mixed_ms\": %.3f, \"mixed_tflops\": %.2f, \"mixed_over_sum\": %.3f, \"mixed_over_max\": %.3f}\n",
        ctas, tm, fm / tm / 1e9, tf, ff / tf / 1e9, tx, (fm + ff) / tx / 1e9, tx / (tm + tf), tx / (tm > tf ? tm : tf));
  }
  return cudaGetLastError() != cudaSuccess;
}
