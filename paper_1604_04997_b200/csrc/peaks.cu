// Pipe-throughput probes: the measured denominators of the instruction
// roofline that SURVEY §8(d) asks for (config 4 is bound by the instruction
// pipes; MEASURED_PEAKS.json holds only HBM and bf16 tensor figures).
//
// Every thread runs 8 independent dependency chains of one PTX instruction
// (inline asm volatile, so ptxas keeps exactly one SASS instruction per step):
//   kind 0  mad.lo.u32          -> IMAD  (integer multiply-add)
//   kind 1  lop3.b32            -> LOP3  (integer ALU pipe)
//   kind 2  fma.rn.f64          -> DFMA  (FP64 pipe)
//   kind 3  IMAD and LOP3 alternating: two pipes fed at once, i.e. the
//           warp-scheduler issue rate for the integer mix the eval / argmin
//           kernels execute
// at full occupancy (8 CTAs x 256 threads per SM). The result is lane
// operations per second; the loop's own 3 instructions per 128 steps are not
// counted, so the figure is a slight underestimate of the pipe peak.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "kcg_kernels.hpp"

namespace {

constexpr int kChains = 8;
constexpr int kUnroll = 16;

template <int KIND>
__global__ void __launch_bounds__(256) kcg_peak_probe(unsigned long long iters, unsigned seed,
                                                      unsigned long long* sink) {
  if constexpr (KIND == 2) {
    double a[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = 1.0 + 1e-9 * (threadIdx.x + c + seed);
    const double b = 0.999999, d = 1e-12;
    for (unsigned long long i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
#pragma unroll
        for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[c]) : "d"(b), "d"(d));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += a[c];
    if (s == 12345.0) sink[0] = 1;
  } else {
    unsigned a[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = threadIdx.x * 2654435761u + c + seed;
    const unsigned b = seed | 1u, d = 0x9e3779b9u;
    for (unsigned long long i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
          if (KIND == 0 || (KIND == 3 && (c & 1) == 0))
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(b), "r"(d));
          else
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(b), "r"(d));
        }
    }
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= a[c];
    if (s == 0x12345678u) sink[0] = s;
  }
}

// HBM stream with a given read/write mix: R int64 columns in, W fp64
// columns out (16-byte vector accesses, streaming cache hints) -- the
// "same-mix" bandwidth a kernel that reads R and writes W columns of n
// points can at best reach (e.g. R = 3, W = 6 for the one-pass six-variant
// evaluate + predict: one third reads)
template <int R, int W>
__global__ void __launch_bounds__(256) kcg_stream_probe(const long long* __restrict__ in, double* __restrict__ out,
                                                        long long n) {
  const long long nv = n >> 1;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv; v += (long long)gridDim.x * blockDim.x) {
    long long a = 0, b = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const longlong2 x = __ldcs(reinterpret_cast<const longlong2*>(in + j * n) + v);
      a += x.x;
      b += x.y;
    }
#pragma unroll
    for (int j = 0; j < W; ++j)
      __stcs(reinterpret_cast<double2*>(out + j * n) + v, make_double2((double)(a + j), (double)(b + j)));
  }
}

// the same mix with the outputs staged in shared memory and written by
// cp.async.bulk (TP-point tiles, one staging buffer): HBM takes a write-
// heavy mix faster from bulk stores than from 16-byte streaming stores
template <int R, int W>
__global__ void __launch_bounds__(256) kcg_stream_probe_bulk(const long long* __restrict__ in,
                                                             double* __restrict__ out, long long n) {
  constexpr int TP = 1024;
  extern __shared__ __align__(128) double sm[];
  const long long ntiles = n / TP;
  int k = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    if (k > 0 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int u = 0; u < TP / 256; ++u) {
      const long long i = tile * TP + u * 256 + threadIdx.x;
      long long a = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) a += __ldcs(in + j * n + i);
#pragma unroll
      for (int j = 0; j < W; ++j) sm[j * TP + u * 256 + threadIdx.x] = (double)(a + j);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned sb = (unsigned)__cvta_generic_to_shared(sm);
      for (int j = 0; j < W; ++j)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + j * n + tile * TP),
                     "r"(sb + j * TP * 8), "r"(TP * 8)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

namespace kcg {

double measure_pipe_peak(int kind, unsigned long long iters) {
  const unsigned grid = static_cast<unsigned>(num_sms()) * 8;
  unsigned long long* sink = nullptr;
  check(cudaMalloc(&sink, sizeof(unsigned long long)), "cudaMalloc");
  cudaEvent_t e0, e1;
  check(cudaEventCreate(&e0), "cudaEventCreate");
  check(cudaEventCreate(&e1), "cudaEventCreate");
  auto launch = [&](unsigned long long it) {
    switch (kind) {
      case 0: kcg_peak_probe<0><<<grid, 256>>>(it, 7u, sink); break;
      case 1: kcg_peak_probe<1><<<grid, 256>>>(it, 7u, sink); break;
      case 2: kcg_peak_probe<2><<<grid, 256>>>(it, 7u, sink); break;
      default: kcg_peak_probe<3><<<grid, 256>>>(it, 7u, sink); break;
    }
    check(cudaGetLastError(), "kcg_peak_probe launch");
  };
  launch(iters / 8 + 1);  // warm-up (clocks up, module loaded)
  std::vector<float> ms;
  for (int r = 0; r < 3; ++r) {
    check(cudaEventRecord(e0), "cudaEventRecord");
    launch(iters);
    check(cudaEventRecord(e1), "cudaEventRecord");
    check(cudaEventSynchronize(e1), "cudaEventSynchronize");
    float t = 0;
    check(cudaEventElapsedTime(&t, e0, e1), "cudaEventElapsedTime");
    ms.push_back(t);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  std::sort(ms.begin(), ms.end());
  const double ops = static_cast<double>(grid) * 256.0 * static_cast<double>(iters) * kUnroll * kChains;
  return ops / (ms[1] / 1e3);
}

double measure_stream(int R, int W, unsigned long long n) {
  n &= ~1ull;
  long long* in = nullptr;
  double* out = nullptr;
  check(cudaMalloc(&in, n * 8 * R), "cudaMalloc");
  check(cudaMalloc(&out, n * 8 * W), "cudaMalloc");
  check(cudaMemset(in, 1, n * 8 * R), "cudaMemset");
  const unsigned grid = static_cast<unsigned>(num_sms()) * 8;
  auto launch = [&] {
    const long long nn = static_cast<long long>(n);
    if (R == 3 && W == 6) kcg_stream_probe<3, 6><<<grid, 256>>>(in, out, nn);
    else if (R == 3 && W == 1) kcg_stream_probe<3, 1><<<grid, 256>>>(in, out, nn);
    else if (R == 1 && W == 6) kcg_stream_probe<1, 6><<<grid, 256>>>(in, out, nn);
    else if (R == 1 && W == 1) kcg_stream_probe<1, 1><<<grid, 256>>>(in, out, nn);
    else throw std::runtime_error("unsupported stream mix");
    check(cudaGetLastError(), "kcg_stream_probe launch");
  };
  cudaEvent_t e0, e1;
  check(cudaEventCreate(&e0), "cudaEventCreate");
  check(cudaEventCreate(&e1), "cudaEventCreate");
  auto best_ms = [&](auto&& run) {
    run();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      check(cudaEventRecord(e0), "cudaEventRecord");
      run();
      check(cudaEventRecord(e1), "cudaEventRecord");
      check(cudaEventSynchronize(e1), "cudaEventSynchronize");
      float t = 0;
      check(cudaEventElapsedTime(&t, e0, e1), "cudaEventElapsedTime");
      best = std::min(best, t);
    }
    return best;
  };
  float ms = best_ms(launch);
  // bulk-store variants (2 and 3 CTAs per SM): the best of all is the ceiling
  if (W > 0 && n % 1024 == 0) {
    const size_t smem = static_cast<size_t>(W) * 1024 * 8;
    auto bulk = [&](int ctas) {
      const long long nn = static_cast<long long>(n);
      const unsigned g = static_cast<unsigned>(num_sms()) * ctas;
      if (R == 3 && W == 6) kcg_stream_probe_bulk<3, 6><<<g, 256, smem>>>(in, out, nn);
      else if (R == 3 && W == 1) kcg_stream_probe_bulk<3, 1><<<g, 256, smem>>>(in, out, nn);
      else if (R == 1 && W == 6) kcg_stream_probe_bulk<1, 6><<<g, 256, smem>>>(in, out, nn);
      else kcg_stream_probe_bulk<1, 1><<<g, 256, smem>>>(in, out, nn);
      check(cudaGetLastError(), "kcg_stream_probe_bulk launch");
    };
    if (R == 3 && W == 6) check(cudaFuncSetAttribute(kcg_stream_probe_bulk<3, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    if (R == 1 && W == 6) check(cudaFuncSetAttribute(kcg_stream_probe_bulk<1, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    if ((R == 3 || R == 1) && (W == 6 || W == 1))
      for (int ctas : {2, 3}) ms = std::min(ms, best_ms([&] { bulk(ctas); }));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(in);
  cudaFree(out);
  return static_cast<double>(n) * 8.0 * (R + W) / (ms / 1e3);
}

}  // namespace kcg
