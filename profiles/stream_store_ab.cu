// A/B of HBM write paths for the headline's traffic mix (3 int64 columns
// read, 6 fp64 columns written per point): plain 16-byte streaming stores
// (what kcg_multi_v6_tma does) against shared-memory staging + TMA bulk
// stores (cp.async.bulk.global.shared::cta). Standalone:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_store_ab profiles/stream_store_ab.cu
//   ./stream_store_ab [n_points]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

constexpr int R = 3, W = 6, TP = 1024;

__global__ void __launch_bounds__(256) plain(const long long* __restrict__ in, double* __restrict__ out,
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

// per tile of TP points: loads by the threads, outputs staged in shared
// memory (two buffers), one elected thread issues W bulk stores of TP * 8 B
template <int STAGES>
__global__ void __launch_bounds__(256) bulk(const long long* __restrict__ in, double* __restrict__ out,
                                            long long n) {
  extern __shared__ __align__(128) double sm[];
  const long long ntiles = n / TP;
  int k = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    double* buf = sm + (k % STAGES) * W * TP;
    if (threadIdx.x == 0)  // the buffer's previous bulk stores have read it
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
    __syncthreads();
#pragma unroll
    for (int u = 0; u < TP / 256; ++u) {
      const long long i = tile * TP + u * 256 + threadIdx.x;
      long long a = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) a += __ldcs(in + j * n + i);
#pragma unroll
      for (int j = 0; j < W; ++j) buf[j * TP + u * 256 + threadIdx.x] = (double)(a + j);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned sb = (unsigned)__cvta_generic_to_shared(buf);
      for (int j = 0; j < W; ++j)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + j * n + tile * TP),
                     "r"(sb + j * TP * 8), "r"(TP * 8)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      std::printf("%s: %s\n", #x, cudaGetErrorString(e));                  \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? std::atoll(argv[1]) : (1ll << 27);
  long long* in;
  double* out;
  CK(cudaMalloc(&in, 8 * R * n));
  CK(cudaMalloc(&out, 8 * W * n));
  CK(cudaMemset(in, 1, 8 * R * n));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = 8.0 * (R + W) * n;
  const float tp = timeit([&] { plain<<<sms * 8, 256>>>(in, out, n); });
  std::printf("{\"plain_stcs_GBps\": %.0f", bytes / tp / 1e6);
  for (int ctas : {1, 2, 3}) {
    const size_t smem2 = 2 * W * TP * 8, smem1 = 1 * W * TP * 8;
    CK(cudaFuncSetAttribute(bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    CK(cudaFuncSetAttribute(bulk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1));
    const float t2 = timeit([&] { bulk<2><<<sms * ctas, 256, smem2>>>(in, out, n); });
    const float t1 = timeit([&] { bulk<1><<<sms * ctas, 256, smem1>>>(in, out, n); });
    CK(cudaGetLastError());
    std::printf(", \"bulk_2buf_%dcta_GBps\": %.0f, \"bulk_1buf_%dcta_GBps\": %.0f", ctas, bytes / t2 / 1e6, ctas,
                bytes / t1 / 1e6);
  }
  std::printf("}\n");
  return 0;
}
