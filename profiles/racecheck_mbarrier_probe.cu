// Does compute-sanitizer racecheck order shared-memory accesses through an
// mbarrier? Warp 1 reads a shared buffer and arrives on an mbarrier; warp 0
// waits on the barrier phase and then overwrites the buffer, either with
// plain stores (mode 0) or with a cp.async.bulk copy (mode 1). Mode 2 has no
// barrier at all (a true race, the positive control).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o rc profiles/racecheck_mbarrier_probe.cu
//   compute-sanitizer --tool racecheck ./rc <mode>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__global__ void probe(const double* src, double* out, int mode) {
  __shared__ __align__(128) double buf[256];
  __shared__ __align__(8) unsigned long long bar, full;
  const int tid = threadIdx.x, warp = tid >> 5;
  const unsigned eb = (unsigned)__cvta_generic_to_shared(&bar);
  const unsigned fb = (unsigned)__cvta_generic_to_shared(&full);
  const unsigned bb = (unsigned)__cvta_generic_to_shared(buf);
  for (int i = tid; i < 256; i += blockDim.x) buf[i] = i;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(eb));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) {
    double s = 0;
    for (int i = tid & 31; i < 256; i += 32) s += buf[i];
    out[tid] = s;
    __syncwarp();
    if ((tid & 31) == 0 && mode != 2) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(eb) : "memory");
  } else if (warp == 0 && tid == 0) {
    if (mode != 2) {
      unsigned done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(eb), "r"(0u)
                     : "memory");
    }
    if (mode == 1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(2048u) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(bb),
                   "l"(src), "r"(2048u), "r"(fb)
                   : "memory");
      unsigned done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(fb), "r"(0u)
                     : "memory");
    } else {
      for (int i = 0; i < 256; ++i) buf[i] = -i;
    }
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? std::atoi(argv[1]) : 0;
  double *src, *out;
  cudaMalloc(&src, 2048);
  cudaMalloc(&out, 64 * 8);
  cudaMemset(src, 0, 2048);
  probe<<<1, 64>>>(src, out, mode);
  const cudaError_t e = cudaDeviceSynchronize();
  std::printf("mode %d: %s\n", mode, cudaGetErrorString(e));
  return e != cudaSuccess;
}
