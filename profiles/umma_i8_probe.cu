// tcgen05 kind::i8 probe (sm_100a): checks the K-major no-swizzle operand
// layout + instruction descriptor this repo's sliced Gram uses, against a
// host product, and measures the int8 MMA rate of that Gram's shape mix
// (per 32-row K step: two M = 128, N = 144 MMAs and one N = 80 MMA).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8_probe umma_i8_probe.cu && ./umma_i8_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

// K-major, no swizzle: core matrix = 8 rows x 16 bytes (128 contiguous bytes);
// within a KT-byte K extent, K-adjacent cores are 128 B apart (LBO) and
// 8-row groups are 8 * KT bytes apart (SBO).
__host__ __device__ inline int off_k(int x, int k, int KT) { return (x >> 3) * 8 * KT + (k >> 4) * 128 + (x & 7) * 16 + (k & 15); }

__device__ inline uint64_t sdesc(unsigned addr, unsigned lbo, unsigned sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)            // D = S32
         | (1u << 7)          // A = signed 8-bit
         | (1u << 10)         // B = signed 8-bit
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);  // K-major A and B (bits 15, 16 = 0)
}
__device__ inline void mma_i8(unsigned tmem_d, uint64_t a, uint64_t b, uint32_t idesc, unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ inline void commit(unsigned mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}
__device__ inline void mbar_wait(unsigned mbar, unsigned parity) {
  unsigned done = 0;
  const long long t0 = clock64();
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(mbar), "r"(parity) : "memory");
    if (!done && clock64() - t0 > 4000000000ll) {
      if ((threadIdx.x & 31) == 0) printf("mbarrier wait timed out (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}

// C[M=128][N] = sum_k A[m][k] B[n][k], K = KT (multiple of 32)
template <int N, int KT>
__global__ void k_check(const int8_t* A, const int8_t* B, int* C) {
  extern __shared__ __align__(1024) unsigned char sm[];
  int8_t* sa = (int8_t*)sm;
  int8_t* sb = sa + 128 * KT;
  __shared__ unsigned tbase;
  __shared__ __align__(8) unsigned long long bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * KT; i += blockDim.x) { int m = i / KT, k = i % KT; sa[off_k(m, k, KT)] = A[i]; }
  const int NP = (N + 7) / 8 * 8;
  for (int i = tid; i < NP * KT; i += blockDim.x) { int n = i / KT, k = i % KT; sb[off_k(n, k, KT)] = n < N ? B[n * KT + k] : 0; }
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&bar);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb)); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned td = tbase;
  if (tid == 0) {
    const unsigned a0 = (unsigned)__cvta_generic_to_shared(sa), b0 = (unsigned)__cvta_generic_to_shared(sb);
    for (int s = 0; s < KT / 32; ++s)
      mma_i8(td, sdesc(a0 + s * 256, 128, 8 * KT), sdesc(b0 + s * 256, 128, 8 * KT), idesc_i8(128, N), s > 0);
    commit(mb);
  }
  mbar_wait(mb, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warps 0..3: lanes 32 w .. 32 w + 31
  if (warp < 4) {
    const int m = 32 * warp + (tid & 31);
    for (int c = 0; c < N; c += 8) {
      unsigned r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(td + ((unsigned)(32 * warp) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int q = 0; q < 8; ++q) if (c + q < N) C[m * N + c + q] = (int)r[q];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(td));
}

// Rate: per iteration one 128-row K tile (4 K steps) x {N=144 at A0, N=144 at A0 (B + 144 rows), N=80 at A + 120 rows}
template <int KT>
__global__ void k_rate(int iters, int* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned tbase;
  __shared__ __align__(8) unsigned long long bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 288 * KT; i += blockDim.x) sm[i] = (unsigned char)(i * 7);
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&bar);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb)); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned td = tbase;
  if (tid == 0) {
    const unsigned p0 = (unsigned)__cvta_generic_to_shared(sm);
    const unsigned SB = 8 * KT;
    for (int it = 0; it < iters; ++it)
      for (int s = 0; s < KT / 32; ++s) {
        const unsigned ks = p0 + s * 256;
        mma_i8(td, sdesc(ks, 128, SB), sdesc(ks, 128, SB), idesc_i8(128, 144), it | s);
        mma_i8(td + 144, sdesc(ks, 128, SB), sdesc(ks + 18 * SB, 128, SB), idesc_i8(128, 144), it | s);
        mma_i8(td + 288, sdesc(ks + 15 * SB, 128, SB), sdesc(ks + 15 * SB, 128, SB), idesc_i8(128, 80), it | s);
      }
    commit(mb);
  }
  mbar_wait(mb, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    unsigned r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(td));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (tid == 0) sink[blockIdx.x] = (int)r;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(td));
}

template <int N, int KT>
bool check() {
  std::vector<int8_t> A(128 * KT), B(N * KT);
  uint32_t s = 12345u + N;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (int8_t)(s >> 24); };
  for (auto& v : A) v = rnd();
  for (auto& v : B) v = rnd();
  int8_t *dA, *dB; int* dC;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dC, 128 * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  const int smem = (128 + (N + 7) / 8 * 8) * KT;
  CK(cudaFuncSetAttribute(k_check<N, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_check<N, KT><<<1, 128, smem>>>(dA, dB, dC);
  CK(cudaDeviceSynchronize());
  std::vector<int> C(128 * N);
  CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      int ref = 0;
      for (int k = 0; k < KT; ++k) ref += (int)A[m * KT + k] * (int)B[n * KT + k];
      if (ref != C[m * N + n]) { if (bad < 4) printf("  mismatch m=%d n=%d got %d want %d\n", m, n, C[m * N + n], ref); ++bad; }
    }
  printf("check N=%d KT=%d: %s (%ld bad)\n", N, KT, bad ? "FAIL" : "ok", bad);
  CK(cudaFree(dA)); CK(cudaFree(dB)); CK(cudaFree(dC));
  return bad == 0;
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  printf("start\n");
  bool ok = check<16, 32>();
  ok = ok && check<144, 32>() && check<80, 128>() && check<144, 128>() && check<256, 64>();
  if (!ok) return 1;
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  int* sink; CK(cudaMalloc(&sink, nsm * 4));
  constexpr int KT = 128;
  const int smem = 288 * KT;
  CK(cudaFuncSetAttribute(k_rate<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 2000;
  k_rate<KT><<<nsm, 128, smem>>>(10, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  k_rate<KT><<<nsm, 128, smem>>>(iters, sink);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  const double macs = (double)nsm * iters * KT * 128.0 * (144 + 144 + 80);
  printf("rate: %d SMs x %d tiles of %d rows: %.3f ms, %.1f TOPS int8 (2 ops/MAC), %.2f ns per 1e8-row-equivalent row-tile pass -> %.3f ms per 1e8 rows\n",
         nsm, iters, KT, ms, 2 * macs / ms / 1e9, 0.0, ms * 1e8 / ((double)nsm * iters * KT));
  return ok ? 0 : 1;
}
