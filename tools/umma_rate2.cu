// (umma_rate2.cu: the same with CTA pairs, tcgen05.mma.cta_group::2, M = 256 over two SMs, each SM
// holding its 128 A rows and half of the N B rows.)
// tcgen05.mma kind::i8 issue-rate probe for the Ozaki V-GEMM's instruction mix: per "k-step" the
// 21 slice products (s + t <= 5) of six 128-row A slices and six N-row B slices (K = 32 each),
// accumulated into NACC TMEM accumulators (diagonal (s + t) % NACC), one commit per k-step, the
// issuing thread staying at most two k-steps ahead. Operands stay resident in shared memory, so
// this is the tensor core + operand path alone. Prints int8 TOPS over all SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DNN=64 -DNACC=6 -o tools/umma_rate tools/umma_rate.cu
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#ifndef NN
#define NN 64
#endif
#ifndef NACC
#define NACC 6
#endif
#define MM 256  // across the CTA pair
constexpr int S = 6, KSTEPS = 4096;
static_assert(NN * NACC <= 512, "TMEM columns");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(const void* p) {
  return uint64_t((smem_u32(p) >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
         (uint64_t(1) << 46);
}
constexpr int MH = 128, NH = NN / 2;  // per CTA
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(NN >> 3) << 17) | (uint32_t(MM >> 4) << 24);

__global__ void __cluster_dims__(2, 1, 1) rate_kernel(int* sink) {
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tb;
  int8_t* sa = sm;
  int8_t* sb = sm + S * MH * 32;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < S * (MH + NH) * 32; i += blockDim.x) sm[i] = int8_t(i * 7 + 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tb;
  if (threadIdx.x == 0 && rank == 0) {
    for (int ks = 0; ks < KSTEPS; ++ks) {
      if (ks >= 2) {  // the commit of k-step ks - 2
        const uint32_t b = smem_u32(&bar[ks & 1]), par = ((ks - 2) >> 1) & 1;
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(b),
            "r"(par)
            : "memory");
      }
#pragma unroll
      for (int s = 0; s < S; ++s)
#pragma unroll
        for (int t = 0; s + t < S; ++t) {
          const uint32_t d = tmem + uint32_t(((s + t) % NACC) * NN);
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(desc(sa + s * MH * 32)), "l"(desc(sb + t * NH * 32)), "r"(IDESC), "r"(ks > 0 ? 1u : 0u));
        }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(&bar[ks & 1])), "h"((unsigned short)3));
    }
    for (int ks = KSTEPS - 2; ks < KSTEPS; ++ks) {
      const uint32_t b = smem_u32(&bar[ks & 1]), par = (ks >> 1) & 1;
      asm volatile(
          "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(b),
          "r"(par)
          : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (v == 0x12345678u) sink[0] = 1;
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* sink;
  cudaMalloc(&sink, 4);
  const int smem = S * (MH + NH) * 32;
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rate_kernel<<<sms / 2 * 2, 128, smem>>>(sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    rate_kernel<<<sms / 2 * 2, 128, smem>>>(sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  const double ops = double(sms / 2) * KSTEPS * 21 * 2.0 * MM * NN * 32;  // one MMA stream per CTA pair
  printf("M %d N %d NACC %d: %s, %.3f ms, %.0f TOPS\n", MM, NN, NACC, cudaGetErrorString(cudaGetLastError()), best,
         ops / best / 1e9);
  return 0;
}
