// Does FP64 SIMT work slow down while tcgen05.mma kind::i8 runs on the same SM? One CTA per SM:
// thread 0 issues the Ozaki V-GEMM's MMA mix (21 x M128 N80 K32 per k-step, commit per k-step)
// for KSTEPS k-steps (or nothing), while 8 other warps run a fixed loop of one instruction kind
// (8 independent chains). Prints the work warps' cycles with and without the MMA stream, and the MMA
// stream's cycles per MMA (does the work slow the MMAs down?). -DNN=128 for the N = 128 mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_vs_umma tools/fp64_vs_umma.cu
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#ifndef NN
#define NN 80
#endif
#ifndef WORK
#define WORK 4096
#endif
constexpr int S = 6, MM = 128, KSTEPS = 2048;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(const void* p) {
  return uint64_t((smem_u32(p) >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
         (uint64_t(1) << 46);
}
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(NN >> 3) << 17) | (uint32_t(MM >> 4) << 24);

template <int OP>
__device__ __forceinline__ void work(double* out, long long* cyc, const int8_t* sm) {
  const long long* sml = reinterpret_cast<const long long*>(sm);
  double a[8];
  float f[8];
  long long q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-3 + i, f[i] = float(a[i]), q[i] = threadIdx.x + i;
  const long long t0 = clock64();
  for (int it = 0; it < WORK; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fma(a[i], 0.999999, 1e-7);          // DFMA
      if (OP == 1) a[i] = a[i] * 0.9999999;                   // DMUL
      if (OP == 2) a[i] += double(q[i] + it);                  // I2F.F64.S64 + DADD
      if (OP == 3) f[i] = fmaf(f[i], 0.999999f, 1e-7f);       // FFMA
      if (OP == 4) q[i] = q[i] * 128 + it;                     // int64 IMAD
      if (OP == 5) q[i] += sml[(threadIdx.x + 32 * i + 8 * it) & 2047];  // LDS.64 (the operand region)
      if (OP == 6) {  // the contraction's mix: LDS.64 o, int64 -> FP64, DFMA, a double shuffle
        const long long o = sml[((threadIdx.x >> 3) * 4 + (threadIdx.x & 3) + 64 * i + 8 * it) & 2047];
        a[i] = fma(__longlong_as_double((o & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL), double(q[i] + it), a[i]);
        a[i] += __shfl_xor_sync(0xffffffffu, a[i], 1);
      }
      if (OP == 7) {  // FP32 mix: LDS.64, FFMA, a float shuffle
        const long long o = sml[((threadIdx.x >> 3) * 4 + (threadIdx.x & 3) + 64 * i + 8 * it) & 2047];
        f[i] = fmaf(__int_as_float(int(o) | 0x3F800000), float(it), f[i]);
        f[i] += __shfl_xor_sync(0xffffffffu, f[i], 1);
      }
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + f[i] + double(q[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

template <int OP>
__global__ void probe(int mma, double* out, long long* cyc, long long* mma_cyc) {
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tb;
  int8_t* sa = sm;
  int8_t* sb = sm + S * MM * 32;
  for (int i = threadIdx.x; i < S * (MM + NN) * 32; i += blockDim.x) sm[i] = int8_t(i * 7 + 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tb;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0 && mma) {
      const long long t0 = clock64();
      for (int ks = 0; ks < KSTEPS; ++ks) {
        if (ks >= 2) {
          const uint32_t b = smem_u32(&bar[ks & 1]), par = ((ks - 2) >> 1) & 1;
          asm volatile(
              "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(b),
              "r"(par)
              : "memory");
        }
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
          for (int t = 0; s + t < S; ++t)
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + uint32_t(((s + t) % (512 / NN)) * NN)),
                "l"(desc(sa + s * MM * 32)), "l"(desc(sb + t * NN * 32)), "r"(IDESC), "r"(ks > 0 ? 1u : 0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar[ks & 1])));
      }
      for (int ks = KSTEPS - 2; ks < KSTEPS; ++ks) {
        const uint32_t b = smem_u32(&bar[ks & 1]), par = (ks >> 1) & 1;
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(b),
            "r"(par)
            : "memory");
      }
      atomicMax((unsigned long long*)mma_cyc, (unsigned long long)(clock64() - t0));
    }
  } else {
    work<OP>(out, cyc, sm);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int OP>
void run(const char* name, int sms, double* out, long long* d) {
  const int smem = S * (MM + NN) * 32;
  cudaFuncSetAttribute(probe<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[2][2];
  for (int mma = 0; mma < 2; ++mma) {
    cudaMemset(d, 0, 16);
    probe<OP><<<sms, 288, smem>>>(mma, out, d, d + 1);
    cudaMemset(d, 0, 16);
    probe<OP><<<sms, 288, smem>>>(mma, out, d, d + 1);
    cudaMemcpy(h[mma], d, 16, cudaMemcpyDeviceToHost);
  }
  printf("N %d %-18s work warps: %8lld cycles alone, %8lld cycles beside the MMA stream (x%.2f); MMA stream %lld cycles "
         "(%.1f per MMA) -- %s\n",
         NN, name, h[0][0], h[1][0], double(h[1][0]) / h[0][0], h[1][1], double(h[1][1]) / (KSTEPS * 21.0),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* d;
  cudaMalloc(&out, sizeof(double) * sms * 288);
  cudaMalloc(&d, 16);
  run<0>("DFMA", sms, out, d);
  run<1>("DMUL", sms, out, d);
  run<2>("I2F.F64.S64+DADD", sms, out, d);
  run<3>("FFMA", sms, out, d);
  run<4>("IMAD int64", sms, out, d);
  run<5>("LDS.64", sms, out, d);
  run<6>("mix FP64", sms, out, d);
  run<7>("mix FP32", sms, out, d);
  return 0;
}
