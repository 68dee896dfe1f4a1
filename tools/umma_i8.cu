// tcgen05 INT8 building block for the planned Ozaki pair kernel:
//   C[M=128][N] (s32, TMEM) = A[M][K] . B[N][K]^T (s8, shared memory, K-major, no swizzle)
// issued by one thread (tcgen05.mma.cta_group::1.kind::i8), completion through tcgen05.commit
// on an mbarrier, read back with tcgen05.ld. Checked bit-exactly against a host int64 product,
// then timed in a loop for the per-SM INT8 tensor rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8 tools/umma_i8.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 192;  // K in int8 elements (6 UMMA k-steps of 32)
constexpr int KSTEPS = K / 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// shared memory descriptor (cute::UMMA::SmemDescriptor): K-major, SWIZZLE_NONE, version 1
__device__ __forceinline__ uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((smem_u32(p) >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version (Blackwell)
  return d;                // base offset 0, lbo mode 0, layout type 0 (no swizzle)
}

// instruction descriptor (cute::UMMA::InstrDescriptor): S32 accumulator, s8 x s8, K-major both
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4)                  // c_format S32
         | (1u << 7) | (1u << 10)  // a_format, b_format: signed int8
         | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

// element (r, k) of an R x K operand in the canonical K-major no-swizzle layout:
// [kstep][r / 8][kchunk (16 B)][r % 8][16 B]; LBO = 128 B (next kchunk), SBO = 256 B (next 8 rows)
__host__ __device__ inline int op_index(int r, int k, int R) {
  const int ks = k / 32, kc = (k / 16) & 1, kb = k & 15;
  return ((ks * (R / 8) + r / 8) * 2 + kc) * 128 + (r % 8) * 16 + kb;
}

__global__ void umma_i8_kernel(const int8_t* A, const int8_t* B, int32_t* C, int reps) {
  __shared__ __align__(128) int8_t sA[M * K];
  __shared__ __align__(128) int8_t sB[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) sA[op_index(i / K, i % K, M)] = A[i];
  for (int i = tid; i < N * K; i += blockDim.x) sB[op_index(i / K, i % K, N)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> tensor core
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_i8(M, N);
    for (int r = 0; r < reps; ++r)
      for (int ks = 0; ks < KSTEPS; ++ks) {
        const uint64_t da = smem_desc(sA + ks * (M / 8) * 256, 128, 256);
        const uint64_t db = smem_desc(sB + ks * (N / 8) * 256, 128, 256);
        const uint32_t acc = (r > 0 || ks > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&mbar)));
  }
  // wait for the MMAs (phase 0 of the mbarrier)
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(&mbar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp w reads TMEM lanes 32w..32w+31 = rows of C; 16 columns per load
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t addr = tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = warp * 32 + lane;
    for (int j = 0; j < 16; ++j) C[size_t(blockIdx.x) * M * N + row * N + c0 + j] = int32_t(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(N));
}

int main() {
  std::vector<int8_t> A(M * K), B(N * K);
  srand(7);
  for (auto& x : A) x = int8_t(rand() % 255 - 127);
  for (auto& x : B) x = int8_t(rand() % 255 - 127);
  int8_t *dA, *dB;
  int32_t* dC;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dC, size_t(sms) * M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  umma_i8_kernel<<<1, 128>>>(dA, dB, dC, 1);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch: %s\n", cudaGetErrorString(e));
  std::vector<int32_t> C(M * N);
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += long(A[i * K + k]) * long(B[j * K + k]);
      if (s != C[i * N + j] && bad++ < 5) printf("mismatch C[%d][%d] = %d, expected %ld\n", i, j, C[i * N + j], s);
    }
  printf("exactness: %ld mismatches of %d\n", bad, M * N);
  // rate: every SM, reps x KSTEPS MMAs of 128 x 64 x 32
  const int reps = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  umma_i8_kernel<<<sms, 128>>>(dA, dB, dC, 100);
  cudaEventRecord(e0);
  umma_i8_kernel<<<sms, 128>>>(dA, dB, dC, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = double(sms) * reps * KSTEPS * 2.0 * M * N * 32;
  printf("tcgen05 kind::i8 M%d N%d: %.3f ms, %.0f TOPS (one CTA per SM, one MMA stream)\n", M, N, ms, ops / ms / 1e9);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
