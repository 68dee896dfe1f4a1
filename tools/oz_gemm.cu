// Throughput probe of the planned INT8 (Ozaki) V-GEMM of the pair stage:
// persistent CTAs over the cfg4 walker-tile triangle (16 Q walkers = 128 A rows x 8 P walkers =
// 64 B rows per tile, K' = 576), a producer thread streaming each k-step's six A and six B
// slices (36 KB) by cp.async.bulk into an mbarrier ring, one thread issuing the 21 slice-pair
// tcgen05.mma.kind::i8 products into six int32 TMEM accumulators (one per slice diagonal), and
// four epilogue warps recombining them in FP64 (optionally writing V). Checked against a host
// int64 product on sampled tiles, then timed with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/oz_gemm tools/oz_gemm.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int S = 6;                  // slices per operand
constexpr int KS = 18;                // k-steps of 32 (K' = 576)
constexpr int MA = 128, NB = 64;      // A rows (Q side), B rows (P side) per tile
constexpr int A_KS = S * MA * 32;     // bytes of one k-step of A (all slices)
constexpr int B_KS = S * NB * 32;
constexpr int STAGE = A_KS + B_KS;    // 36 KB
#ifndef STAGES
#define STAGES 5
#endif
constexpr int THREADS = 6 * 32;       // warps 0-3 epilogue, 4 producer, 5 MMA

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint64_t smem_desc(const void* p) {  // K-major, no swizzle, LBO 128, SBO 256
  return uint64_t((smem_u32(p) >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
         (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__host__ __device__ inline int op_off(int r, int kk) { return ((r / 8) * 2 + (kk / 16)) * 128 + (r % 8) * 16 + (kk & 15); }

// tile t of the triangle: Q block a (16 walkers), P block b < 2 (a + 1); t = a (a + 1) + b
__device__ __forceinline__ void oz_tile(int t, int& a, int& b) {
  int r = int((sqrt(4.0 * double(t) + 1.0) - 1.0) * 0.5);
  while ((r + 1) * (r + 2) <= t) ++r;
  while (r * (r + 1) > t) --r;
  a = r;
  b = t - r * (r + 1);
}

template <int N>
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}

__global__ void __launch_bounds__(THREADS, 1)
    oz_kernel(const int8_t* __restrict__ SA, const int8_t* __restrict__ SB, const int* __restrict__ ea,
              const double* __restrict__ sbv, int ntiles, double* __restrict__ V, double* __restrict__ sink) {
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull, tempty;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const int my = int(blockIdx.x) < ntiles ? (ntiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;

  if (warp == 4) {
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int it = 0; it < my; ++it) {
        int a, b;
        oz_tile(int(blockIdx.x) + it * int(gridDim.x), a, b);
        for (int ks = 0; ks < KS; ++ks) {
          mbar_wait(&empty[stage], ph ^ 1u);
          int8_t* dst = sm + stage * STAGE;
#ifdef NO_LOAD  // probe: MMA and epilogue alone on stale shared memory
          (void)dst;
          mbar_arrive(&full[stage]);
#else
          mbar_expect_tx(&full[stage], STAGE);
          bulk_g2s(dst, SA + (size_t(a) * KS + ks) * A_KS, A_KS, &full[stage]);
          bulk_g2s(dst + A_KS, SB + (size_t(b) * KS + ks) * B_KS, B_KS, &full[stage]);
#endif
          if (++stage == STAGES) stage = 0, ph ^= 1u;
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(MA, NB);
      int stage = 0;
      uint32_t ph = 0;
      for (int it = 0; it < my; ++it) {
        mbar_wait(&tempty, (it & 1) ^ 1u);  // the epilogue has drained the accumulators
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int ks = 0; ks < KS; ++ks) {
          mbar_wait(&full[stage], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const int8_t* sa = sm + stage * STAGE;
          const int8_t* sb = sa + A_KS;
#ifndef NO_MMA  // probe: the operand stream alone
#ifdef A_TMEM  // A slices copied once per k-step into TMEM (tcgen05.cp), MMAs read A from TMEM
          const uint32_t abuf = tmem + 384u + uint32_t((ks & 1) * 48);
#pragma unroll
          for (int s = 0; s < S; ++s)
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(abuf + 8u * s),
                         "l"(smem_desc(sa + s * MA * 32)));
#pragma unroll
          for (int s = 0; s < S; ++s)
#pragma unroll
            for (int t = 0; s + t < S; ++t) {
              const uint32_t d = tmem + uint32_t((s + t) * NB);
              const uint32_t acc = ks > 0 || s > 0 ? 1u : 0u;
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                  "r"(abuf + 8u * s), "l"(smem_desc(sb + t * NB * 32)), "r"(idesc), "r"(acc));
            }
#else
#pragma unroll
          for (int s = 0; s < S; ++s)
#pragma unroll
            for (int t = 0; s + t < S; ++t) {
              const uint32_t d = tmem + uint32_t((s + t) * NB);
              const uint32_t acc = ks > 0 || s > 0 ? 1u : 0u;
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                  "l"(smem_desc(sa + s * MA * 32)), "l"(smem_desc(sb + t * NB * 32)), "r"(idesc), "r"(acc));
            }
#endif
#else
          (void)sb;
#endif
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(&empty[stage])));
          if (++stage == STAGES) stage = 0, ph ^= 1u;
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&tfull)));
      }
    }
  } else {
    const int row = warp * 32 + lane;
    double chk = 0.0;
    for (int it = 0; it < my; ++it) {
      const int t = int(blockIdx.x) + it * int(gridDim.x);
      int a, b;
      oz_tile(t, a, b);
      mbar_wait(&tfull, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      // drain the six diagonals into one exact int64 per column (|X| < 2^59), release TMEM, then
      // convert once per column: V = X 2^(ea + eb - 14 - 35)
      long long X[NB];
#pragma unroll
      for (int c0 = 0; c0 < NB; c0 += 16) {
        uint32_t v[S][16];
#ifndef NO_EPI
#pragma unroll
        for (int d = 0; d < S; ++d) tmem_ld16<16>(tmem + (uint32_t(warp * 32) << 16) + uint32_t(d * NB + c0), v[d]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#else
#pragma unroll
        for (int d = 0; d < S; ++d)
#pragma unroll
          for (int c = 0; c < 16; ++c) v[d][c] = d + c + it;
#endif
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          long long x = int32_t(v[0][c]);
#pragma unroll
          for (int d = 1; d < S; ++d) x = x * 128 + int32_t(v[d][c]);
          X[c0 + c] = x;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&tempty);
      const double sr = ldexp(1.0, ea[a * MA + row] - 49);
      if (V) {
        double2* dst = reinterpret_cast<double2*>(V + (size_t(t) * MA + row) * NB);
#pragma unroll
        for (int c = 0; c < NB / 2; ++c)
          dst[c] = make_double2(double(X[2 * c]) * sr * sbv[b * NB + 2 * c], double(X[2 * c + 1]) * sr * sbv[b * NB + 2 * c + 1]);
      } else {
#pragma unroll
        for (int c = 0; c < NB; ++c) chk += double(X[c]) * sr * sbv[b * NB + c];
      }

    }
    if (!V && chk == 12345.678) sink[0] = chk;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 2048;
  const int nqb = m / 16, npb = m / 8, ntiles = nqb * (nqb + 1);
  const size_t sa_bytes = size_t(nqb) * KS * A_KS, sb_bytes = size_t(npb) * KS * B_KS;
  std::vector<int8_t> hA(sa_bytes), hB(sb_bytes);
  srand(7);
  for (auto& x : hA) x = int8_t(rand() % 255 - 127);
  for (auto& x : hB) x = int8_t(rand() % 255 - 127);
  std::vector<int> hea(nqb * MA), heb(npb * NB);
  for (auto& e : hea) e = rand() % 5 - 2;
  for (auto& e : heb) e = rand() % 5 - 2;
  int8_t *dA, *dB;
  int *dea, *deb;
  double *dV, *dsink;
  cudaMalloc(&dA, sa_bytes);
  cudaMalloc(&dB, sb_bytes);
  cudaMalloc(&dea, hea.size() * 4);
  cudaMalloc(&deb, heb.size() * 4);
  cudaMalloc(&dsink, 8);
  const size_t v_bytes = size_t(ntiles) * MA * NB * 8;
  if (cudaMalloc(&dV, v_bytes) != cudaSuccess) return printf("V alloc failed\n"), 1;
  cudaMemcpy(dA, hA.data(), sa_bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), sb_bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(dea, hea.data(), hea.size() * 4, cudaMemcpyHostToDevice);
  std::vector<double> hsb(heb.size());
  for (size_t i = 0; i < heb.size(); ++i) hsb[i] = ldexp(1.0, heb[i]);
  double* dsb;
  cudaMalloc(&dsb, hsb.size() * 8);
  cudaMemcpy(dsb, hsb.data(), hsb.size() * 8, cudaMemcpyHostToDevice);
  const int smem = STAGES * STAGE;
  cudaFuncSetAttribute(oz_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  oz_kernel<<<sms, THREADS, smem>>>(dA, dB, dea, dsb, ntiles, dV, dsink);
  cudaError_t e = cudaDeviceSynchronize();
  printf("m %d tiles %d slices %.1f MB: run %s\n", m, ntiles, (sa_bytes + sb_bytes) / 1e6, cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  // exactness on sampled tiles
  std::vector<double> hV(size_t(MA) * NB);
  long bad = 0;
  for (int t : {0, 1, 7, ntiles / 3, ntiles - 1}) {
    int a = 0;
    while ((a + 1) * (a + 2) <= t) ++a;
    const int b = t - a * (a + 1);
    cudaMemcpy(hV.data(), dV + size_t(t) * MA * NB, hV.size() * 8, cudaMemcpyDeviceToHost);
    for (int r = 0; r < MA; ++r)
      for (int c = 0; c < NB; ++c) {
        long long acc[S] = {};
        for (int s = 0; s < S; ++s)
          for (int u = 0; s + u < S; ++u)
            for (int k = 0; k < KS * 32; ++k)
              acc[s + u] += (long long)(hA[((size_t(a) * KS + k / 32) * S + s) * MA * 32 + op_off(r, k % 32)]) *
                            hB[((size_t(b) * KS + k / 32) * S + u) * NB * 32 + op_off(c, k % 32)];
        double x = 0.0;
        for (int d = S - 1; d >= 0; --d) x = x * 0x1p-7 + double(acc[d]);
        x = ldexp(x, hea[a * MA + r] + heb[b * NB + c] - 14);
        if (std::fabs(x - hV[r * NB + c]) > 1e-15 * std::fabs(x) && bad++ < 5)
          printf("tile %d (%d,%d): %.17g vs %.17g\n", t, r, c, hV[r * NB + c], x);
      }
  }
  printf("exactness: %ld mismatches\n", bad);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double ops = double(ntiles) * 21 * 2.0 * MA * NB * KS * 32;
  for (int wv = 0; wv < 2; ++wv) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      oz_kernel<<<sms, THREADS, smem>>>(dA, dB, dea, dsb, ntiles, wv ? dV : nullptr, dsink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("%s V: %.3f ms, %.0f TOPS int8, %.1f GB/s L2->smem, V write %.2f GB\n", wv ? "writing" : "no", best,
           ops / best / 1e9, double(ntiles) * KS * STAGE / best / 1e6, wv ? v_bytes / 1e9 : 0.0);
  }
  return 0;
}
