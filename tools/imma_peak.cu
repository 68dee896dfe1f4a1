// Legacy-tensor-path (mma.sync) INT8 and FP16 throughput on B200 (sm_100a), next to DMMA:
// is an Ozaki-style FP64 emulation on exact int8 x int8 -> int32 products
// reachable with mma.sync, or only with tcgen05? nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void imma(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void hmma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NACC>
__global__ void imma_loop(int* out, int iters) {
  int c[NACC][4] = {};
  uint32_t a = 0x01020304u + threadIdx.x, b = 0x05060708u ^ threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) imma(c[i], a, a + 1, a + 2, a + 3, b, b + 1);
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void hmma_loop(float* out, int iters) {
  float c[NACC][4] = {};
  uint32_t a = 0x3c003c00u, b = 0x3c003c00u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) hmma(c[i], a, a, a, a, b, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  printf("device %s SMs %d\n", prop.name, sms);
  int* iout;
  float* fout;
  cudaMalloc(&iout, 4096);
  cudaMalloc(&fout, 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    const int iters = 20000;
    imma_loop<8><<<sms, threads>>>(iout, 100);
    cudaEventRecord(e0);
    imma_loop<8><<<sms, threads>>>(iout, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = double(sms) * threads / 32 * iters * 8 * (16.0 * 8 * 32 * 2);
    printf("IMMA m16n8k32 s8 threads %d: %.3f ms  %.1f TOPS\n", threads, ms, ops / ms / 1e9);
    hmma_loop<8><<<sms, threads>>>(fout, 100);
    cudaEventRecord(e0);
    hmma_loop<8><<<sms, threads>>>(fout, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = double(sms) * threads / 32 * iters * 8 * (16.0 * 8 * 16 * 2);
    printf("HMMA m16n8k16 f16->f32 threads %d: %.3f ms  %.1f TFLOP/s\n", threads, ms, fl / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
