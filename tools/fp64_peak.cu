// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) and DFMA.
// Used to measure the roofline denominator for the FP64 GEMM stages (not in MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double a0, double b0) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0.0;
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double a0, double b0) {
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = threadIdx.x * 1e-3 + i;
  double a = a0, b = b0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clock(kHz) %d\n", prop.name, prop.multiProcessorCount, clk);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = prop.multiProcessorCount;
  for (int threads : {128, 256, 512}) {
    for (int ctas_per_sm : {1, 2, 4}) {
      const int iters = 20000;
      dmma_loop<8><<<sms * ctas_per_sm, threads>>>(out, 100, 1.0, 1.0);
      cudaEventRecord(e0);
      dmma_loop<8><<<sms * ctas_per_sm, threads>>>(out, iters, 1.0, 1.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double warps = double(sms) * ctas_per_sm * threads / 32;
      double flops = warps * iters * 8 * 8 * 8 * 4 * 2.0;
      printf("DMMA threads %d ctas/sm %d: %.3f ms  %.2f TFLOP/s\n", threads, ctas_per_sm, ms,
             flops / ms / 1e9);
    }
  }
  for (int threads : {256, 512, 1024}) {
    const int iters = 20000;
    dfma_loop<8><<<sms * 2, threads>>>(out, 100, 1.0000001, 1e-7);
    cudaEventRecord(e0);
    dfma_loop<8><<<sms * 2, threads>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = double(sms) * 2 * threads * iters * 8 * 2.0;
    printf("DFMA threads %d: %.3f ms  %.2f TFLOP/s\n", threads, ms, flops / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
