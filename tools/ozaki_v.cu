// Checkpoint of the planned INT8 pair kernel: the V block of one tile,
//   V[q][p] = sum_j A[q][j] conj(B[p][j])   (complex; A: 128 rows, B: 16 rows, K = KV spinors)
// as six-slice Ozaki sums of exact tcgen05 kind::i8 products, against a host long-double product.
// Operands: A' = [Re A | Im A], B're = [Re B | Im B], B'im = [-Im B | Re B] over K' = 2 KV
// (V_re = A' B're^T, V_im = A' B'im^T), every row scaled by its power-of-two maximum and cut into
// 6 slices of 7 bits; slice products with s + t = d accumulate in TMEM accumulator d (int32,
// exact: |acc| < 6 K' 127^2 < 2^31). Row magnitudes span e^0..e^-20 like the sqrt(exp(-eps tau))
// weights of Phi_v.    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ozaki_v tools/ozaki_v.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int KV = 280;                     // virtual spinors (cfg4: 278 -> 70 groups of 4)
constexpr int KP = 576;                     // K' = 2 KV padded to a multiple of 32
constexpr int KS = KP / 32;                 // UMMA k-steps
constexpr int S = 6;                        // slices
constexpr int MA = 128, NB = 32;            // A rows, B' rows (16 B rows x {re', im'})

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t smem_desc(const void* p) {  // K-major, no swizzle, LBO 128, SBO 256
  return uint64_t((smem_u32(p) >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
         (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
// (row r, k) of an R-row operand k-step in the canonical K-major no-swizzle layout
__host__ __device__ inline int op_off(int r, int kk) {  // kk in [0, 32)
  return ((r / 8) * 2 + (kk / 16)) * 128 + (r % 8) * 16 + (kk & 15);
}

// slice one row of K' doubles: exponent e (row max <= 2^e), slices[s][k] int8
__device__ void slice_row(const double* x, int n, int8_t* out /*[S][KS][R-layout]*/, int row, int R, int* e_out) {
  // one warp per row
  const int lane = threadIdx.x & 31;
  double mx = 0;
  for (int k = lane; k < n; k += 32) mx = fmax(mx, fabs(x[k]));
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0) e = ilogb(mx) + 1;  // mx < 2^e
  if (lane == 0) *e_out = e;
  for (int k = lane; k < KP; k += 32) {
    double r = k < n ? ldexp(x[k], -e) : 0.0;
    for (int s = 0; s < S; ++s) {
      r *= 128.0;
      const double q = trunc(r);
      r -= q;
      out[size_t(s) * KS * R * 32 + (k / 32) * R * 32 + op_off(row, k % 32)] = int8_t(q);
    }
  }
}

__global__ void slice_kernel(const double* Are, const double* Aim, const double* Bre, const double* Bim, int8_t* sa,
                             int8_t* sb, int* ea, int* eb) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  __shared__ double buf[8][KP];
  double* x = buf[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  if (w < MA) {
    for (int k = lane; k < KV; k += 32) x[k] = Are[w * KV + k], x[KV + k] = Aim[w * KV + k];
    __syncwarp();
    slice_row(x, 2 * KV, sa, w, MA, &ea[w]);
  } else if (w < MA + NB) {
    const int r = w - MA, b = r >> 1, part = r & 1;  // B' row: b re' (part 0) or im' (part 1)
    for (int k = lane; k < KV; k += 32) {
      x[k] = part ? -Bim[b * KV + k] : Bre[b * KV + k];
      x[KV + k] = part ? Bre[b * KV + k] : Bim[b * KV + k];
    }
    __syncwarp();
    slice_row(x, 2 * KV, sb, r, NB, &eb[r]);
  }
}

__global__ void vblock_kernel(const int8_t* sa, const int8_t* sb, const int* ea, const int* eb, double* V) {
  extern __shared__ __align__(128) int8_t sm[];
  int8_t* const smA = sm;                       // [S][MA x 32] for one k-step
  int8_t* const smB = sm + S * MA * 32;         // [S][NB x 32]
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  constexpr uint32_t idesc = idesc_i8(MA, NB);
  for (int ks = 0; ks < KS; ++ks) {
    // stage the k-step (plain copies in this checkpoint; TMA in the kernel)
    for (int s = 0; s < S; ++s) {
      const int4* ga = reinterpret_cast<const int4*>(sa + (size_t(s) * KS + ks) * MA * 32);
      const int4* gb = reinterpret_cast<const int4*>(sb + (size_t(s) * KS + ks) * NB * 32);
      for (int i = tid; i < MA * 2; i += blockDim.x) reinterpret_cast<int4*>(smA + s * MA * 32)[i] = ga[i];
      for (int i = tid; i < NB * 2; i += blockDim.x) reinterpret_cast<int4*>(smB + s * NB * 32)[i] = gb[i];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int s = 0; s < S; ++s)
        for (int t = 0; s + t < S; ++t) {
          const uint32_t d = tmem + uint32_t((s + t) * NB);  // accumulator of diagonal s + t
          // the first write of diagonal s + t in k-step 0 is the (s = 0, t = s + t) product
          const uint32_t accum = ks > 0 || s > 0 ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(smem_desc(smA + s * MA * 32)), "l"(smem_desc(smB + t * NB * 32)), "r"(idesc), "r"(accum));
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar)));
    }
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(&mbar)),
        "r"(ks & 1)
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  // epilogue: row = 32 warp + lane; V'[row][col] = sum_d acc_d 2^(-7 (d + 2)) 2^(ea + eb)
  const int row = warp * 32 + lane;
  double out[NB];
  for (int c = 0; c < NB; ++c) out[c] = 0.0;
  for (int d = 0; d < S; ++d) {
    uint32_t v[NB];
    const uint32_t addr = tmem + (uint32_t(warp * 32) << 16) + uint32_t(d * NB);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const double sc = ldexp(1.0, -7 * (d + 2));
    for (int c = 0; c < NB; ++c) out[c] += double(int32_t(v[c])) * sc;
  }
  for (int c = 0; c < NB; ++c) V[row * NB + c] = ldexp(out[c], ea[row] + eb[c]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  std::vector<double> Are(MA * KV), Aim(MA * KV), Bre(16 * KV), Bim(16 * KV);
  srand(11);
  auto u = [] { return double(rand()) / RAND_MAX - 0.5; };
  std::vector<double> wk(KV);
  for (int k = 0; k < KV; ++k) wk[k] = std::exp(-20.0 * k / KV);  // spinor weights e^0 .. e^-20
  for (int i = 0; i < MA; ++i)
    for (int k = 0; k < KV; ++k) Are[i * KV + k] = u() * wk[k] * (1 + i % 7), Aim[i * KV + k] = u() * wk[k];
  for (int i = 0; i < 16; ++i)
    for (int k = 0; k < KV; ++k) Bre[i * KV + k] = u() * wk[k], Bim[i * KV + k] = u() * wk[k] * 3;
  double *dAre, *dAim, *dBre, *dBim, *dV;
  int8_t *dsa, *dsb;
  int *dea, *deb;
  cudaMalloc(&dAre, Are.size() * 8);
  cudaMalloc(&dAim, Aim.size() * 8);
  cudaMalloc(&dBre, Bre.size() * 8);
  cudaMalloc(&dBim, Bim.size() * 8);
  cudaMalloc(&dsa, size_t(S) * KS * MA * 32);
  cudaMalloc(&dsb, size_t(S) * KS * NB * 32);
  cudaMalloc(&dea, MA * 4);
  cudaMalloc(&deb, NB * 4);
  cudaMalloc(&dV, MA * NB * 8);
  cudaMemcpy(dAre, Are.data(), Are.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dAim, Aim.data(), Aim.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dBre, Bre.data(), Bre.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dBim, Bim.data(), Bim.size() * 8, cudaMemcpyHostToDevice);
  slice_kernel<<<(MA + NB) / 8, 256>>>(dAre, dAim, dBre, dBim, dsa, dsb, dea, deb);
  const int smem = S * (MA + NB) * 32;
  cudaFuncSetAttribute(vblock_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  vblock_kernel<<<1, 128, smem>>>(dsa, dsb, dea, deb, dV);
  cudaError_t e = cudaDeviceSynchronize();
  printf("run: %s\n", cudaGetErrorString(e));
  std::vector<double> V(MA * NB);
  cudaMemcpy(V.data(), dV, V.size() * 8, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxv = 0;
  for (int i = 0; i < MA; ++i)
    for (int b = 0; b < 16; ++b) {
      long double re = 0, im = 0;
      for (int k = 0; k < KV; ++k) {
        const long double ar = Are[i * KV + k], ai = Aim[i * KV + k], br = Bre[b * KV + k], bi = Bim[b * KV + k];
        re += ar * br + ai * bi;
        im += ai * br - ar * bi;
      }
      const double gr = V[i * NB + 2 * b], gi = V[i * NB + 2 * b + 1];
      maxerr = fmax(maxerr, fmax(fabs(gr - double(re)), fabs(gi - double(im))));
      maxv = fmax(maxv, fmax(fabs(double(re)), fabs(double(im))));
    }
  printf("V block 128 x 16 complex, K = %d: max |error| %.3e, max |V| %.3e, relative %.3e\n", KV, maxerr, maxv,
         maxerr / maxv);
  return 0;
}
