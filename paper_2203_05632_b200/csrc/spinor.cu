// spinor.cu — spinor evaluation at the walker points and the MO transform
// (reference proj/core/src/model.cpp:55-64 BasisFunction::value, :166-178
// SpinorSet::evaluate_into, greens.cpp:63-71 set_tau scaling).
//
// One CTA owns PTS points and one channel x:
//   1. exp(-zeta |r - A|^2) once per unique (centre, zeta) and point (the reference
//      evaluates it per primitive per function; values are identical),
//   2. chi^x_mu(pt) = S_lm(r - A) * sum_k c_k exp(...) into shared memory ([mu][pt]),
//   3. Phi^x[pt][p] = sum_mu chi^x_mu(pt) C[off_x + mu][p] (real x complex), scaled by
//      sqrt(guarded_exp(+-eps_p tau)) and scattered into the pair kernel's fragment layout.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace mcmp2dev {

namespace {
constexpr int PTS = 16;
constexpr int THREADS = 128;

__device__ __forceinline__ double ipow(double x, int n) {
  // std::pow(x, n) for n in 0..3 (gaussian.cpp:87-92)
  return n == 0 ? 1.0 : n == 1 ? x : n == 2 ? x * x : x * x * x;
}

// real solid harmonic S_lm as Cartesian monomials (gaussian.cpp:21-39, 87-92)
__device__ double solid_harmonic(int l, int m, double x, double y, double z) {
  constexpr double kS00 = 0.28209479177387814, kS1 = 0.4886025119029199;
  constexpr double kS2a = 1.0925484305920792, kS2b = 0.31539156525252005,
                   kS2c = 0.5462742152960396;
  constexpr double kS3a = 0.5900435899266435, kS3b = 2.890611442640554,
                   kS3c = 0.4570457994644658, kS3d = 0.3731763325901154;
  double s = 0.0;
  auto t = [&](double c, int ix, int iy, int iz) { s += c * ipow(x, ix) * ipow(y, iy) * ipow(z, iz); };
  switch (l) {
    case 0: t(kS00, 0, 0, 0); break;
    case 1:
      if (m == -1) t(kS1, 0, 1, 0);
      else if (m == 0) t(kS1, 0, 0, 1);
      else t(kS1, 1, 0, 0);
      break;
    case 2:
      switch (m) {
        case -2: t(kS2a, 1, 1, 0); break;
        case -1: t(kS2a, 0, 1, 1); break;
        case 0: t(2 * kS2b, 0, 0, 2); t(-kS2b, 2, 0, 0); t(-kS2b, 0, 2, 0); break;
        case 1: t(kS2a, 1, 0, 1); break;
        default: t(kS2c, 2, 0, 0); t(-kS2c, 0, 2, 0); break;
      }
      break;
    default:
      switch (m) {
        case -3: t(3 * kS3a, 2, 1, 0); t(-kS3a, 0, 3, 0); break;
        case -2: t(kS3b, 1, 1, 1); break;
        case -1: t(4 * kS3c, 0, 1, 2); t(-kS3c, 2, 1, 0); t(-kS3c, 0, 3, 0); break;
        case 0: t(2 * kS3d, 0, 0, 3); t(-3 * kS3d, 2, 0, 1); t(-3 * kS3d, 0, 2, 1); break;
        case 1: t(4 * kS3c, 1, 0, 2); t(-kS3c, 3, 0, 0); t(-kS3c, 1, 2, 0); break;
        case 2: t(kS2c, 2, 0, 1); t(-kS2c, 0, 2, 1); break;
        default: t(kS3a, 3, 0, 0); t(-3 * kS3a, 1, 2, 0); break;
      }
  }
  return s;
}
}  // namespace

__global__ void __launch_bounds__(THREADS) spinor_kernel(SpinorParams P) {
  extern __shared__ double smem[];
  const int x = blockIdx.y;                      // channel
  const int pt0 = blockIdx.x * PTS;
  const int f0 = P.ch_fn_off[x], nx = P.ch_fn_off[x + 1] - f0;
  double* s_pos = smem;                          // [PTS][3]
  double* s_exp = s_pos + 3 * PTS;               // [nuniq][PTS]
  double* s_chi = s_exp + P.nuniq * PTS;         // [nx][PTS]
  const int tid = threadIdx.x;

  if (tid < 3 * PTS) {
    const int pt = tid / 3, k = tid % 3;
    const int gp = pt0 + pt;
    double v = 0.0;
    if (gp < P.npts) v = P.walkers.at((gp & 1) * 3 + k, gp >> 1);  // 2p <- r1, 2p+1 <- r2
    s_pos[tid] = v;
  }
  __syncthreads();
  for (int i = tid; i < P.nuniq * PTS; i += THREADS) {
    const int u = i / PTS, pt = i % PTS;
    const double dx = s_pos[3 * pt] - P.uniq_center[3 * u];
    const double dy = s_pos[3 * pt + 1] - P.uniq_center[3 * u + 1];
    const double dz = s_pos[3 * pt + 2] - P.uniq_center[3 * u + 2];
    const double r2 = dx * dx + dy * dy + dz * dz;
    s_exp[i] = exp(-P.uniq_zeta[u] * r2);
  }
  __syncthreads();
  for (int i = tid; i < nx * PTS; i += THREADS) {
    const int mu = i / PTS, pt = i % PTS, f = f0 + mu;
    const double dx = s_pos[3 * pt] - P.fn_center[3 * f];
    const double dy = s_pos[3 * pt + 1] - P.fn_center[3 * f + 1];
    const double dz = s_pos[3 * pt + 2] - P.fn_center[3 * f + 2];
    const double ang = solid_harmonic(P.fn_lm[2 * f], P.fn_lm[2 * f + 1], dx, dy, dz);
    double v = 0.0;
    if (ang != 0.0) {  // model.cpp:58 early-out
      double radial = 0.0;
      for (int k = P.fn_prim_off[f]; k < P.fn_prim_off[f + 1]; ++k)
        radial += P.prim_coeff[k] * s_exp[P.prim_uniq[k] * PTS + pt];
      v = ang * radial;
    }
    s_chi[i] = v;
  }
  __syncthreads();

  for (int col = tid; col < P.n_p; col += THREADS) {
    double ar[PTS], ai[PTS];
#pragma unroll
    for (int p = 0; p < PTS; ++p) ar[p] = ai[p] = 0.0;
    const double2* cptr = P.C + size_t(f0) * P.n_p + col;
    for (int mu = 0; mu < nx; ++mu) {
      const double2 c = __ldg(cptr + size_t(mu) * P.n_p);
      const double2* chi2 = reinterpret_cast<const double2*>(s_chi + mu * PTS);
#pragma unroll
      for (int p = 0; p < PTS / 2; ++p) {
        const double2 h = chi2[p];
        ar[2 * p] += h.x * c.x;
        ai[2 * p] += h.x * c.y;
        ar[2 * p + 1] += h.y * c.x;
        ai[2 * p + 1] += h.y * c.y;
      }
    }
    const double w = P.sw[col];
    const bool occ = col < P.n_occ;
    const int kidx = occ ? col : col - P.n_occ;
    const int g = occ ? (kidx >> 2) : P.Go + (kidx >> 2);
    const int kk = kidx & 3;
    const int chunk = g / KC4, gg = g % KC4;
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
      const int gp = pt0 + p;
      if (gp < P.npts) {
        double* dst = P.phi + ((size_t(chunk) * P.npts_pad + gp) * KC4 + gg) * 32 + x * 4 + kk;
        dst[0] = ar[p] * w;
        dst[16] = ai[p] * w;
      }
    }
  }
}

int spinor_smem_bytes(const SpinorParams& P) {
  return int(sizeof(double)) * (3 * PTS + P.nuniq * PTS + P.max_ch * PTS);
}

cudaError_t spinor_kernel_setup() {
  return cudaFuncSetAttribute(spinor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

void launch_spinor(const SpinorParams& P, cudaStream_t s) {
  const int smem = spinor_smem_bytes(P);
  dim3 grid((P.npts + PTS - 1) / PTS, P.ncomp);
  spinor_kernel<<<grid, THREADS, smem, s>>>(P);
}

}  // namespace mcmp2dev
