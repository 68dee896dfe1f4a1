// spinor.cu — spinor values at the walker points and the MO transform
// (reference proj/core/src/model.cpp:55-64 BasisFunction::value, :166-178
// SpinorSet::evaluate_into, greens.cpp:63-71 set_tau scaling).
//
// Two kernels per step:
//  chi_kernel  basis values chi^g_mu(pt) for every basis group g (a channel, or a Kramers
//              channel pair sharing one basis list), exp(-zeta |r-A|^2) once per unique
//              (centre, zeta) and point, written in DMMA A-fragment order
//              A_g[pt/8][mu/4][lane] (lane = (pt%8)*4 + mu%4).
//  mo_kernel   Phi = chi C as a real x (re|im) DMMA GEMM (mma.sync m8n8k4 f64). B is the
//              coefficient matrix pre-arranged at create time in B-fragment order, so both
//              operands stream from L2 as coalesced 256-byte warp loads. The epilogue scales
//              by sqrt(guarded_exp(+-eps tau)) and scatters into the pair kernel's Phi layout.
// On the Kramers path (exact time-reversal pairs, see pair_kr.cu) only the even columns are
// transformed: for the partner column, Phi^{a}_{2j+1} = -conj Phi^{b}_{2j} and
// Phi^{b}_{2j+1} = conj Phi^{a}_{2j} exactly (same products, negated), halving the GEMM.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "pair_common.cuh"

namespace mcmp2dev {

namespace {
using pairk::dmma;
constexpr int CHI_PTS = 8;
#ifndef CHI_THREADS_N
// measured (cfg4 / cfg2 spinor stage, ms): 128 -> 0.185 / 0.032, 256 -> 0.168 / 0.028,
// 512 -> 0.166 / 0.026 (the basis loops are latency-bound: more threads per 8 points)
#define CHI_THREADS_N 512
#endif
constexpr int CHI_THREADS = CHI_THREADS_N;
#ifndef CHI_UNROLL
#define CHI_UNROLL 1
#endif
constexpr int kChiUnroll = CHI_UNROLL;
constexpr int MO_THREADS = 128;  // 2x2 warps, warp tile 32 points x 4 n-fragments
// k4 steps per cp.async stage and ring depth; measured cfg4 spinor stage (ms): (4, 3) 0.178,
// (2, 4) 0.167, (2, 6) 0.170, (4, 2) 0.173, (1, 8) 0.169; cfg2 prefers (4, 3) by 1 us
#ifndef MO_KS
#define MO_KS 2
#endif
#ifndef MO_STAGES
#define MO_STAGES 4
#endif

__device__ __forceinline__ double ipow(double x, int n) {
  // std::pow(x, n) for n in 0..3 (gaussian.cpp:87-92)
  return n == 0 ? 1.0 : n == 1 ? x : n == 2 ? x * x : x * x * x;
}

// real solid harmonic S_lm as Cartesian monomials (gaussian.cpp:21-39, 87-92)
__device__ double solid_harmonic(int l, int m, double x, double y, double z) {
  constexpr double kS00 = 0.28209479177387814, kS1 = 0.4886025119029199;
  constexpr double kS2a = 1.0925484305920792, kS2b = 0.31539156525252005, kS2c = 0.5462742152960396;
  constexpr double kS3a = 0.5900435899266435, kS3b = 2.890611442640554, kS3c = 0.4570457994644658,
                   kS3d = 0.3731763325901154;
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

__global__ void __launch_bounds__(CHI_THREADS) chi_kernel(SpinorParams P) {
  extern __shared__ double smem[];
  double* s_pos = smem;              // [CHI_PTS][3]
  double* s_exp = s_pos + 3 * CHI_PTS;  // [nuniq][CHI_PTS]
  const int tid = threadIdx.x, pf = blockIdx.x, pt0 = pf * CHI_PTS;
  if (tid < 3 * CHI_PTS) {
    const int pt = tid / 3, k = tid % 3, gp = pt0 + pt;
    s_pos[tid] = gp < P.npts ? P.walkers.at((gp & 1) * 3 + k, gp >> 1) : 0.0;  // 2p <- r1, 2p+1 <- r2
  } else if (tid < 3 * CHI_PTS + CHI_PTS / 2) {
    // walker weight of the pair term: inv_w = N_g^2 / (g1p g2p g1q g2q w(tau)) (estimator.cpp:55)
    // is evaluated as (N_g^2 / w(tau)) hinv_p hinv_q, hinv = 1 / (g1 g2), with hinv folded into
    // Phi_v by mo_kernel (a few ulp from the reference's association)
    const int w = (pt0 >> 1) + tid - 3 * CHI_PTS;
    if (2 * w < P.npts) P.hinv[w] = 1.0 / (P.walkers.at(6, w) * P.walkers.at(7, w));
  }
  __syncthreads();
  for (int i = tid; i < P.nuniq * CHI_PTS; i += CHI_THREADS) {
    const int u = i / CHI_PTS, pt = i % CHI_PTS;
    const double dx = s_pos[3 * pt] - P.uniq_center[3 * u];
    const double dy = s_pos[3 * pt + 1] - P.uniq_center[3 * u + 1];
    const double dz = s_pos[3 * pt + 2] - P.uniq_center[3 * u + 2];
    s_exp[i] = exp(-P.uniq_zeta[u] * (dx * dx + dy * dy + dz * dz));
  }
  __syncthreads();
  for (int g = 0; g < P.ngroups; ++g) {
    const int f0 = P.grp_fn_off[g], nx = P.grp_nfn[g], k4n = P.grp_k4[g];
    double* A = P.chi + P.grp_chi_off[g] + size_t(pf) * k4n * 32;
#pragma unroll kChiUnroll
    for (int i = tid; i < k4n * 32; i += CHI_THREADS) {
      const int k4 = i >> 5, l = i & 31, pt = l >> 2, mu = k4 * 4 + (l & 3);
      double v = 0.0;
      if (mu < nx && pt0 + pt < P.npts) {
        const int f = f0 + mu;
        const double dx = s_pos[3 * pt] - P.fn_center[3 * f];
        const double dy = s_pos[3 * pt + 1] - P.fn_center[3 * f + 1];
        const double dz = s_pos[3 * pt + 2] - P.fn_center[3 * f + 2];
        const double ang = solid_harmonic(P.fn_lm[2 * f], P.fn_lm[2 * f + 1], dx, dy, dz);
        if (ang != 0.0) {  // model.cpp:58 early-out
          double radial = 0.0;
          for (int k = P.fn_prim_off[f]; k < P.fn_prim_off[f + 1]; ++k)
            radial += P.prim_coeff[k] * s_exp[P.prim_uniq[k] * CHI_PTS + pt];
          v = ang * radial;
        }
      }
      A[i] = v;
    }
  }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
  // 16-byte cp.async, zero-filled when !ok (src-size 0)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(pairk::smem_u32(dst)), "l"(src),
               "r"(ok ? 16 : 0)
               : "memory");
}

// Tile: 64 points (8 point fragments) x 8 n fragments of one basis group; 2x2 warps of 4 x 4
// fragments. A (chi) and B (coefficients) k-slices of MO_KS k4 steps stream through a
// MO_STAGES-deep cp.async ring in shared memory, so the DMMAs wait on shared memory, not on
// L2 latency.
using StageA = double[8][MO_KS][32];  // [ptf][k4][lane]
using StageB = double[MO_KS][8][32];  // [k4][nf][lane]
__device__ __forceinline__ void mo_tile(const SpinorParams& P, int g, int ptf_base, int nf_base, StageA* sA,
                                        StageB* sB) {
  const int k4n = P.grp_k4[g], nf_total = P.grp_nf[g];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ptf0 = ptf_base + (warp >> 1) * 4;  // 4 point fragments per warp
  const int nf0 = nf_base + (warp & 1) * 4;     // 4 n fragments per warp (nf_total is a multiple of 4)
  const bool active = nf0 < nf_total;
  const double* A = P.chi + P.grp_chi_off[g];
  const double* B = P.bfrag + P.grp_b_off[g];
  const int nkb = (k4n + MO_KS - 1) / MO_KS;
  auto load_stage = [&](int kb, int st) {
#pragma unroll
    for (int i = tid; i < 8 * MO_KS * 16; i += MO_THREADS) {  // A: 16-byte pieces
      const int ptf = i / (MO_KS * 16), k = (i / 16) % MO_KS, c = i % 16;
      const int k4 = kb * MO_KS + k;
      const bool ok = k4 < k4n;
      cp_async16(&sA[st][ptf][k][2 * c], A + (size_t(ptf_base + ptf) * k4n + (ok ? k4 : 0)) * 32 + 2 * c, ok);
    }
#pragma unroll
    for (int i = tid; i < MO_KS * 8 * 16; i += MO_THREADS) {  // B
      const int k = i / 128, f = (i / 16) % 8, c = i % 16;
      const int k4 = kb * MO_KS + k, nf = nf_base + f;
      const bool ok = k4 < k4n && nf < nf_total;
      cp_async16(&sB[st][k][f][2 * c], B + (size_t(ok ? k4 : 0) * nf_total + (ok ? nf : 0)) * 32 + 2 * c, ok);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int f = 0; f < 4; ++f) acc[i][f][0] = acc[i][f][1] = 0.0;
#pragma unroll
  for (int st = 0; st < MO_STAGES - 1; ++st) {
    if (st < nkb) load_stage(st, st);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kb = 0; kb < nkb; ++kb) {
    asm volatile("cp.async.wait_group %0;" ::"n"(MO_STAGES - 2) : "memory");
    __syncthreads();  // stage kb landed for every thread; stage kb-1 is free
    const int nk = kb + MO_STAGES - 1;
    if (nk < nkb) load_stage(nk, nk % MO_STAGES);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (active) {
      const int st = kb % MO_STAGES;
#pragma unroll
      for (int k = 0; k < MO_KS; ++k) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sA[st][(warp >> 1) * 4 + i][k][lane];
#pragma unroll
        for (int f = 0; f < 4; ++f) b[f] = sB[st][k][(warp & 1) * 4 + f][lane];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int f = 0; f < 4; ++f) dmma(acc[i][f], a[i], b[f]);
      }
    }
  }
  if (!active) return;
  // epilogue: scale and scatter into Phi (layout in common.cuh)
  const PhiChunks ch{P.Go, P.Gv};
  // the walker weight hinv = 1 / (g1 g2) of inv_w (estimator.cpp:55) is folded into the virtual
  // columns of electron-1 points: V(2q, 2p) then carries hinv_q hinv_p, V(2q+1, 2p) hinv_p and
  // V(2q, 2p+1) hinv_q, so both the direct (va vb) and the exchange (vc vd) products of a pair
  // carry exactly hinv_p hinv_q (chi_kernel wrote hinv this step)
  auto put = [&](int x, int pt, double hp, int col, double re, double im) {
    const bool occ = col < P.n_occ;
    const double w = occ ? P.sw[col] : P.sw[col] * hp;
    const int kidx = occ ? col : col - P.n_occ;
    const int grp = occ ? (kidx >> 2) : P.Go + (kidx >> 2);
    double* dst = P.phi + ch.offset(grp, pt, P.npts_pad) + ((x * 4 + (kidx & 3)) ^ phi_swz(pt));
    dst[0] = re * w;
    dst[16] = im * w;
  };
  const int xa = P.grp_chan[2 * g], xb = P.grp_chan[2 * g + 1];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int pt = (ptf0 + i) * 8 + (lane >> 2);
    if (pt >= P.npts) continue;
    const double hp = (pt & 1) ? 1.0 : P.hinv[pt >> 1];
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      const int r8 = 2 * (lane & 3) + jj;
      if (xb < 0) {  // general: two units of 8 columns, fragments (re, im)
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const int col = (nf0 / 2 + uu) * 8 + r8;
          if (col < P.n_p) put(xa, pt, hp, col, acc[i][2 * uu][jj], acc[i][2 * uu + 1][jj]);
        }
      } else {  // Kramers pair: fragments (a re, a im, b re, b im) of even column 2j
        const int j = (nf0 / 4) * 8 + r8, col = 2 * j;
        if (col < P.n_p) {
          const double ar = acc[i][0][jj], ai = acc[i][1][jj], br = acc[i][2][jj], bi = acc[i][3][jj];
          put(xa, pt, hp, col, ar, ai);
          put(xb, pt, hp, col, br, bi);
          put(xa, pt, hp, col + 1, -br, bi);  // -conj(Phi^b_2j)
          put(xb, pt, hp, col + 1, ar, -ai);  //  conj(Phi^a_2j)
        }
      }
    }
  }
}

// One tile per CTA (measured faster than persistent CTAs walking the tiles largest-K first:
// cfg4 spinor stage 0.172 vs 0.186 ms).
__global__ void __launch_bounds__(MO_THREADS) mo_kernel(SpinorParams P) {
  __shared__ __align__(128) StageA sA[MO_STAGES];
  __shared__ __align__(128) StageB sB[MO_STAGES];
  const int g = blockIdx.z, nf_base = blockIdx.y * 8;
  if (nf_base >= P.grp_nf[g]) return;  // uniform over the CTA
  mo_tile(P, g, blockIdx.x * 8, nf_base, sA, sB);
}

int spinor_smem_bytes(const SpinorParams& P) { return int(sizeof(double)) * (3 * CHI_PTS + P.nuniq * CHI_PTS); }

cudaError_t spinor_kernel_setup() {
  return cudaFuncSetAttribute(chi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

void launch_spinor(const SpinorParams& P, cudaStream_t s) {
  const int ptf = (P.npts + CHI_PTS - 1) / CHI_PTS;
  chi_kernel<<<ptf, CHI_THREADS, spinor_smem_bytes(P), s>>>(P);
  const int mtiles = (P.npts + 63) / 64;
  dim3 grid(mtiles, (P.max_nf + 7) / 8, P.ngroups);
  mo_kernel<<<grid, MO_THREADS, 0, s>>>(P);
}

}  // namespace mcmp2dev
