// spinor.cu — spinor values at the walker points and the MO transform
// (reference proj/core/src/model.cpp:55-64 BasisFunction::value, :166-178
// SpinorSet::evaluate_into, greens.cpp:63-71 set_tau scaling).
//
// Two kernels per step:
//  chi_kernel  basis values chi^g_mu(pt) for every basis group g (a channel, or a Kramers
//              channel pair sharing one basis list), exp(-zeta |r-A|^2) once per unique
//              (centre, zeta) and point, written in DMMA A-fragment order
//              A_g[pt/8][mu/4][lane] (lane = (pt%8)*4 + mu%4).
//  mo_kernel   Phi = chi C as a real x (re|im) DMMA GEMM (mma.sync m8n8k4 f64): persistent
//              CTAs, a producer warp streaming contiguous k-slices of A (chi) and B (the
//              coefficients, pre-arranged at create time in B-fragment order) by cp.async.bulk
//              into an mbarrier ring, tiles handed out longest-K first by an atomic counter.
//              The epilogue scales by sqrt(guarded_exp(+-eps tau)) and scatters into the pair
//              kernel's Phi layout.
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
constexpr int CHI_THREADS = CHI_THREADS_N;  // default; chi_kernel is a template on its thread count
#ifndef CHI_UNROLL
#define CHI_UNROLL 1
#endif
constexpr int kChiUnroll = CHI_UNROLL;
// k4 steps per ring stage, ring depth and CTAs per SM of mo_kernel. Measured (ms, spinor stage
// = chi + mo, cfg4 / cfg3): this kernel (KS 4, 4 stages, 3 CTAs, 64-point tiles) 0.163 / 0.042;
// (2, 6) 0.163 / 0.043; (8, 2) 0.168 / 0.042; 4 CTAs (96 registers, spills) 0.179-0.181;
// 128-point tiles (8 DMMA warps) 0.177-0.184; 256-point tiles 0.201. ncu (cfg4): DMMA pipe 61% of
// active cycles; the stall mix is dominated by the epilogue's wait for the last DMMAs of a tile.
// The previous design (one 64x8 tile per CTA, cp.async ring + __syncthreads, 1408 CTAs) measured
// (KS 4, 3 stages) 0.178, (2, 4) 0.165 / 0.038, (2, 6) 0.170, (4, 2) 0.173, (1, 8) 0.169
#ifndef MO_KS
#define MO_KS 4
#endif
#ifndef MO_STAGES
#define MO_STAGES 4
#endif
#ifndef MO_CTAS
#define MO_CTAS 3
#endif
#ifndef MO_WP
#define MO_WP 2  // consumer warps along the points of a tile (tile = 32 MO_WP points x 8 n fragments)
#endif
constexpr int MO_PTF = 4 * MO_WP;  // 8-point fragments per tile

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

template <int CHI_THREADS>
__global__ void __launch_bounds__(CHI_THREADS) chi_kernel(SpinorParams P) {
  pdl_wait();  // this step's walkers are visible
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
    // A fragments of a 64-point tile: [pf / 8][k4][pf % 8][lane], so one k-slice of a tile is
    // contiguous (one bulk copy in mo_kernel)
    double* A = P.chi + P.grp_chi_off[g] + (size_t(pf / MO_PTF) * k4n * MO_PTF + (pf % MO_PTF)) * 32;
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
      A[k4 * MO_PTF * 32 + l] = v;
    }
  }
  pdl_trigger();  // several waves: the MO transform launches once every CTA is done
}

// MO transform: persistent, warp-specialised. Tile = 64 points (8 point fragments) x 8 n
// fragments of one basis group; tiles are handed out longest-K first by an atomic counter
// (dynamic list scheduling: an SM whose CTAs finish early takes more tiles, no static tail).
// A producer warp streams the tile's k-slices (MO_KS k4 steps of A = chi and B = coefficient
// fragments, each one contiguous cp.async.bulk) into a MO_STAGES ring with full/empty
// mbarriers and runs ahead across tile boundaries; 4 DMMA warps (2 x 2, warp tile 32 points x
// 4 n fragments) consume the ring and scatter the tile into Phi.
constexpr int MO_CONSUMERS = 2 * MO_WP;
constexpr int MO_THREADS = 32 * (MO_CONSUMERS + 1);
constexpr int MO_ASLICE = MO_PTF * MO_KS * 32;  // doubles of A per stage
constexpr int MO_BSLICE = 8 * MO_KS * 32;       // doubles of B per stage
constexpr int MO_STAGE = MO_ASLICE + MO_BSLICE;
constexpr int MO_SMEM = MO_STAGES * MO_STAGE * 8 + 2 * MO_STAGES * 8 + MO_STAGES * 8;

__device__ __forceinline__ void mo_decode(const SpinorParams& P, int t, int& g, int& ptile, int& ntile) {
  g = 0;
  while (g + 1 < P.ngroups && t >= P.grp_tile0[g + 1]) ++g;
  const int r = t - P.grp_tile0[g];
  ptile = r / P.grp_nt[g];
  ntile = r % P.grp_nt[g];
}

__global__ void __launch_bounds__(MO_THREADS, MO_CTAS) mo_kernel(SpinorParams P) {
  pdl_wait();     // chi of this step is visible
  pdl_trigger();  // persistent: the pair kernel may launch (it cannot co-reside, so it waits)
  extern __shared__ __align__(128) double mo_sm[];
  uint64_t* const full = reinterpret_cast<uint64_t*>(mo_sm + MO_STAGES * MO_STAGE);
  uint64_t* const empty = full + MO_STAGES;
  int* const head = reinterpret_cast<int*>(empty + MO_STAGES);  // tile id per stage (-1: done)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntiles = P.mo_ntiles;
  if (tid == 0) {
    for (int s = 0; s < MO_STAGES; ++s) {
      pairk::mbar_init(&full[s], 1);
      pairk::mbar_init(&empty[s], MO_CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == MO_CONSUMERS) {
    if (lane == 0) {  // producer
      int stage = 0;
      uint32_t phase = 0;
      for (;;) {
        const int t = int(atomicAdd(&P.st->mo_next, 1u));
        pairk::mbar_wait(&empty[stage], phase ^ 1u);
        if (t >= ntiles) {
          head[stage] = -1;
          pairk::mbar_arrive(&full[stage]);
          break;
        }
        int g, ptile, ntile;
        mo_decode(P, t, g, ptile, ntile);
        const int k4n = P.grp_k4[g];
        const double* A = P.chi + P.grp_chi_off[g] + size_t(ptile) * k4n * MO_PTF * 32;
        const double* B = P.bfrag + P.grp_b_off[g] + size_t(ntile) * k4n * 256;
        for (int k0 = 0; k0 < k4n; k0 += MO_KS) {
          if (k0) pairk::mbar_wait(&empty[stage], phase ^ 1u);
          const int kk = min(MO_KS, k4n - k0);
          head[stage] = t;
          double* dst = mo_sm + stage * MO_STAGE;
          const uint32_t abytes = uint32_t(kk) * MO_PTF * 256u, bbytes = uint32_t(kk) * 2048u;
          pairk::mbar_expect_tx(&full[stage], abytes + bbytes);
          pairk::bulk_g2s(dst, A + size_t(k0) * MO_PTF * 32, abytes, &full[stage]);
          pairk::bulk_g2s(dst + MO_ASLICE, B + size_t(k0) * 256, bbytes, &full[stage]);
          if (++stage == MO_STAGES) stage = 0, phase ^= 1u;
        }
      }
    }
  } else {
    const int wp = warp >> 1, wn = warp & 1;  // warp tile: 4 point fragments x 4 n fragments
    int stage = 0;
    uint32_t phase = 0;
    const PhiChunks ch{P.Go, P.Gv};
    for (;;) {
      pairk::mbar_wait(&full[stage], phase);
      const int t = head[stage];
      if (t < 0) break;
      int g, ptile, ntile;
      mo_decode(P, t, g, ptile, ntile);
      const int k4n = P.grp_k4[g], nf_total = P.grp_nf[g];
      const int nf0 = ntile * 8 + wn * 4;
      const int xa = P.grp_chan[2 * g], xb = P.grp_chan[2 * g + 1];
      // epilogue scale factors, loaded now so their latency hides behind the k loop:
      // sqrt(guarded_exp) of this thread's columns (Kramers partners share the energy) and the
      // walker weight hinv of its electron-1 points
      double swc[2][2], hpv[4];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const int r8 = 2 * (lane & 3) + jj;
          const int col = xb < 0 ? (nf0 / 2 + uu) * 8 + r8 : 2 * ((nf0 / 4) * 8 + r8);
          swc[jj][uu] = (nf0 < nf_total && col < P.n_p && !P.ens_pts) ? P.sw[col] : 0.0;
        }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int pt = (ptile * MO_PTF + wp * 4 + i) * 8 + (lane >> 2);
        hpv[i] = (pt < P.npts && !(pt & 1)) ? P.hinv[pt >> 1] : 1.0;
      }
      double acc[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int f = 0; f < 4; ++f) acc[i][f][0] = acc[i][f][1] = 0.0;
      for (int k0 = 0; k0 < k4n; k0 += MO_KS) {
        if (k0) pairk::mbar_wait(&full[stage], phase);
        const double* sA = mo_sm + stage * MO_STAGE;
        const double* sB = sA + MO_ASLICE;
        const int kk = min(MO_KS, k4n - k0);
#pragma unroll
        for (int k = 0; k < MO_KS; ++k) {
          if (k >= kk) break;
          double a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = sA[(k * MO_PTF + wp * 4 + i) * 32 + lane];
#pragma unroll
          for (int f = 0; f < 4; ++f) b[f] = sB[(k * 8 + wn * 4 + f) * 32 + lane];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int f = 0; f < 4; ++f) pairk::dmma(acc[i][f], a[i], b[f]);
        }
        __syncwarp();
        if (lane == 0) pairk::mbar_arrive(&empty[stage]);
        if (++stage == MO_STAGES) stage = 0, phase ^= 1u;
      }
      if (nf0 >= nf_total) continue;
      // epilogue: scale and scatter into Phi (layout in common.cuh). The walker weight
      // hinv = 1 / (g1 g2) of inv_w (estimator.cpp:55) is folded into the virtual columns of
      // electron-1 points: V(2q, 2p) then carries hinv_q hinv_p, V(2q+1, 2p) hinv_p and
      // V(2q, 2p+1) hinv_q, so both the direct (va vb) and the exchange (vc vd) products of a
      // pair carry exactly hinv_p hinv_q (chi_kernel wrote hinv this step)
      auto put = [&](int x, int pt, double w, int col, double re, double im) {
        const int kidx = col < P.n_occ ? col : col - P.n_occ;
        const int grp = col < P.n_occ ? (kidx >> 2) : P.Go + (kidx >> 2);
        double* dst = P.phi + ch.offset(grp, pt, P.npts_pad) + ((x * 4 + (kidx & 3)) ^ phi_swz(pt));
        dst[0] = re * w;
        dst[16] = im * w;
      };
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int pt = (ptile * MO_PTF + wp * 4 + i) * 8 + (lane >> 2);
        if (pt >= P.npts) continue;
        // batched ensembles: this point's ensemble has its own tau (8-point fragments never
        // straddle ensembles: ens_pts is a multiple of 32)
        const double* swb = P.ens_pts ? P.sw + size_t(pt / P.ens_pts) * P.sw_stride : nullptr;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int r8 = 2 * (lane & 3) + jj;
          if (xb < 0) {  // general: two units of 8 columns, fragments (re, im)
#pragma unroll
            for (int uu = 0; uu < 2; ++uu) {
              const int col = (nf0 / 2 + uu) * 8 + r8;
              const double sv = swb ? (col < P.n_p ? swb[col] : 0.0) : swc[jj][uu];
              const double w = col < P.n_occ ? sv : sv * hpv[i];
              if (col < P.n_p) put(xa, pt, w, col, acc[i][2 * uu][jj], acc[i][2 * uu + 1][jj]);
            }
          } else {  // Kramers pair: fragments (a re, a im, b re, b im) of even column 2j
            const int j = (nf0 / 4) * 8 + r8, col = 2 * j;
            if (col < P.n_p) {
              const double sv = swb ? swb[col] : swc[jj][0];
              const double w = col < P.n_occ ? sv : sv * hpv[i];
              const double ar = acc[i][0][jj], ai = acc[i][1][jj], br = acc[i][2][jj], bi = acc[i][3][jj];
              // columns 2j (a, b) and 2j + 1 (-conj b, conj a) are neighbours in Phi (n_occ is even
              // on this path, so both sit in one group of four): one 16-byte store per plane
              const int kidx = col < P.n_occ ? col : col - P.n_occ;
              const int grp = col < P.n_occ ? (kidx >> 2) : P.Go + (kidx >> 2);
              double* base = P.phi + ch.offset(grp, pt, P.npts_pad);
              double* da = base + ((xa * 4 + (kidx & 3)) ^ phi_swz(pt));
              double* db = base + ((xb * 4 + (kidx & 3)) ^ phi_swz(pt));
              *reinterpret_cast<double2*>(da) = make_double2(ar * w, -br * w);       // re: a, -conj b
              *reinterpret_cast<double2*>(da + 16) = make_double2(ai * w, bi * w);   // im
              *reinterpret_cast<double2*>(db) = make_double2(br * w, ar * w);        // re: b, conj a
              *reinterpret_cast<double2*>(db + 16) = make_double2(bi * w, -ai * w);  // im
            }
          }
        }
      }
    }
  }
  // the last CTA out resets the tile counter for the next launch
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&P.st->mo_done, 1u) == gridDim.x - 1) {
      P.st->mo_next = 0;
      P.st->mo_done = 0;
    }
  }
}

int spinor_smem_bytes(const SpinorParams& P) { return int(sizeof(double)) * (3 * CHI_PTS + P.nuniq * CHI_PTS); }

cudaError_t spinor_kernel_setup() {
  cudaError_t e = cudaFuncSetAttribute(chi_kernel<CHI_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(chi_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(mo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MO_SMEM);
}

void launch_spinor(const SpinorParams& P, cudaStream_t s) {
  const int ptf = (P.npts + CHI_PTS - 1) / CHI_PTS;
  // small bases (few values per 8-point fragment, e.g. cfg1: 384 values + 96 exps): 128 threads
  // per fragment, more CTAs resident per SM; measured (cfg1 x 1184 ensembles) in profiles/README
  int work = P.nuniq * CHI_PTS;
  for (int g = 0; g < P.ngroups; ++g) work += P.grp_k4[g] * 32;
  if (work <= 640) pdl_launch(chi_kernel<128>, dim3(ptf), dim3(128), spinor_smem_bytes(P), s, P);
  else pdl_launch(chi_kernel<CHI_THREADS>, dim3(ptf), dim3(CHI_THREADS), spinor_smem_bytes(P), s, P);
  SpinorParams q = P;
  const int ptiles = (P.npts + 8 * MO_PTF - 1) / (8 * MO_PTF);  // tiles are numbered group-major, so the tile range of
  int total = 0;                            // this launch's point count is recomputed here
  for (int g = 0; g < P.ngroups; ++g) {
    q.grp_tile0[g] = total;
    total += ptiles * P.grp_nt[g];
  }
  q.mo_ntiles = total;
  int grid = P.mo_slots;
  if (grid > total) grid = total;
  pdl_launch(mo_kernel, dim3(grid), dim3(MO_THREADS), MO_SMEM, s, q);
}

int mo_ctas_per_sm() { return MO_CTAS; }

}  // namespace mcmp2dev
