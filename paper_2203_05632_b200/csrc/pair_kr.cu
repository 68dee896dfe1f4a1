// pair_kr.cu — the pair kernel for Kramers-paired spinor sets (time-reversal symmetric
// references; the generator's inputs and the reference's syn4c fixture, oracle.cpp:346-393).
//
// When the spinor columns come in Kramers pairs (phi, K phi) with K phi = (-Lb*, La*, -Sb*, Sa*)
// and equal energies, every O/V block M = sum_pairs w (phi phi'^H + K phi (K phi')^H) obeys
//   M[beta i, beta j] = conj M[alpha i, alpha j],   M[beta i, alpha j] = -conj M[alpha i, beta j]
// for channels ordered (L alpha, L beta, S alpha, S beta). The literal element-wise sum of the
// reference pair term (estimator.cpp:26-29) then splits as
//   sum_{x,y} o(x,y) v(x,y) = 2 Re sum_{x in {La, Sa}, y} o(x,y) v(x,y),
// so only the alpha rows of V (Q side) and the alpha columns of O~ (P side) are computed: half
// the DMMA work of pair.cu, with identical results to rounding (f1d, f2d, f1x, f2x are real,
// the imaginary residue is exactly 0 where the reference carries ~1e-16 noise).
//
// Structure: persistent CTAs over (8 QB) x 8 walker tiles (QB = 2: 16 Q x 8 P), a TMA producer
// warp filling a 2-stage ring (full/empty mbarriers, running ahead across tiles), 8 QB DMMA
// warps, 3M complex products.
//  * phase 1 (O, K = n_occ): warp w computes O~_e for e = w&1 over 4 Q x 4 P walkers and
//    writes o = conj O~ into the CTA's shared o table (named barriers of four warps between
//    the phases);
//  * phase 2 (V, K = n_vir): warp (wq, wp) owns 4 Q x 2 P walkers (12 accumulator tiles, 96
//    registers), 16 DMMA warps per SM;
//  * epilogue: the element-wise contraction is reduced with shuffles and the four f values of a
//    pair meet in one lane by shuffles; the walker weights are already in Phi_v (mo_kernel).
// OZ instantiation (single ensembles, pair_oz.cu): phase 2 is replaced by the V tile that
// oz_vgemm_kernel wrote for this tile (INT8 tensor cores); the ring carries the O chunks only.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "pair_common.cuh"

#ifdef OZ_OVERLAP_TL
#if defined(KR_PW4_VARIANT)
OVERLAP_TL_DEFINE(g_tl_opass, mcmp2dev_debug_tl_opass)
#elif defined(KR_QB1_VARIANT)
OVERLAP_TL_DEFINE(g_tl_opass, mcmp2dev_debug_tl_opass_qb1)
#else
OVERLAP_TL_DEFINE(g_tl_opass, mcmp2dev_debug_tl_opass_pw2)
#endif
#endif

namespace mcmp2dev {

namespace {
using namespace pairk;
#ifndef KR_STAGES
#define KR_STAGES 2
#endif
// This file is compiled twice (csrc/Makefile): the default QB = 2 build, and with
// -DKR_QB1_VARIANT a QB = 1 build whose entry points carry the suffix _qb1 (kernel
// pair_kr_kernel_qb1). The host takes the QB = 1 variant for ensembles of fewer than 64 walkers:
// 8 x 8 tiles waste fewer pairs of the small triangles and two CTAs per SM overlap the short
// tiles' latencies (batched cfg1, m = 16: pair stage 0.157 -> 0.115 ms at 1184 ensembles), while
// larger m keeps QB = 2 (batched cfg2: 0.146 vs 0.154 ms; cfg4: 4.09 vs 4.18 ms).
#ifdef KR_QB1_VARIANT
#define KR_QB 1
#define KR_API(name) name##_qb1
#elif defined(KR_PW4_VARIANT)
// third build (csrc/Makefile): 8 phase-1 warps of 4 x 8 walkers (NB1 = 2 fragments, more
// independent DMMA chains per warp) for the O-only pass of the INT8 path
#define KR_PW 4
#define KR_API(name) name##_pw4
#else
#define KR_API(name) name
#endif
#ifndef KR_QB
// Q-side walker blocks (of WB) per tile: tile = 8 QB Q walkers x 8 P walkers. Measured cfg4:
// QB 2 (16 DMMA warps, 1 CTA/SM, 25% less stage traffic per DMMA) 4.09 ms, QB 1 (2 CTAs/SM) 4.18 ms
#define KR_QB 2
#endif
// Measured and rejected (cfg4, pair ms): producer in its own warpgroup handing registers to the
// DMMA warps via setmaxnreg (24/112) 4.38; that plus operand double-buffering across k groups
// 4.22; double-buffering within the 96-register cap (spills) 4.41; per-chunk branch-free
// full-chunk path 4.15; 3 stages 4.14; epilogue hinv prefetched at tile start (spills) 4.07; no
// producer warp, the last DMMA warp to release a stage refills it (16 warps, 109 registers) 4.58;
// epilogue hinv fetched by cp.async into shared memory at tile start 4.06; V-phase operand sums
// (ar + ai, br - bi) formed once per stage by the producer warp into shared memory, KC4 6:
// 9.7 (the one warp cannot keep up; removing the DADDs outright would be worth 4.7%); this
// kernel 3.96.
constexpr int STAGES = KR_STAGES;  // ring depth at the widest chunk (KC4 groups)
constexpr int MAX_RING = 16;       // ring depth for narrow chunks: same bytes, more stages
constexpr int QB = KR_QB;
constexpr int QW = WB * QB;                           // Q walkers per tile
#ifndef KR_PW
// PW 4 (8 DMMA warps of 4 x 4 walkers, 9 warps so 168 registers, no spills): cfg4 3.967 ms vs
// 3.961 for PW 2 (16 warps, 96 registers); cfg5-2 5.97 vs 5.08 ms
#define KR_PW 2
#endif
constexpr int PW = KR_PW;                             // P walkers per phase-2 warp (2 or 4)
constexpr int NPW = WB / PW;                          // phase-2 warps per Q group of 4 walkers
constexpr int CONSUMERS = (QW / 4) * NPW;             // 4 Q walkers x PW P walkers per warp
constexpr int P1W = CONSUMERS / ((QW / 4) * 2);       // phase-1 P splits (warp: q group, e, split)
constexpr int NB1 = 2 / P1W;                          // phase-1 n fragments (4 P walkers) per warp
constexpr int GW = CONSUMERS / (QW / 4);              // warps sharing one Q group's o rows
constexpr int THREADS = 32 * (CONSUMERS + 1);
constexpr int MINB = QB == 1 ? 2 : 1;                 // CTAs per SM
constexpr int HALF_PTS = 2 * WB;                      // P points per tile
constexpr int QPTS = 2 * QW;                          // Q points per tile
constexpr int STAGE_DOUBLES = (QPTS + HALF_PTS) * KC4 * 32;
constexpr int SO_DOUBLES = 2 * QW * WB * 4 * 2 * 2;  // CTA o table [e][q][p][y][x_alpha] complex
#ifndef KR_OBUF
#define KR_OBUF ((STAGES * STAGE_DOUBLES + 2 * SO_DOUBLES) * 8 + 2 * MAX_RING * 8 <= 227 * 1024 ? 2 : 1)
#endif
// o tables: with two, tile t writes table t % 2 while no warp can still read it (every warp
// passed tile t-1's "o table complete" barrier after its tile t-2 epilogue), so one CTA barrier
// per tile suffices
constexpr int OBUF = KR_OBUF;
constexpr int SMEM_BYTES =
    (STAGES * STAGE_DOUBLES + OBUF * SO_DOUBLES) * 8 + 2 * MAX_RING * 8;

// The o table rows of Q walkers 4g..4g+3 are written in phase 1 by warps 4g..4g+3 (all (p1w, e1))
// and read in phase 2 by the same four warps (wp = 0..3), so the phase switch synchronises
// groups of four warps (named barriers 1..QB*2), not the whole CTA.
#ifndef KR_GROUP_BARRIER
#define KR_GROUP_BARRIER 1
#endif
__device__ __forceinline__ void consumer_barrier(int group) {
  if (KR_GROUP_BARRIER)
    asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "n"(32 * GW) : "memory");
  else
    asm volatile("bar.sync 1, %0;" ::"n"(CONSUMERS * 32) : "memory");
}

// y is XOR-swizzled by the parity of (q, e): the epilogue's 16-byte reads of one warp then cover
// both halves of a 128-byte row instead of 4 lanes per bank group (4-way -> 2 wavefronts); x_alpha
// by the parity of p, so the phase-1 writes spread over all 8 16-byte slots (8 -> 4 wavefronts).
__device__ __forceinline__ int o_index(int e, int q, int p, int y, int xa) {
  return ((((e * QW + q) * WB + p) * 4 + (y ^ ((q ^ e) & 1))) * 2 + (xa ^ (p & 1))) * 2;
}

// tiles: Q row a covers walker blocks [QB a, QB a + QB), P block b in [0, QB a + QB);
// t = QB a (a + 1) / 2 + b
__device__ __forceinline__ void kr_tile(int t, int& a, int& b) {
  int r = int((sqrt(8.0 * double(t) / QB + 1.0) - 1.0) * 0.5);
  while (QB * (r + 1) * (r + 2) / 2 <= t) ++r;
  while (QB * r * (r + 1) / 2 > t) --r;
  a = r;
  b = t - QB * r * (r + 1) / 2;
}

// the CTA's tile sequence t0, t0 + stride, ... walked without the square root of kr_tile
struct TileWalk {
  int a, b;
  __device__ explicit TileWalk(int t0) { kr_tile(t0, a, b); }
  __device__ void next(int stride) {
    b += stride;
    while (b >= QB * (a + 1)) {  // row a holds QB (a + 1) tiles
      b -= QB * (a + 1);
      ++a;
    }
  }
};

__host__ __device__ constexpr int kr_ntiles(int nb) {
  const int nbq = (nb + QB - 1) / QB;
  return QB * nbq * (nbq + 1) / 2;
}
}  // namespace

// OZ (single ensembles, pair_oz.cu; the ring streams the occupied chunks only):
//  1: the V blocks come precomputed per tile (P.vtiles); the V phase becomes one load per lane
//     and (h, pp) -- the physical estimator;
//  2: O only: the tile's o values go to HBM (P.otiles, [Q block row][p][q][x_alpha][re/im][e_p][y] doubles)
//     and oz_vgemm_kernel<true> contracts them with its V blocks -- the literal estimator
template <bool PHYS, int OZ>
__global__ void __launch_bounds__(THREADS, MINB) KR_API(pair_kr_kernel)(PairParams P) {
  pdl_wait();     // Phi of this step is visible
  pdl_trigger();  // persistent: the next step's walk may launch next to it
  // the INT8 path's guard launch: nothing to do unless this step failed the INT8 checks (the
  // main pass without refinement, or the refinement pass: oz_trip 2)
  if (P.guard_fallback && *reinterpret_cast<volatile const int*>(&P.st->oz_trip) != 2) return;
  if constexpr (OZ == 2) OVERLAP_TL_BEGIN(g_tl_opass);
  extern __shared__ __align__(128) double sm[];
  double* const sO0 = sm + STAGES * STAGE_DOUBLES;
  uint64_t* const full = reinterpret_cast<uint64_t*>(sO0 + OBUF * SO_DOUBLES);
  uint64_t* const empty = full + MAX_RING;
  // ring of P.ring stages of P.ring_doubles each, sized on the host from the widest chunk:
  // the stage region holds STAGES widest stages, and more when every chunk is narrower
  const int ring = P.ring, ring_doubles = P.ring_doubles;
  __shared__ double s_red[CONSUMERS][2];
  __shared__ bool s_last;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // batched ensembles (P.nens > 1): ensemble e owns tiles [e ens_tiles, (e+1) ens_tiles) over its
  // own walkers (points from e 2m), and the pair sums are kept per tile and ensemble
  const bool batched = P.nens > 1;
  const int ntiles = batched ? P.nens * P.ens_tiles : kr_ntiles(P.nb);
  const PhiChunks ch{P.Go, P.Gv};
  const int cO = ch.occ_chunks();  // chunks hold occupied or virtual groups, never both
  const int nchunks = OZ ? cO : ch.count();
  static_assert(OZ != 2 || !PHYS, "the O-only mode serves the literal estimator");
  const int my_tiles = int(blockIdx.x) < ntiles ? (ntiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;

  if (tid == 0) {
    for (int s = 0; s < ring; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CONSUMERS) {
    if (lane == 0) {  // TMA producer
      int stage = 0;
      uint32_t phase = 0;
      TileWalk tw(int(blockIdx.x));
      for (int it = 0; it < my_tiles; ++it, tw.next(int(gridDim.x))) {
        int ta = tw.a, bp = tw.b, pbase = 0;
        if (batched) {
          const int tt = int(blockIdx.x) + it * int(gridDim.x), e = tt / P.ens_tiles;
          kr_tile(tt - e * P.ens_tiles, ta, bp);
          pbase = e * 2 * P.m;
        }
        for (int c = 0; c < nchunks; ++c) {
          mbar_wait(&empty[stage], phase ^ 1u);
          double* dst = sm + stage * ring_doubles;
          const int f = ch.first(c), uc = ch.width(c);
          const uint32_t q_bytes = QPTS * uc * 32 * 8, p_bytes = HALF_PTS * uc * 32 * 8;
          const double* srcq = P.phi + (size_t(f) * P.npts_pad + size_t(pbase + QPTS * ta) * uc) * 32;
          const double* srcp = P.phi + (size_t(f) * P.npts_pad + size_t(pbase + HALF_PTS * bp) * uc) * 32;
          mbar_expect_tx(&full[stage], q_bytes + p_bytes);
          bulk_g2s(dst, srcq, q_bytes, &full[stage]);
          bulk_g2s(dst + QPTS * uc * 32, srcp, p_bytes, &full[stage]);
          if (++stage == ring) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else {
    const int hl = lane >> 4, l16 = lane & 15;
    const int xa_off = 8 * ((lane >> 2) & 1) + (lane & 3);  // alpha channel x = 0 or 2, k = lane & 3
    // phase-1 role: electron e1, 4 Q walkers (4 q1w ..), 4 NB1 P walkers (4 NB1 p1w ..)
    const int e1 = warp & 1, p1w = (warp >> 1) % P1W, q1w = warp / (2 * P1W);
    // phase-2 role: 4 Q walkers (4 wq ..) x PW P walkers (PW wp ..)
    const int wq = warp / NPW, wp = warp % NPW;
    const double cw = P.ng2 / P.st_ro->wtau;
    double acc_d = 0.0, acc_x = 0.0;
    int stage = 0;
    uint32_t phase = 0;
    auto acquire = [&]() -> const double* {
      mbar_wait(&full[stage], phase);
      return sm + stage * ring_doubles;
    };
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == ring) {
        stage = 0;
        phase ^= 1u;
      }
    };

    TileWalk tw(int(blockIdx.x));
    for (int it = 0; it < my_tiles; ++it, tw.next(int(gridDim.x))) {
      int ta = tw.a, bp = tw.b;
      const int tt = int(blockIdx.x) + it * int(gridDim.x);
      if (batched) {
        const int e = tt / P.ens_tiles;
        kr_tile(tt - e * P.ens_tiles, ta, bp);
      }
      const int q0 = QW * ta, p0 = WB * bp;  // first walkers of the tile (within its ensemble)
      double* const sO = sO0 + (it % OBUF) * SO_DOUBLES;
      // OZ: this lane's V values (h, pp) of the tile, loaded before the O phase hides their latency
      double2 ovr[2][PW], ovi[2][PW];
      if constexpr (OZ == 1) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int pp = 0; pp < PW; ++pp) {
            const double* src = P.vtiles + size_t(tt) * 8192 + (4 * wq + 2 * h + hl) * 512 + (PW * wp + pp) * 64 +
                                (lane & 15) * 2;
            ovr[h][pp] = __ldcs(reinterpret_cast<const double2*>(src));
            ovi[h][pp] = __ldcs(reinterpret_cast<const double2*>(src + 32));
          }
      }

      // ---- phase 1: O~_e1 rows (q, y) all channels, cols (p, x_alpha) ----
      {
        double t1[2][NB1][2], t2[2][NB1][2], t3[2][NB1][2];  // [h][n fragment][j]
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int n = 0; n < NB1; ++n) t1[h][n][0] = t1[h][n][1] = t2[h][n][0] = t2[h][n][1] = t3[h][n][0] = t3[h][n][1] = 0.0;
        for (int c = 0; c < cO; ++c) {
          const double* S = acquire();
          const int uc = ch.width(c);
#pragma unroll
          for (int gg = 0; gg < KC4; ++gg) {
            if (gg >= uc) break;  // narrower last chunk
            auto at = [&](int ptl, int plane, int off) {
              return S[(ptl * uc + gg) * 32 + plane * 16 + (off ^ phi_swz(ptl))];
            };
            double br[NB1], bi[NB1], db[NB1];
#pragma unroll
            for (int n = 0; n < NB1; ++n) {
              const int pb = QPTS + 2 * (4 * (NB1 * p1w + n) + (lane >> 3)) + e1;
              br[n] = at(pb, 0, xa_off);
              bi[n] = at(pb, 1, xa_off);
              db[n] = br[n] - bi[n];
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int pa = 2 * (4 * q1w + 2 * h + hl) + e1;
              const double ar = at(pa, 0, l16), ai = at(pa, 1, l16), sa = ar + ai;
#pragma unroll
              for (int n = 0; n < NB1; ++n) {
                dmma(t1[h][n], ar, br[n]);
                dmma(t2[h][n], ai, bi[n]);
                dmma(t3[h][n], sa, db[n]);
              }
            }
          }
          release();
        }
        const int y = (lane >> 2) & 3, pp = lane & 3;
        if constexpr (OZ == 2) {  // o = conj O~ to the tile's O block in HBM; no V phase here
          // The tile's 4096 o values are staged in shared memory in their HBM order,
          //   [p 8][q 16][quad c = (x_alpha, re/im, e_p) ^ (p & 3)][y 4]
          // (the P walkers of a Q block row are contiguous in HBM, so a tile is one 32 KB block and
          // any 10-walker P block of the V-GEMM's tiles one bulk copy; the XOR spreads the four p
          // of a store over the 32-byte slots of a 128-byte row), and leave with one bulk store.
          if (it > 0) {  // the previous tile's store has read the buffer
            if (tid == 0) bulk_store_wait_read();
            asm volatile("bar.sync 15, %0;" ::"n"(CONSUMERS * 32) : "memory");
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int n = 0; n < NB1; ++n)
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const int q = 4 * q1w + 2 * h + hl, p = 4 * (NB1 * p1w + n) + pp;
                double* d = sO0 + p * 512 + q * 32 + y;
                d[(((j * 2 + 0) * 2 + e1) ^ pp) * 4] = t1[h][n][j] + t2[h][n][j];
                d[(((j * 2 + 1) * 2 + e1) ^ pp) * 4] = -(t3[h][n][j] - t1[h][n][j] + t2[h][n][j]);
              }
          fence_proxy_async();
          asm volatile("bar.sync 15, %0;" ::"n"(CONSUMERS * 32) : "memory");
          if (tid == 0) bulk_s2g(P.otiles + size_t(ta) * (ta + 1) * 4096 + size_t(p0) * 512, sO0, 4096 * 8);
          continue;
        }
        if constexpr (OBUF == 1) consumer_barrier(q1w);  // the group is done reading the previous o rows
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int n = 0; n < NB1; ++n)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int idx = o_index(e1, 4 * q1w + 2 * h + hl, 4 * (NB1 * p1w + n) + pp, y, j);
              sO[idx] = t1[h][n][j] + t2[h][n][j];                   // o = conj O~
              sO[idx + 1] = -(t3[h][n][j] - t1[h][n][j] + t2[h][n][j]);
            }
        consumer_barrier(q1w);  // the group's o rows are complete
      }

      // ---- phase 2: V rows (q, e_q, x_alpha), cols (p, e_p, y) ----
      double u1[2][PW][2], u2[2][PW][2], u3[2][PW][2];  // [hq][pp][j]
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < PW; ++j)
          u1[i][j][0] = u1[i][j][1] = u2[i][j][0] = u2[i][j][1] = u3[i][j][0] = u3[i][j][1] = 0.0;
      for (int c = cO; c < nchunks; ++c) {
        const double* S = acquire();
        const int uc = ch.width(c);
#pragma unroll
        for (int gg = 0; gg < KC4; ++gg) {
          if (gg >= uc) break;  // narrower last chunk
          auto at = [&](int ptl, int plane, int off) {
            return S[(ptl * uc + gg) * 32 + plane * 16 + (off ^ phi_swz(ptl))];
          };
          double ar[2], ai[2], sa[2], br[PW], bi[PW], db[PW];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int pa = 2 * (4 * wq + 2 * h + hl) + ((lane >> 3) & 1);
            ar[h] = at(pa, 0, xa_off);
            ai[h] = at(pa, 1, xa_off);
            sa[h] = ar[h] + ai[h];
          }
#pragma unroll
          for (int pp = 0; pp < PW; ++pp) {
            const int pb = QPTS + 2 * (PW * wp + pp) + hl;
            br[pp] = at(pb, 0, l16);
            bi[pp] = at(pb, 1, l16);
            db[pp] = br[pp] - bi[pp];
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int pp = 0; pp < PW; ++pp) {
              dmma(u1[h][pp], ar[h], br[pp]);
              dmma(u2[h][pp], ai[h], bi[pp]);
              dmma(u3[h][pp], sa[h], db[pp]);
            }
        }
        release();
      }

      if constexpr (PHYS) {
        // ---- opt-in physical epilogue: -w_d Tr(o1 va) Tr(o2 vb), -w_x Tr(o1 vd o2 vc) ----
        // Every block M here has the Kramers form M = [[A, B], [-conj B, conj A]] over (alpha | beta)
        // channels with A[i][k] = M(alpha_i, alpha_k), B[i][k] = M(alpha_i, beta_k) (alpha_i = 2i,
        // beta_i = 2i + 1), so MN has A = A_M A_N - B_M conj B_N, B = A_M B_N + B_M conj A_N and
        // Tr(MN) = 2 Re sum_ik (A_M[i][k] A_N[k][i] - B_M[i][k] conj B_N[k][i]). The warp holds the
        // alpha rows of V; lane bits: 0 = y / 2, 1 = e_p, 2 = x_alpha, 3 = e_q, 4 = hl, and
        // register j = y % 2. The o table holds the alpha rows of o1 (e = 0) and o2 (e = 1).
        const int yb = lane & 1, epl = (lane >> 1) & 1, xal = (lane >> 2) & 1, eql = (lane >> 3) & 1;
        const int base = lane & 16;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int pp = 0; pp < PW; ++pp) {
            const int q = 4 * wq + 2 * h + hl, p = PW * wp + pp;
            double vr[2], vi[2];
            if constexpr (OZ == 1) {
              vr[0] = ovr[h][pp].x, vr[1] = ovr[h][pp].y, vi[0] = ovi[h][pp].x, vi[1] = ovi[h][pp].y;
            } else {
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                vr[j] = u1[h][pp][j] + u2[h][pp][j];
                vi[j] = u3[h][pp][j] - u1[h][pp][j] + u2[h][pp][j];
              }
            }
            auto o = [&](int e, int row, int col, double& re, double& im) {  // o_e(alpha_row, col)
              const int idx = o_index(e, q, p, col, row);
              re = sO[idx];
              im = sO[idx + 1];
            };
            // direct traces: lanes of va (e_q = e_p = 0) and vb (1, 1) hold v(alpha_xal, 2 yb + j)
            double tr = 0.0;
            {
              const int e = eql;
              double ar, ai, br, bi;
              o(e, yb, 2 * xal, ar, ai);      // A_o[yb][xal] against A_v[xal][yb] = v(alpha_xal, alpha_yb)
              o(e, yb, 2 * xal + 1, br, bi);  // B_o[yb][xal] against conj B_v[xal][yb] = v(alpha_xal, beta_yb)
              tr = (ar * vr[0] - ai * vi[0]) - (br * vr[1] + bi * vi[1]);
            }
            tr += __shfl_xor_sync(0xffffffffu, tr, 1);
            tr += __shfl_xor_sync(0xffffffffu, tr, 4);
            tr *= 2.0;                                            // lane base + 0: Tr(o1 va)
            const double t2 = __shfl_xor_sync(0xffffffffu, tr, 10);  // lane base + 10: Tr(o2 vb)
            // exchange: lane (i = xal, k2 = yb) forms A/B of (o1 vd)[i][k2] and (o2 vc)[k2][i]
            const int i = xal, c2 = yb;
            double dAr[2], dAi[2], dBr[2], dBi[2], cAr[2], cAi[2], cBr[2], cBi[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int sd = base | (k << 2) | 2 | c2;  // vd = V(e_q 0, e_p 1), column c2
              const int sc = base | 8 | (k << 2) | i;   // vc = V(e_q 1, e_p 0), column i
              dAr[k] = __shfl_sync(0xffffffffu, vr[0], sd);
              dAi[k] = __shfl_sync(0xffffffffu, vi[0], sd);
              dBr[k] = __shfl_sync(0xffffffffu, vr[1], sd);
              dBi[k] = __shfl_sync(0xffffffffu, vi[1], sd);
              cAr[k] = __shfl_sync(0xffffffffu, vr[0], sc);
              cAi[k] = __shfl_sync(0xffffffffu, vi[0], sc);
              cBr[k] = __shfl_sync(0xffffffffu, vr[1], sc);
              cBi[k] = __shfl_sync(0xffffffffu, vi[1], sc);
            }
            double a1r = 0, a1i = 0, b1r = 0, b1i = 0, a2r = 0, a2i = 0, b2r = 0, b2i = 0;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              double oar, oai, obr, obi;
              o(0, i, 2 * k, oar, oai);      // A_o1[i][k]
              o(0, i, 2 * k + 1, obr, obi);  // B_o1[i][k]
              // A1 += A_o1 A_vd - B_o1 conj B_vd; B1 += A_o1 B_vd + B_o1 conj A_vd
              a1r += oar * dAr[k] - oai * dAi[k] - (obr * dBr[k] + obi * dBi[k]);
              a1i += oar * dAi[k] + oai * dAr[k] - (obi * dBr[k] - obr * dBi[k]);
              b1r += oar * dBr[k] - oai * dBi[k] + (obr * dAr[k] + obi * dAi[k]);
              b1i += oar * dBi[k] + oai * dBr[k] + (obi * dAr[k] - obr * dAi[k]);
              o(1, c2, 2 * k, oar, oai);      // A_o2[c2][k]
              o(1, c2, 2 * k + 1, obr, obi);  // B_o2[c2][k]
              a2r += oar * cAr[k] - oai * cAi[k] - (obr * cBr[k] + obi * cBi[k]);
              a2i += oar * cAi[k] + oai * cAr[k] - (obi * cBr[k] - obr * cBi[k]);
              b2r += oar * cBr[k] - oai * cBi[k] + (obr * cAr[k] + obi * cAi[k]);
              b2i += oar * cBi[k] + oai * cBr[k] + (obi * cAr[k] - obr * cAi[k]);
            }
            // Re(A1 A2 - B1 conj B2)
            double tx = (a1r * a2r - a1i * a2i) - (b1r * b2r + b1i * b2i);
            tx += __shfl_xor_sync(0xffffffffu, tx, 1);
            tx += __shfl_xor_sync(0xffffffffu, tx, 4);
            tx *= 2.0;
            if ((lane & 15) == 0) {
              const int qg = q0 + q, pg = p0 + p;
              if (qg < P.m && pg < P.m && qg > pg) {
                acc_d += (-P.w_direct * tr) * t2;
                acc_x += -P.w_exchange * tx;
              }
            }
          }
      } else {
      // ---- epilogue: f = 2 Re sum_{x alpha, y} o v per (e_q, e_p), then real pair terms ----
        const int xa = (lane >> 2) & 1, ep = (lane & 3) >> 1;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int pp = 0; pp < PW; ++pp) {
            const int q = 4 * wq + 2 * h + hl, p = PW * wp + pp;
            double f = 0.0;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int y = 2 * (lane & 1) + j;
              const int idx = o_index(ep, q, p, y, xa);
              const double vr = OZ == 1 ? (j ? ovr[h][pp].y : ovr[h][pp].x) : u1[h][pp][j] + u2[h][pp][j];
              const double vi = OZ == 1 ? (j ? ovi[h][pp].y : ovi[h][pp].x) : u3[h][pp][j] - u1[h][pp][j] + u2[h][pp][j];
              f += sO[idx] * vr - sO[idx + 1] * vi;
            }
            f += __shfl_xor_sync(0xffffffffu, f, 1);
            f += __shfl_xor_sync(0xffffffffu, f, 4);
            f *= 2.0;
            // lanes hl*16 + (e_q << 3) + (e_p << 1) hold f(e_q, e_p) of pair (q, p):
            // f1d = f(0,0), f2x = f(0,1), f1x = f(1,0), f2d = f(1,1)
            const double f2d = __shfl_xor_sync(0xffffffffu, f, 10);
            const double f1x = __shfl_xor_sync(0xffffffffu, f, 8);
            const double f2x = __shfl_xor_sync(0xffffffffu, f, 2);
            if ((lane & 15) == 0) {  // lanes 0, 16: pair (q, p) of this hl
              const int qg = q0 + q, pg = p0 + p;
              if (qg < P.m && pg < P.m && qg > pg) {
                // estimator.cpp:32; the walker weights hinv_p hinv_q of inv_w (estimator.cpp:55) ride
                // in the virtual Phi of the electron-1 points (mo_kernel), the constant
                // N_g^2 / w(tau) is applied once per warp below
                acc_d += (-P.w_direct * f) * f2d;
                acc_x += (-P.w_exchange * f1x) * f2x;
              }
            }
          }
      }
      if (batched) {  // this tile's sums, per warp, unscaled (N_g^2 / w(tau_e) applied per ensemble)
        const double d = acc_d + __shfl_down_sync(0xffffffffu, acc_d, 16);
        const double x = acc_x + __shfl_down_sync(0xffffffffu, acc_x, 16);
        if (lane == 0) {
          P.partials[(size_t(tt) * CONSUMERS + warp) * 2 + 0] = d;
          P.partials[(size_t(tt) * CONSUMERS + warp) * 2 + 1] = x;
        }
        acc_d = acc_x = 0.0;
      }
    }
    acc_d += __shfl_down_sync(0xffffffffu, acc_d, 16);  // lanes 0 and 16 hold the sums
    acc_x += __shfl_down_sync(0xffffffffu, acc_x, 16);
    if (lane == 0) {
      s_red[warp][0] = acc_d * cw;
      s_red[warp][1] = acc_x * cw;
    }
  }
  if constexpr (OZ == 2) {  // the step's sums are oz_vgemm_kernel<true>'s
    if (tid == 0) bulk_store_wait_read();  // the last tile's store is done with shared memory
    OVERLAP_TL_END(g_tl_opass);
    return;
  }
  __syncthreads();
  if (batched) {
    if (tid == 0) {
      __threadfence();
      s_last = atomicAdd(&P.st->done_pair, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // fixed-order sums per ensemble: tiles in order, warps in order
    for (int e = tid; e < P.nens; e += blockDim.x) {
      double d = 0.0, x = 0.0;
      const double* pe = P.partials + size_t(e) * P.ens_tiles * CONSUMERS * 2;
      for (int k = 0; k < P.ens_tiles * CONSUMERS; ++k) {
        d += pe[2 * k];
        x += pe[2 * k + 1];
      }
      const double cwe = P.ng2 / P.st_ro[e].wtau;  // estimator.cpp:55
      d *= cwe;
      x *= cwe;
      const double npairs = 0.5 * P.m * (P.m - 1);
      double* out = P.step_out + size_t(e) * 6;
      out[0] = (d + x) / npairs;
      out[1] = 0.0;
      out[2] = d;
      out[3] = 0.0;
      out[4] = x;
      out[5] = 0.0;
    }
    if (tid == 0) P.st->done_pair = 0;
    return;
  }
  if (tid == 0) {
    double d = 0.0, x = 0.0;
    for (int w = 0; w < CONSUMERS; ++w) {
      d += s_red[w][0];
      x += s_red[w][1];
    }
    P.partials[size_t(blockIdx.x) * 4 + 0] = d;
    P.partials[size_t(blockIdx.x) * 4 + 1] = 0.0;
    P.partials[size_t(blockIdx.x) * 4 + 2] = x;
    P.partials[size_t(blockIdx.x) * 4 + 3] = 0.0;
    __threadfence();
    const unsigned done = atomicAdd(&P.st->done_pair, 1u);
    s_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) {  // fixed-order sum of the per-CTA partials
    double d = 0.0, x = 0.0;
    for (unsigned t = 0; t < gridDim.x; ++t) {
      d += P.partials[size_t(t) * 4 + 0];
      x += P.partials[size_t(t) * 4 + 2];
    }
    const double npairs = 0.5 * P.m * (P.m - 1);
    P.step_out[0] = (d + x) / npairs;
    P.step_out[1] = 0.0;
    P.step_out[2] = d;
    P.step_out[3] = 0.0;
    P.step_out[4] = x;
    P.step_out[5] = 0.0;
    P.st->done_pair = 0;
    if (P.guard_fallback) P.st->oz_trip = 0;
  }
}

namespace {
int g_sms_kr[64];
}

double KR_API(pair_kr_block_tiles)(int nb) { return double(kr_ntiles(nb)) * QB; }
int KR_API(pair_kr_tiles)(int nb) { return kr_ntiles(nb); }
int KR_API(pair_kr_consumers)() { return CONSUMERS; }

void KR_API(pair_kr_ring)(int max_width, int& ring, int& ring_doubles) {
  ring_doubles = (QPTS + HALF_PTS) * max_width * 32;
  ring = (STAGES * STAGE_DOUBLES) / ring_doubles;
  if (ring > MAX_RING) ring = MAX_RING;
}

cudaError_t KR_API(pair_kr_kernel_setup)() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_sms_kr[dev & 63], cudaDevAttrMultiProcessorCount, dev);
  for (auto k : {KR_API(pair_kr_kernel)<false, 0>, KR_API(pair_kr_kernel)<true, 0>, KR_API(pair_kr_kernel)<false, 1>,
                 KR_API(pair_kr_kernel)<true, 1>, KR_API(pair_kr_kernel)<false, 2>}) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

void KR_API(launch_pair_kr)(const PairParams& P, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int ntiles = P.nens > 1 ? P.nens * P.ens_tiles : kr_ntiles(P.nb);
  const int slots = MINB * (g_sms_kr[dev & 63] > 0 ? g_sms_kr[dev & 63] : 148);
  const int grid = ntiles < slots ? ntiles : slots;
  const bool single = P.nens <= 1;
  auto k = P.physical ? (single && P.vtiles ? KR_API(pair_kr_kernel)<true, 1> : KR_API(pair_kr_kernel)<true, 0>)
           : single && P.otiles ? KR_API(pair_kr_kernel)<false, 2>
           : single && P.vtiles ? KR_API(pair_kr_kernel)<false, 1>
                                : KR_API(pair_kr_kernel)<false, 0>;
  pdl_launch(k, dim3(grid), dim3(THREADS), SMEM_BYTES, s, P);
}

}  // namespace mcmp2dev
