// pair.cu — O/V Green's-function blocks for all walker pairs at one tau, the fused
// direct/exchange integrand and the deterministic block reduction
// (reference proj/core/src/greens.cpp:73-79, estimator.cpp:15-63).
//
// For walkers p < q the reference forms six 4x4 complex blocks (estimator.cpp:17-24):
//   o1 = O(2p, 2q), o2 = O(2p+1, 2q+1)             O(d,o) = Phi_o(d) diag(w) Phi_o(o)^H
//   va = V(2q, 2p), vb = V(2q+1, 2p+1), vc = V(2q+1, 2p), vd = V(2q, 2p+1)
// and the literal element-wise sums f1d = sum o1.va, f2d = sum o2.vb, f1x = sum o1.vc,
// f2x = sum o2.vd. Over all pairs these are batched Hermitian-type complex GEMMs. Here one
// CTA owns an 8x8 tile of walker pairs (Q block x P block, Q >= P): the V products over the
// tile are an (8 walkers x 2 electrons x 4 channels)^2 complex GEMM with K = n_vir, the O
// products two (8 x 4)^2 GEMMs (one per electron) with K = n_occ. Each complex GEMM is four
// real DMMA products (mma.sync m8n8k4 f64; tcgen05 has no f64 kind) on real-split operands
// staged by TMA bulk copies. G is never written to memory: the accumulators are contracted
// in registers and only four doubles per CTA leave the SM.
//
// Persistent: one CTA per SM walks a static list of tiles. Warp 8 is the TMA producer (bulk
// copies into a 4-stage ring guarded by full/empty mbarriers, running ahead across tile
// boundaries so the next tile's first stages land during this tile's epilogue); warps 0-7
// issue the DMMAs. Complex products use 3 real products (3M): t1 = ar br, t2 = ai bi,
// t3 = (ar + ai)(br - bi); re = t1 + t2, im = t3 - t1 + t2.
//
// Warp (wq, wp) owns Q walkers 2wq..2wq+1 x P walkers 4wp..4wp+3 (8 pairs). One m8n8k4
// accumulator tile of V is exactly one walker pair (rows = q's (electron, channel), cols =
// p's). The O tiles are computed transposed (rows = Q side) and exchanged through shared
// memory, since the literal contraction pairs p's channel x with q's channel x.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "pair_common.cuh"

namespace mcmp2dev {

namespace {
constexpr int CONSUMERS = 8;                              // MMA warps (wq 0..3 x wp 0..1)
constexpr int THREADS = 32 * (CONSUMERS + 1);             // + one TMA producer warp
constexpr int HALF_PTS = 2 * WB;                          // 16 points per walker block
constexpr int STAGE_DOUBLES = 2 * HALF_PTS * KC4 * 32;    // 32 points x KC4 groups x 32
constexpr int SO_DOUBLES = 512;                           // per consumer warp: 2x2x4 blocks of 4x4 complex
constexpr int SV_DOUBLES = 8 * 64 * 2;                    // physical epilogue: 8 pairs x 8x8 complex V

template <bool PHYS>
struct Cfg {
  static constexpr int FIXED_BYTES = (CONSUMERS * SO_DOUBLES + (PHYS ? CONSUMERS * SV_DOUBLES : 0)) * 8;
  static constexpr int FIT = (227 * 1024 - FIXED_BYTES) / (STAGE_DOUBLES * 8 + 16);  // stages that fit
  static constexpr int STAGES = (PHYS ? 3 : 4) < FIT ? (PHYS ? 3 : 4) : FIT;
  static_assert(STAGES >= 2, "KC4 too large for a two-stage ring");
  static constexpr int SMEM_BYTES = FIXED_BYTES + STAGES * (STAGE_DOUBLES * 8 + 16);
};

}  // namespace
using namespace pairk;

template <bool PHYS>
__global__ void __launch_bounds__(THREADS, 1) pair_kernel(PairParams P) {
  pdl_wait();
  pdl_trigger();
  constexpr int STAGES = Cfg<PHYS>::STAGES;
  extern __shared__ __align__(128) double sm[];
  double* const sO = sm + STAGES * STAGE_DOUBLES;  // [warp][e][qi][pj][y][x] complex o
  double* const sV = sO + CONSUMERS * SO_DOUBLES;  // PHYS only: [warp][pair][e_q][e_p][x][y]
  uint64_t* const full = reinterpret_cast<uint64_t*>(sV + (PHYS ? CONSUMERS * SV_DOUBLES : 0));
  uint64_t* const empty = full + STAGES;
  __shared__ double s_red[CONSUMERS][4];
  __shared__ bool s_last;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // batched ensembles (P.nens > 1): ensemble e owns tiles [e ens_tiles, (e+1) ens_tiles) of its
  // own triangle (points from e 2m); sums are kept per tile and reduced per ensemble
  const bool batched = P.nens > 1;
  const int ntiles = batched ? P.nens * P.ens_tiles : P.nb * (P.nb + 1) / 2;
  const PhiChunks ch{P.Go, P.Gv};
  const int nchunks = ch.count();
  const int cO = ch.occ_chunks();  // chunks hold occupied or virtual groups, never both
  const int my_tiles = int(blockIdx.x) < ntiles ? (ntiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CONSUMERS) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      long long seq = 0;
      for (int it = 0; it < my_tiles; ++it) {
        int bq, bp, pbase = 0;
        {
          int tt = int(blockIdx.x) + it * int(gridDim.x);
          if (batched) {
            const int e = tt / P.ens_tiles;
            tt -= e * P.ens_tiles;
            pbase = e * 2 * P.m;
          }
          tile_coords(tt, bq, bp);
        }
        for (int c = 0; c < nchunks; ++c, ++seq) {
          const int stage = int(seq % STAGES);
          mbar_wait(&empty[stage], uint32_t(((seq / STAGES) & 1) ^ 1));
          double* dst = sm + stage * STAGE_DOUBLES;
          const int f = ch.first(c), uc = ch.width(c);
          const uint32_t half_bytes = HALF_PTS * uc * 32 * 8;
          const double* srcq = P.phi + (size_t(f) * P.npts_pad + size_t(pbase + HALF_PTS * bq) * uc) * 32;
          const double* srcp = P.phi + (size_t(f) * P.npts_pad + size_t(pbase + HALF_PTS * bp) * uc) * 32;
          mbar_expect_tx(&full[stage], 2 * half_bytes);
          bulk_g2s(dst, srcq, half_bytes, &full[stage]);
          bulk_g2s(dst + HALF_PTS * uc * 32, srcp, half_bytes, &full[stage]);
        }
      }
    }
  } else {
    // ---------------- DMMA consumers ----------------
    const int wq = warp >> 1, wp = warp & 1;
    const int hl = lane >> 4, l16 = lane & 15;
    double* const so = sO + warp * SO_DOUBLES;
    const double cw = P.ng2 / P.st_ro->wtau;
    double acc_dr = 0.0, acc_di = 0.0, acc_xr = 0.0, acc_xi = 0.0;
    long long seq = 0;
    auto acquire = [&]() -> const double* {
      const int stage = int(seq % STAGES);
      mbar_wait(&full[stage], uint32_t((seq / STAGES) & 1));
      return sm + stage * STAGE_DOUBLES;
    };
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[int(seq % STAGES)]);
      ++seq;
    };

    for (int it = 0; it < my_tiles; ++it) {
      int bq, bp;
      const int tt = int(blockIdx.x) + it * int(gridDim.x);
      tile_coords(batched ? tt % P.ens_tiles : tt, bq, bp);
      // batched: this tile's sums, per warp, unscaled (N_g^2 / w(tau_e) applied per ensemble)
      auto flush_tile = [&]() {
        if (!batched) return;
        double r[4] = {acc_dr, acc_di, acc_xr, acc_xi};
        if constexpr (PHYS) {  // lanes 0..7 hold the tile's partial sums
#pragma unroll
          for (int o = 4; o; o >>= 1)
#pragma unroll
            for (int k = 0; k < 4; ++k) r[k] += __shfl_down_sync(0xffffffffu, r[k], o);
        }
        if (lane == 0)
          for (int k = 0; k < 4; ++k) P.partials[(size_t(tt) * CONSUMERS + warp) * 4 + k] = r[k];
        acc_dr = acc_di = acc_xr = acc_xi = 0.0;
      };

      // ---- phase 1: O~_e(q,y; p,x) = sum_i Phi_o(q,e,y,i) conj Phi_o(p,e,x,i) ----
      {
        double t1[2][2][2], t2[2][2][2], t3[2][2][2];
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < 2; ++j) t1[e][h][j] = t2[e][h][j] = t3[e][h][j] = 0.0;
        for (int c = 0; c < cO; ++c) {
          const double* S = acquire();
          const int uc = ch.width(c);
#pragma unroll
          for (int gg = 0; gg < KC4; ++gg) {
            if (gg >= uc) break;  // narrower last chunk
            auto frag = [&](int ptl, int plane) { return S[(ptl * uc + gg) * 32 + plane * 16 + (l16 ^ phi_swz(ptl))]; };
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int pa = 2 * (2 * wq + hl) + e;
              const double ar = frag(pa, 0), ai = frag(pa, 1), sa = ar + ai;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int pb = HALF_PTS + 2 * (4 * wp + 2 * h + hl) + e;
                const double br = frag(pb, 0), bi = frag(pb, 1);
                dmma(t1[e][h], ar, br);
                dmma(t2[e][h], ai, bi);
                dmma(t3[e][h], sa, br - bi);
              }
            }
          }
          release();
        }
        // o = conj(O~) into this warp's slot
        const int qi = hl, y = (lane >> 2) & 3;
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int pj = 2 * h + ((lane & 3) >> 1), x = 2 * (lane & 1) + j;
              const int idx = ((((e * 2 + qi) * 4 + pj) * 16) + y * 4 + x) * 2;
              so[idx] = t1[e][h][j] + t2[e][h][j];
              so[idx + 1] = -(t3[e][h][j] - t1[e][h][j] + t2[e][h][j]);
            }
      }

      // ---- phase 2: V(q,e_q,x; p,e_p,y) = sum_a Phi_v(q,e_q,x,a) conj Phi_v(p,e_p,y,a) ----
      double u1[2][4][2], u2[2][4][2], u3[2][4][2];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          u1[i][j][0] = u1[i][j][1] = u2[i][j][0] = u2[i][j][1] = u3[i][j][0] = u3[i][j][1] = 0.0;
      for (int c = cO; c < nchunks; ++c) {
        const double* S = acquire();
        const int uc = ch.width(c);
#pragma unroll
        for (int gg = 0; gg < KC4; ++gg) {
          if (gg >= uc) break;  // narrower last chunk
          auto frag = [&](int ptl, int plane) { return S[(ptl * uc + gg) * 32 + plane * 16 + (l16 ^ phi_swz(ptl))]; };
          double ar[2], ai[2], sa[2], br[4], bi[4], db[4];
#pragma unroll
          for (int qi = 0; qi < 2; ++qi) {
            const int pa = 2 * (2 * wq + qi) + hl;
            ar[qi] = frag(pa, 0);
            ai[qi] = frag(pa, 1);
            sa[qi] = ar[qi] + ai[qi];
          }
#pragma unroll
          for (int pj = 0; pj < 4; ++pj) {
            const int pb = HALF_PTS + 2 * (4 * wp + pj) + hl;
            br[pj] = frag(pb, 0);
            bi[pj] = frag(pb, 1);
            db[pj] = br[pj] - bi[pj];
          }
#pragma unroll
          for (int qi = 0; qi < 2; ++qi)
#pragma unroll
            for (int pj = 0; pj < 4; ++pj) {
              dmma(u1[qi][pj], ar[qi], br[pj]);
              dmma(u2[qi][pj], ai[qi], bi[pj]);
              dmma(u3[qi][pj], sa[qi], db[pj]);
            }
        }
        release();
      }

      if constexpr (PHYS) {
        // ---- opt-in physical epilogue: -w_d Tr(o1 va) Tr(o2 vb), -w_x Tr(o1 vd o2 vc)
        double* const sv = sV + warp * SV_DOUBLES;  // [pair][e_q][e_p][x][y] complex
        {
          const int eq = hl, x = (lane >> 2) & 3, ep = (lane & 3) >> 1;
#pragma unroll
          for (int qi = 0; qi < 2; ++qi)
#pragma unroll
            for (int pj = 0; pj < 4; ++pj)
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const int y = 2 * (lane & 1) + j;
                const int idx = (((((qi * 4 + pj) * 2 + eq) * 2 + ep) * 16) + x * 4 + y) * 2;
                sv[idx] = u1[qi][pj][j] + u2[qi][pj][j];
                sv[idx + 1] = u3[qi][pj][j] - u1[qi][pj][j] + u2[qi][pj][j];
              }
        }
        __syncwarp();
        if (lane < 8) {
          const int qi = lane >> 2, pj = lane & 3;
          const int q = WB * bq + 2 * wq + qi, p = WB * bp + 4 * wp + pj;
          if (q < P.m && p < P.m && q > p) {
            auto O = [&](int e, int x, int y, int c) { return so[((((e * 2 + qi) * 4 + pj) * 16) + y * 4 + x) * 2 + c]; };
            auto V = [&](int eq, int ep, int x, int y, int c) {
              return sv[(((((qi * 4 + pj) * 2 + eq) * 2 + ep) * 16) + x * 4 + y) * 2 + c];
            };
            // t1 = Tr(o1 va), t2 = Tr(o2 vb): va = V(eq 0, ep 0), vb = V(1, 1)
            double t1r = 0, t1i = 0, t2r = 0, t2i = 0;
            for (int x = 0; x < 4; ++x)
              for (int y = 0; y < 4; ++y) {
                double ar = O(0, x, y, 0), ai = O(0, x, y, 1), br = V(0, 0, y, x, 0), bi = V(0, 0, y, x, 1);
                t1r += ar * br - ai * bi;
                t1i += ar * bi + ai * br;
                ar = O(1, x, y, 0), ai = O(1, x, y, 1), br = V(1, 1, y, x, 0), bi = V(1, 1, y, x, 1);
                t2r += ar * br - ai * bi;
                t2i += ar * bi + ai * br;
              }
            // tx = Tr(m1 m2), m1 = o1 vd (vd = V(0, 1)), m2 = o2 vc (vc = V(1, 0))
            double m1[4][4][2], m2[4][4][2];
            for (int x = 0; x < 4; ++x)
              for (int y = 0; y < 4; ++y) {
                double ar = 0, ai = 0, br = 0, bi = 0;
                for (int k = 0; k < 4; ++k) {
                  const double o1r = O(0, x, k, 0), o1i = O(0, x, k, 1), dr = V(0, 1, k, y, 0), di = V(0, 1, k, y, 1);
                  ar += o1r * dr - o1i * di;
                  ai += o1r * di + o1i * dr;
                  const double o2r = O(1, x, k, 0), o2i = O(1, x, k, 1), cr = V(1, 0, k, y, 0), ci = V(1, 0, k, y, 1);
                  br += o2r * cr - o2i * ci;
                  bi += o2r * ci + o2i * cr;
                }
                m1[x][y][0] = ar, m1[x][y][1] = ai, m2[x][y][0] = br, m2[x][y][1] = bi;
              }
            double txr = 0, txi = 0;
            for (int x = 0; x < 4; ++x)
              for (int y = 0; y < 4; ++y) {
                txr += m1[x][y][0] * m2[y][x][0] - m1[x][y][1] * m2[y][x][1];
                txi += m1[x][y][0] * m2[y][x][1] + m1[x][y][1] * m2[y][x][0];
              }
            // hinv_p hinv_q of inv_w ride in Phi_v (mo_kernel); N_g^2 / w(tau) is applied per warp
            const double adr = -P.w_direct * t1r, adi = -P.w_direct * t1i;
            acc_dr += adr * t2r - adi * t2i;
            acc_di += adr * t2i + adi * t2r;
            acc_xr += -P.w_exchange * txr;
            acc_xi += -P.w_exchange * txi;
          }
        }
        __syncwarp();
        flush_tile();
        continue;
      }

      // ---- epilogue: literal element-wise contraction of o with V (estimator.cpp:26-32) ----
      const int xx = (lane >> 2) & 3, ep = (lane & 3) >> 1;
#pragma unroll
      for (int qi = 0; qi < 2; ++qi)
#pragma unroll
        for (int pj = 0; pj < 4; ++pj) {
          double fr = 0.0, fi = 0.0;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int y = 2 * (lane & 1) + j;
            const int idx = ((((ep * 2 + qi) * 4 + pj) * 16) + y * 4 + xx) * 2;
            const double orr = so[idx], oii = so[idx + 1];
            const double vr = u1[qi][pj][j] + u2[qi][pj][j];
            const double vi = u3[qi][pj][j] - u1[qi][pj][j] + u2[qi][pj][j];
            fr += orr * vr - oii * vi;
            fi += orr * vi + oii * vr;
          }
#pragma unroll
          for (int o = 1; o <= 8; o <<= 1) {
            if (o == 2) continue;
            fr += __shfl_xor_sync(0xffffffffu, fr, o);
            fi += __shfl_xor_sync(0xffffffffu, fi, o);
          }
          // lane 0: (e_q,e_p) = (0,0) f1d; lane 18: (1,1) f2d; lane 16: (1,0) f1x; lane 2: (0,1) f2x
          const double f1dr = __shfl_sync(0xffffffffu, fr, 0), f1di = __shfl_sync(0xffffffffu, fi, 0);
          const double f2dr = __shfl_sync(0xffffffffu, fr, 18), f2di = __shfl_sync(0xffffffffu, fi, 18);
          const double f1xr = __shfl_sync(0xffffffffu, fr, 16), f1xi = __shfl_sync(0xffffffffu, fi, 16);
          const double f2xr = __shfl_sync(0xffffffffu, fr, 2), f2xi = __shfl_sync(0xffffffffu, fi, 2);
          if (lane == 0) {
            const int q = WB * bq + 2 * wq + qi, p = WB * bp + 4 * wp + pj;
            if (q < P.m && p < P.m && q > p) {
              // -w_d f1d f2d inv, -w_x f1x f2x inv (estimator.cpp:32); hinv_p hinv_q of inv_w ride
              // in Phi_v (mo_kernel), N_g^2 / w(tau) is applied per warp
              const double adr = -P.w_direct * f1dr, adi = -P.w_direct * f1di;
              const double axr = -P.w_exchange * f1xr, axi = -P.w_exchange * f1xi;
              acc_dr += adr * f2dr - adi * f2di;
              acc_di += adr * f2di + adi * f2dr;
              acc_xr += axr * f2xr - axi * f2xi;
              acc_xi += axr * f2xi + axi * f2xr;
            }
          }
        }
      __syncwarp();  // all lanes done reading `so` before the next tile rewrites it
      flush_tile();
    }
    if constexpr (PHYS) {  // lanes 0..7 hold partial sums: fixed shuffle tree into lane 0
#pragma unroll
      for (int o = 4; o; o >>= 1) {
        acc_dr += __shfl_down_sync(0xffffffffu, acc_dr, o);
        acc_di += __shfl_down_sync(0xffffffffu, acc_di, o);
        acc_xr += __shfl_down_sync(0xffffffffu, acc_xr, o);
        acc_xi += __shfl_down_sync(0xffffffffu, acc_xi, o);
      }
    }
    if (lane == 0) {
      s_red[warp][0] = acc_dr * cw;
      s_red[warp][1] = acc_di * cw;
      s_red[warp][2] = acc_xr * cw;
      s_red[warp][3] = acc_xi * cw;
    }
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
    for (int e = tid; e < P.nens; e += THREADS) {  // fixed order: tiles, then warps
      double a[4] = {0, 0, 0, 0};
      const double* pe = P.partials + size_t(e) * P.ens_tiles * CONSUMERS * 4;
      for (int k = 0; k < P.ens_tiles * CONSUMERS; ++k)
        for (int j = 0; j < 4; ++j) a[j] += pe[4 * k + j];
      const double cwe = P.ng2 / P.st_ro[e].wtau;  // estimator.cpp:55
      for (int j = 0; j < 4; ++j) a[j] *= cwe;
      const double npairs = 0.5 * P.m * (P.m - 1);  // estimator.cpp:61
      double* out = P.step_out + size_t(e) * 6;
      out[0] = (a[0] + a[2]) / npairs;
      out[1] = (a[1] + a[3]) / npairs;
      out[2] = a[0];
      out[3] = a[1];
      out[4] = a[2];
      out[5] = a[3];
    }
    if (tid == 0) P.st->done_pair = 0;
    return;
  }
  if (tid == 0) {
    double r[4] = {0, 0, 0, 0};
    for (int w = 0; w < CONSUMERS; ++w)
      for (int k = 0; k < 4; ++k) r[k] += s_red[w][k];
    for (int k = 0; k < 4; ++k) P.partials[size_t(blockIdx.x) * 4 + k] = r[k];
    __threadfence();
    const unsigned done = atomicAdd(&P.st->done_pair, 1u);
    s_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // ---- last CTA: fixed-order sum over the per-CTA partials -> StepEstimate ----
  double r[4] = {0, 0, 0, 0};
  for (unsigned t = tid; t < gridDim.x; t += THREADS)
    for (int k = 0; k < 4; ++k) r[k] += P.partials[size_t(t) * 4 + k];
  double* red = sm;  // [THREADS][4]
  for (int k = 0; k < 4; ++k) red[tid * 4 + k] = r[k];
  __syncthreads();
  if (tid == 0) {
    double a[4] = {0, 0, 0, 0};
    for (int t = 0; t < THREADS; ++t)
      for (int k = 0; k < 4; ++k) a[k] += red[t * 4 + k];
    const double npairs = 0.5 * P.m * (P.m - 1);  // estimator.cpp:61
    P.step_out[0] = (a[0] + a[2]) / npairs;
    P.step_out[1] = (a[1] + a[3]) / npairs;
    P.step_out[2] = a[0];
    P.step_out[3] = a[1];
    P.step_out[4] = a[2];
    P.step_out[5] = a[3];
    P.st->done_pair = 0;
  }
}

namespace {
int g_sms[64];
}

cudaError_t pair_kernel_setup() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_sms[dev & 63], cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaFuncSetAttribute(pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg<false>::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<true>::SMEM_BYTES);
}

int pair_grid(int nb, int nens, int ens_tiles) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int ntiles = nens > 1 ? nens * ens_tiles : nb * (nb + 1) / 2;
  const int sms = g_sms[dev & 63] > 0 ? g_sms[dev & 63] : 148;
  return ntiles < sms ? ntiles : sms;
}

void launch_pair(const PairParams& P, cudaStream_t s) {
  if (P.physical)
    pdl_launch(pair_kernel<true>, dim3(pair_grid(P.nb, P.nens, P.ens_tiles)), dim3(THREADS), Cfg<true>::SMEM_BYTES, s, P);
  else
    pdl_launch(pair_kernel<false>, dim3(pair_grid(P.nb, P.nens, P.ens_tiles)), dim3(THREADS), Cfg<false>::SMEM_BYTES,
               s, P);
}

int pair_consumers() { return CONSUMERS; }

}  // namespace mcmp2dev
