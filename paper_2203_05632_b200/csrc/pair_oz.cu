// pair_oz.cu — the virtual Green's-function blocks of the Kramers pair stage on the INT8 tensor
// cores (tcgen05.mma kind::i8), FP64-accurate by Ozaki splitting.
//
// Over a walker-tile triangle (16 Q walkers x PW P walkers, Q walker > P walker), the V phase
// computes, for Q points q (alpha channels x) and P points p (all channels y),
//   V(q x, p y) = sum_a Phi_v(q, x, a) conj Phi_v(p, y, a)          (greens.cpp:73-79)
// with Phi_v already carrying sqrt(exp(-eps_a tau)) and the walker weights (mo_kernel). As real
// GEMMs over K' = [re | im] (K' = 2 KH, KH = n_vir rounded up to 16):
//   Re V = [re_q | im_q] . [re_p | im_p],   Im V = [im_q | -re_q] . [re_p | im_p],
// so the A operand (Q side) has 128 rows per tile: (q walker 16, e_q 2, x_alpha 2, re/im 2),
// and B (P side) 8 PW rows: (p walker PW, e_p 2, y 4); PW = 10 (N = 80) for the literal
// estimator, PW = 8 (N = 64, pair_kr's own 16 x 8 tiles) for the physical one.
//
// Ozaki splitting: every row (point, channel) is scaled by a power of two 2^e (|x| 2^-e < 127.5 / 128)
// and cut into six int8 slices of balanced radix-256 digits, x 2^-e = sum_s d_s 2^-(7 + 8 s),
// d_s in [-128, 127] (digits4). The 21 slice products with s + t <= 5 are exact int8 x int8 -> int32
// UMMA products; those of one diagonal d = s + t accumulate in one TMEM accumulator
// (|acc| <= 6 K' 2^14 < 2^31). The epilogue merges the accumulators into one int64 per element,
// X = sum_{d <= 4} acc_d 256^(4-d) + rint(acc_5 / 256) (|X| < 2^56; all six would not fit 63
// bits) and rounds once to FP64: V = X 2^(e_q + e_p - 46). The error (slice remainders <= 2^-48
// and the dropped products s + t > 5) is ~2^-46 of |row_q| |row_p| sqrt(K') -- 16x below the
// rounded 7-bit digits of round 1 at the same 21 products, pinned on the oracle by
// tests/test_ozaki_budget.py.
//
// Kernels per step (after mo_kernel):
//  * oz_slice_kernel: one warp per (point, channel): the row exponent, the seven slices of the
//    [re | im] rows (K' in energy order, 16 spinors per k-step), written directly in the UMMA
//    canonical K-major layout of their tile blocks; per point pair the last k-step with a nonzero
//    digit. On the literal path it runs on a side stream beside the O pass;
//  * literal estimator: pair_kr_kernel<false, 2> writes the o blocks of its 16 x 8 tiles, then
//    oz_vgemm_kernel<true> computes each 16 x 10 tile's V blocks and contracts them with the o
//    blocks in its epilogue (the reference's literal pair term), with the step's fixed-order sums;
//  * physical estimator: oz_vgemm_kernel<false> writes V tiles
//    V[t][q 16][p 8][re/im][e_q x_alpha e_p y>>1 (16)][y&1] in the order pair_kr's trace
//    epilogue lanes read them, then pair_kr_kernel<true, 1>.
// oz_vgemm_kernel: persistent CTAs over the tile triangle; a producer thread streams each active
// k-step's 6 A + 6 B slices into a 3-stage mbarrier ring with cp.async.bulk (and the tile's o
// values into a double buffer), one thread issues the k-step's 21 slice products as 9 merged
// tcgen05.mma (oz_issue_diagonals), eight epilogue warps (two per TMEM lane quarter) drain TMEM
// (tcgen05.ld), merge, release the accumulators and finish the tile while the next one runs.
// Measured (cfg4, profiles/r11, r16): 1.11 ms at 2960 int8 TOPS on the full K' loop (0.65 of the
// dense tcgen05 rate; the bound is shared-memory bandwidth, see oz_issue_diagonals), 0.98 ms on
// the chain's tau draws with the empty k-steps skipped, 0.95 ms with the leading zero slices of
// the partly empty k-steps skipped as well (OzParams::lz, oz_issue_partial), vs ~3.6 ms for the
// DMMA V phase of pair_kr.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "pair_common.cuh"

#ifdef OZ_OVERLAP_TL
OVERLAP_TL_DEFINE(g_tl_slice, mcmp2dev_debug_tl_slice)
#endif

namespace mcmp2dev {

namespace {
using namespace pairk;

constexpr int S = OZ_SLICES;        // slices per operand in the main pass (products s + t <= 5)
constexpr int SL = S + 1;           // slices stored per operand: the 7th feeds the refinement pass
constexpr int MA = 128;             // A rows (Q side) of a tile: 16 walkers
constexpr int A_KS = S * MA * 32;   // bytes of one k-step (32 of K') of a Q block's main slices
constexpr int A_KSM = SL * MA * 32; // stored bytes of one k-step of a Q block (the main slices first)
#ifndef OZ_STAGES
#define OZ_STAGES 5
#endif
constexpr int STAGES = OZ_STAGES;
#ifndef OZ_EPW
#define OZ_EPW 8
#endif
// epilogue warps: EPW / 4 per TMEM lane quarter (warp w reads lanes 32 (w % 4) ..), each with
// NB / (EPW / 4) accumulator columns; then the producer warp and the MMA warp
constexpr int EPW = OZ_EPW;
constexpr int THREADS = (EPW + 2) * 32;
constexpr int TMEM_COLS = 512;      // 6 x NB used
constexpr int KA_MAX = 1024, KB_MAX = 2048;  // Q / P blocks with per-block k-step counts in shared memory
// B rows (P side) per tile: 8 walkers (64 rows, the V tiles of the physical path follow
// pair_kr's 16 x 8 tiles) or 10 walkers (80 rows, the fused literal path: a kind::i8 M128 MMA
// costs the same ~61 cycles for N = 32..80 (tools/umma_rate.cu), so N = 80 -- the widest that
// fits six accumulators in 512 TMEM columns -- does 25% more work per instruction)
// CORR: the refinement pass (all SL slices per k-step, one accumulator per P block) on tiles of
// PB P blocks, so each k-step's A slices serve PB blocks (the pass is bound by the L2 -> SMEM
// operand stream)
#ifndef OZ_REFINE_PB
#define OZ_REFINE_PB 3
#endif
// instruction descriptor: s32 accumulator, s8 x s8, both K-major, M = 128, N columns
__host__ __device__ constexpr uint32_t oz_idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
template <bool FUSED, bool CORR = false>
struct OzShape {
  static constexpr int NB = FUSED ? 80 : 64;
  static constexpr int PW = NB / 8;  // P walkers per P block
  static constexpr int PB = CORR ? OZ_REFINE_PB : 1;  // P blocks per tile
  static constexpr int B_KSM = SL * NB * 32;  // stored bytes of one k-step of a P block
  static constexpr int NSL = CORR ? SL : S;   // slices copied per k-step
  static constexpr int A_CP = NSL * MA * 32, B_CP = NSL * NB * 32;
  static constexpr int STAGE = A_CP + PB * B_CP;
  // main fused pass: the tile's o values (16 x PW walker pairs x 32 doubles, one bulk copy from
  // the O pass's [Q block row][p walker][q][x_alpha][re/im][e_p][y] layout) double-buffered in
  // shared memory next to a 3-stage ring (3 / 4 / 5 stages measured alike), so the epilogue never
  // waits on HBM for them
  static constexpr int OT_BYTES = FUSED && !CORR ? PW * 16 * 32 * 8 : 0;
  // ... followed by the P block's NB row-scale exponents (sb_exp)
  static constexpr int OT_BUF = OT_BYTES ? OT_BYTES + (NB * 4 + 127) / 128 * 128 : 0;
  static constexpr int NSTAGE = CORR ? (227 * 1024 - 16 * 1024) / STAGE : FUSED ? 3 : STAGES;
  static constexpr int SMEM_BYTES = NSTAGE * STAGE + 2 * OT_BUF;
  static constexpr int NACC = CORR ? 1 : S;   // accumulators per P block (slice diagonals)
  static constexpr int NSLOT = CORR ? 512 / (PB * NB) : 1;  // tiles in flight in TMEM
  static constexpr int CPW = NB / (EPW / 4);  // columns per epilogue warp
  static constexpr uint32_t IDESC = oz_idesc(NB);
};
static_assert(OzShape<true>::SMEM_BYTES <= 227 * 1024, "stage ring");
static_assert(OzShape<true, true>::SMEM_BYTES <= 227 * 1024, "stage ring");
static_assert(OzShape<true>::NACC * OzShape<true>::NB <= 512 && OzShape<true, true>::NSLOT >= 2 &&
                  OzShape<true, true>::NSTAGE >= 2,
              "TMEM columns / stage ring");

// canonical K-major, no-swizzle UMMA operand layout of one k-step: [row / 8][k / 16][row % 8][16 B]
__host__ __device__ __forceinline__ int op_off(int r, int kk) {
  return ((r >> 3) * 2 + (kk >> 4)) * 128 + (r & 7) * 16 + (kk & 15);
}
__device__ __forceinline__ uint64_t umma_desc(const void* p) {  // LBO 128 B (k chunk), SBO 256 B (8 rows)
  return uint64_t((smem_u32(p) >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
         (uint64_t(1) << 46);
}
template <uint32_t IDESC>
__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void umma_i8_rt(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(addr));
}

// One k-step's slice products of the main pass. A slice s meets B slices t = 0 .. S-1-s, and the
// product (s, t) belongs to the accumulator of diagonal s + t at TMEM columns (s + t) NB. The B
// slices of a stage are consecutive in shared memory ([slice][NB rows x 32], every slice whole
// 8-row groups of the canonical layout) and so are the accumulators in TMEM, so A_s x [B_0; ..;
// B_{S-1-s}] is ONE GEMM of N = NB (S - s) columns landing on diagonals s .. S-1 -- issued as one
// MMA, or two halves when N > 256: 9 MMAs per k-step instead of 21 for the same products. The
// kernel is bound by shared-memory operand reads (an SS-mode MMA reads 128 x 32 B of A and
// N x 32 B of B; 21 N = 80 MMAs read 136 KB per k-step, next to the 39 KB the ring's fills write,
// against 128 B/clk); the merged MMAs read each A slice once or twice instead of 6 - s times
// (88 KB per k-step) and run at the dense rate (N >= 160 is compute-bound).
// The first write of every diagonal is by A slice 0 (acc0 = 0 on k-step 0), the others accumulate.
template <int NB, int s>
__device__ __forceinline__ void oz_issue_diagonals(uint32_t tmem, const int8_t* sa, const int8_t* sb, uint32_t acc0) {
  if constexpr (s < S) {
    constexpr int TOT = NB * (S - s);
    constexpr int N0 = TOT > 256 ? (TOT / 2 + 15) / 16 * 16 : TOT, N1 = TOT - N0;
    static_assert(N0 % 16 == 0 && N0 <= 256 && N1 % 16 == 0 && N1 <= 256, "MMA N");
    const uint64_t da = umma_desc(sa + s * MA * 32);
    const uint32_t acc = s == 0 ? acc0 : 1u;
    umma_i8<oz_idesc(N0)>(tmem + uint32_t(s * NB), da, umma_desc(sb), acc);
    if constexpr (N1 > 0) umma_i8<oz_idesc(N1)>(tmem + uint32_t(s * NB + N0), da, umma_desc(sb + N0 * 32), acc);
    oz_issue_diagonals<NB, s + 1>(tmem, sa, sb, acc0);
  }
}

// A k-step whose A slices below a0 and B slices below b0 are all zero (OzParams::lz, a0 + b0 < S):
// the products (s, t) with s >= a0, t >= b0, s + t <= S - 1 as merged MMAs -- A slice s against
// the consecutive B slices b0 .. S-1-s, landing on diagonals s + b0 .. S-1; the skipped products
// are exact zeros. Never the tile's first k-step (every diagonal is first written there).
template <int NB>
__device__ __forceinline__ void oz_issue_partial(uint32_t tmem, const int8_t* sa, const int8_t* sb, int a0, int b0) {
  const uint64_t db = umma_desc(sb + b0 * NB * 32);
  for (int s = a0; s + b0 < S; ++s) {
    const int tot = NB * (S - s - b0);
    const int n0 = tot > 256 ? (tot / 2 + 15) / 16 * 16 : tot, n1 = tot - n0;
    const uint64_t da = umma_desc(sa + s * MA * 32);
    const uint32_t d = tmem + uint32_t((s + b0) * NB);
    umma_i8_rt(d, da, db, oz_idesc(n0), 1u);
    if (n1 > 0) umma_i8_rt(d + uint32_t(n0), da, umma_desc(sb + (b0 * NB + n0) * 32), oz_idesc(n1), 1u);
  }
}
// slice products of such a k-step (21 for a full one)
__device__ __forceinline__ int oz_products(int a0, int b0) {
  const int n = S - a0 - b0;
  return n > 0 ? n * (n + 1) / 2 : 0;
}

// the tile triangle, row by row: Q block a (walkers 16a ..) holds P blocks b < ceil(16 (a+1) / pw)
// (walkers pw b ..); a CTA walks tiles t0, t0 + stride, ... (for pw = 8, t = a (a + 1) + b is
// pair_kr's tile numbering)
struct OzWalk {
  int a = 0, b, pw;
  __device__ OzWalk(int t0, int pw_) : b(t0), pw(pw_) { settle(); }
  __device__ int len() const { return (16 * (a + 1) + pw - 1) / pw; }
  __device__ void settle() {
    while (b >= len()) b -= len(), ++a;
  }
  __device__ void next(int stride) { b += stride, settle(); }
};
int oz_tiles(int nbq, int pw) {
  int n = 0;
  for (int a = 0; a < nbq; ++a) n += (16 * (a + 1) + pw - 1) / pw;
  return n;
}
// the same triangle in tiles of pb consecutive P blocks (the refinement pass): row a holds
// ceil(len / pb) of them; a tile's P blocks past the row are skipped
struct OzGroupWalk {
  int a = 0, g, pw, pb;
  int rs = 0;  // tile index (pb = 1 numbering) of row a's first P block
  __device__ OzGroupWalk(int t0, int pw_, int pb_) : g(t0), pw(pw_), pb(pb_) { settle(); }
  __device__ int row_blocks() const { return (16 * (a + 1) + pw - 1) / pw; }
  __device__ int len() const { return (row_blocks() + pb - 1) / pb; }
  __device__ void settle() {
    while (g >= len()) g -= len(), rs += row_blocks(), ++a;
  }
  __device__ void next(int stride) { g += stride, settle(); }
};
// the refinement pass's choice for the tile group at w: the main pass's estimates of its P blocks
// against the thresholds the main pass's last CTA set (each at most 1 / groups of the step's
// budget, so the groups left unrefined carry at most the budget between them)
__device__ __forceinline__ bool oz_refine_group(const OzParams& P, const OzGroupWalk& w) {
  const int b0 = w.g * w.pb, nb = min(w.pb, w.row_blocks() - b0);
  double ed = 0.0, ex = 0.0;
  for (int j = 0; j < nb; ++j) {
    const double2 e = reinterpret_cast<const double2*>(P.tile_eps)[w.rs + b0 + j];
    ed += e.x, ex += e.y;
  }
  const volatile double* thr = P.st->oz_thr;
  return ed > thr[0] || ex > thr[1] || ed + ex > thr[2];
}
__device__ int oz_group_tiles_dev(int nbq, int pw, int pb) {
  int n = 0;
  for (int a = 0; a < nbq; ++a) n += ((16 * (a + 1) + pw - 1) / pw + pb - 1) / pb;
  return n;
}
int oz_group_tiles(int nbq, int pw, int pb) {
  int n = 0;
  for (int a = 0; a < nbq; ++a) n += ((16 * (a + 1) + pw - 1) / pw + pb - 1) / pb;
  return n;
}

// SL balanced radix-256 digits of 4 values, |x| < 127.5 / 128 (the row scale guarantees it):
//   x = d_0 2^-7 + sum_{s >= 1} d_s 2^-(7 + 8 s) + rem,  d_s in [-128, 127] (d_0 in [-127, 127]),
// read off the integer X = rint(x 2^(7 + 8 (SL - 1))) from the low end: d = the signed low byte,
// X <- (X - d) / 256. The first S digits are then the S-slice representation rounded to nearest
// (|rem| <= 2^-(8 + 8 (S - 1))), one bit per slice more than rounded 7-bit digits in the same
// int8 operands: the six-slice sums are ~16x closer to FP64 at the same 21 products
// (tests/test_ozaki_budget.py). One FP64 multiply and one conversion per value, the rest
// integer work. A balanced digit -128 has no negative, so the negated rows of the A operand
// take the digits of -x (neg = true), not negated digits.
__device__ __forceinline__ void digits4(const double (&x)[4], uint32_t (&out)[SL], bool neg = false) {
  constexpr double kScale = double(1ull << (7 + 8 * (SL - 1)));
  long long X[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    X[i] = __double2ll_rn(x[i] * kScale);
    if (neg) X[i] = -X[i];
  }
#pragma unroll
  for (int s = SL - 1; s >= 0; --s) {
    const uint32_t b0 = uint32_t(X[0]), b1 = uint32_t(X[1]), b2 = uint32_t(X[2]), b3 = uint32_t(X[3]);
    out[s] = __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
    if (s > 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) X[i] = (X[i] + 128) >> 8;
    }
  }
}

// HELD: n_vir <= 384 (at most 3 quads per lane): one load pass, the values held in registers
// across the row-maximum reduction (3x the loads in flight); otherwise two passes (max, digits).
// With P.pstat (the accuracy guard of the literal path) each warp also reduces its scaled row's
// sum of squares and count of digits-relevant entries (|x| 2^-e > 2^-8) and its channel's share
// of |Phi_o(pt)|^2; the first warp of each point combines the four channels into the point's
// stats S, A, N (oz_vgemm_kernel's error model, see there).
#ifndef OZ_SLICE_MINB
#define OZ_SLICE_MINB 3
#endif
template <bool HELD>
__global__ void __launch_bounds__(256, OZ_SLICE_MINB) oz_slice_kernel(OzParams P) {
  pdl_wait();
  pdl_trigger();
  OVERLAP_TL_BEGIN(g_tl_slice);
  __shared__ double s_st[8][3];
  __shared__ int s_k[8];
  // first main slice with a nonzero digit per k-step, over the CTA's alpha rows [0] and all of
  // its rows [1] (OzParams::lz)
  __shared__ int s_lz[2][OZ_LZ_STRIDE];
  if (P.lz) {
    if (threadIdx.x < 2 * OZ_LZ_STRIDE) (&s_lz[0][0])[threadIdx.x] = S;
    __syncthreads();
  }
  // one warp per (point, channel): 8 warps = 2 points per CTA (npts_oz is a multiple of 32, so
  // every CTA's points exist)
  const int wg = int(blockIdx.x) * 8 + (int(threadIdx.x) >> 5), lane = int(threadIdx.x) & 31;
  const int pt = wg >> 2, x = wg & 3;
  const PhiChunks ch{P.Go, P.Gv};
  const int KH = P.kh, ks_n = P.ks, nq = KH / 4;
  const bool live = pt < P.npts;
  const int swz = phi_swz(pt);
  const int qb = pt >> 5, qrow = ((pt & 31) >> 1) * 8 + (pt & 1) * 4;  // A row of (x_alpha 0, re)
  const int NB = P.nb_rows, bpts = NB / 4;  // B rows and points per P block
  const int pb = pt / bpts, prow = ((pt % bpts) >> 1) * 8 + (pt & 1) * 4;  // B row of channel 0
  int8_t* const sa = P.sa + size_t(qb) * ks_n * A_KSM;
  int8_t* const sb = P.sb + size_t(pb) * ks_n * SL * NB * 32;
  const bool stats = P.pstat != nullptr;
  double ss = 0.0, nbig = 0.0, n2 = 0.0, row_scale = 1.0;
  int kact = 0;  // k-steps up to this lane's last nonzero digit
  {
    // this lane's spinor quads a0 = 4 (lane + 32 j); two passes over them (the row maximum, then
    // the digits), the second from L1, so no values are held across the reduction
    auto load = [&](int qd, double (&re)[4], double (&im)[4]) {
#pragma unroll
      for (int i = 0; i < 4; ++i) re[i] = im[i] = 0.0;
      if (live && 4 * qd < P.n_vir) {
        const double* src = P.phi + ch.offset(P.Go + qd, pt, P.npts_pad);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (4 * qd + i < P.n_vir) {
            re[i] = src[(x * 4 + i) ^ swz];
            im[i] = src[16 + ((x * 4 + i) ^ swz)];
          }
      }
    };
    double mx = 0.0;
    constexpr int MAXJ = HELD ? 3 : 1;
    double hr[MAXJ][4], hi[MAXJ][4];
    if constexpr (HELD) {
#pragma unroll
      for (int j = 0; j < MAXJ; ++j) load(lane + 32 * j < nq ? lane + 32 * j : nq, hr[j], hi[j]);
    }
    // the guard's N stat: this channel's share of |Phi_o(pt)|_F^2 (occupied groups; spinors past
    // n_occ skipped), read here so its latency runs beside the virtual rows'
    if (stats && live)
      for (int g = lane; g < P.Go; g += 32) {
        const double* src = P.phi + ch.offset(g, pt, P.npts_pad);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (4 * g + i < P.n_occ) {
            const double re = src[(x * 4 + i) ^ swz], im = src[16 + ((x * 4 + i) ^ swz)];
            n2 += re * re + im * im;
          }
      }
    if constexpr (HELD) {
#pragma unroll
      for (int j = 0; j < MAXJ; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) mx = fmax(mx, fmax(fabs(hr[j][i]), fabs(hi[j][i])));
    } else {
      for (int qd = lane; qd < nq; qd += 32) {
        double re[4], im[4];
        load(qd, re, im);
#pragma unroll
        for (int i = 0; i < 4; ++i) mx = fmax(mx, fmax(fabs(re[i]), fabs(im[i])));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    // |value| 2^-e < 127.5 / 128: the leading balanced digit fits an int8
    int e = (mx > 0.0 && mx <= 1.7e308) ? ilogb(mx) + 1 : 0;
    if (mx * ldexp(1.0, -e) > 0.995) ++e;
    const double sc = ldexp(1.0, -e);
    row_scale = ldexp(1.0, e);
    const bool alpha = (x & 1) == 0;
    const int ra = qrow + (x >> 1) * 2;  // A rows ra (re variant), ra + 1 (im variant)
    const int rb = prow + x;
    if (lane == 0) {
      P.sb_scale[size_t(pb) * NB + rb] = ldexp(1.0, e);
      P.sb_exp[size_t(pb) * NB + rb] = e * (1 << 20);
      if (alpha) P.sa_scale[size_t(qb) * MA + ra] = P.sa_scale[size_t(qb) * MA + ra + 1] = ldexp(1.0, e - 46);
    }
    auto emit = [&](int qd, double (&xr)[4], double (&xi)[4]) {
#pragma unroll
      for (int i = 0; i < 4; ++i) xr[i] *= sc, xi[i] *= sc;
      if (stats) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          ss += xr[i] * xr[i] + xi[i] * xi[i];
          nbig += (fabs(xr[i]) > 0x1p-8 ? 1.0 : 0.0) + (fabs(xi[i]) > 0x1p-8 ? 1.0 : 0.0);
        }
      }
      uint32_t dr[SL], di[SL], drn[SL];
      digits4(xr, dr);
      digits4(xi, di);
      if (alpha) digits4(xr, drn, true);
      // K' positions: k-step qd / 4 holds spinors 16 (qd / 4) .. + 15 as [re (16) | im (16)], so
      // K' follows the virtual energies (ascending, model.cpp:126-127) and the spinors that
      // exp(-eps tau / 2) has pushed below the last slice fill the trailing k-steps with zeros
      const int kre = (qd >> 2) * 32 + (qd & 3) * 4, kim = kre + 16;
      {
        uint32_t any = 0;
#pragma unroll
        for (int s = 0; s < SL; ++s) any |= dr[s] | di[s];
        if (any) kact = max(kact, (qd >> 2) + 1);
      }
      if (P.lz) {
        int fb = S, fa = S;
#pragma unroll
        for (int s = S - 1; s >= 0; --s) {
          if (dr[s] | di[s]) fb = s;
          if (alpha && (dr[s] | di[s] | drn[s])) fa = s;
        }
        if (fb < S) atomicMin(&s_lz[1][qd >> 2], fb);
        if (fa < S) atomicMin(&s_lz[0][qd >> 2], fa);
      }
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        // B row [re | im]
        *reinterpret_cast<uint32_t*>(sb + (size_t(kre >> 5) * SL + s) * NB * 32 + op_off(rb, kre & 31)) = dr[s];
        *reinterpret_cast<uint32_t*>(sb + (size_t(kim >> 5) * SL + s) * NB * 32 + op_off(rb, kim & 31)) = di[s];
        if (alpha) {  // A rows [re | im] and [im | -re]
          int8_t* a0 = sa + (size_t(kre >> 5) * SL + s) * MA * 32;
          int8_t* a1 = sa + (size_t(kim >> 5) * SL + s) * MA * 32;
          *reinterpret_cast<uint32_t*>(a0 + op_off(ra, kre & 31)) = dr[s];
          *reinterpret_cast<uint32_t*>(a1 + op_off(ra, kim & 31)) = di[s];
          *reinterpret_cast<uint32_t*>(a0 + op_off(ra + 1, kre & 31)) = di[s];
          *reinterpret_cast<uint32_t*>(a1 + op_off(ra + 1, kim & 31)) = drn[s];
        }
      }
    };
    if constexpr (HELD) {
#pragma unroll
      for (int j = 0; j < MAXJ; ++j)
        if (lane + 32 * j < nq) emit(lane + 32 * j, hr[j], hi[j]);
    } else {
      for (int qd = lane; qd < nq; qd += 32) {
        double xr[4], xi[4];
        load(qd, xr, xi);
        emit(qd, xr, xi);
      }
    }
  }
  if (P.ks_cnt) {  // the CTA's point pair: k-steps up to the last nonzero digit of its 8 rows
    kact = __reduce_max_sync(0xffffffffu, kact);
    if (lane == 0) s_k[int(threadIdx.x) >> 5] = kact;
    __syncthreads();
    if (threadIdx.x == 0) {
      int k = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) k = max(k, s_k[w]);
      P.ks_cnt[blockIdx.x] = uint8_t(k);
    }
    if (P.lz && threadIdx.x < OZ_LZ_STRIDE)  // (the barrier above follows every lane's atomicMin)
      P.lz[size_t(blockIdx.x) * OZ_LZ_STRIDE + threadIdx.x] = uint8_t(s_lz[1][threadIdx.x] | (s_lz[0][threadIdx.x] << 4));
  }
  OVERLAP_TL_END(g_tl_slice);
  if (!stats) return;  // uniform over the grid
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    nbig += __shfl_xor_sync(0xffffffffu, nbig, o);
    n2 += __shfl_xor_sync(0xffffffffu, n2, o);
  }
  const int w = int(threadIdx.x) >> 5;
  if (lane == 0) {
    s_st[w][0] = row_scale;
    s_st[w][1] = row_scale * sqrt(ss * (1.0 / 3.0) + 0.6 * nbig);
    s_st[w][2] = n2;
  }
  __syncthreads();
  if (lane == 0 && x == 0) {
    double Sx = 0.0, Ax = 0.0, N2 = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      Sx = fmax(Sx, s_st[w + c][0]);
      Ax = fmax(Ax, s_st[w + c][1]);
      N2 += s_st[w + c][2];
    }
    reinterpret_cast<float4*>(P.pstat)[pt] = make_float4(float(Sx), float(Ax), float(sqrt(N2)), 0.0f);
  }
}

// CORR (FUSED only): the guard's refinement pass. A step whose error estimate failed in the main
// pass (st->oz_trip == 1) gets the next slice diagonal, d = s + t = 6 (seven products per k-step,
// the 7th slices included), in one int32 accumulator per tile: dV = acc 2^(e_q + e_p - 62). The
// main pass stored each pair's f values (P.fstore); this pass adds df = sum o dV, re-forms the
// pair terms from f + df and the step's sums, and re-checks them with the estimate scaled by
// 2^-7; a step that still fails goes on to the DMMA kernel (oz_trip = 2). The accumulator is
// small, so six tiles rotate through TMEM and the drain never stalls the MMAs.
#ifdef OZ_TIMELINE
// debug build (tools/oz_timeline.py): clock64 stamps per CTA and tile -- MMA thread: wait for the
// accumulators, accumulators acquired, last commit issued; each epilogue warp: accumulators full,
// released, tile finished
constexpr int TL_TILES = 128;
__device__ unsigned long long g_oz_tl[160][TL_TILES][3 + 3 * EPW];
#define TL(t, k, v) \
  if ((t) < TL_TILES) g_oz_tl[blockIdx.x][t][k] = (v)
#else
#define TL(t, k, v)
#endif

// the CTA's estimate of one main-pass tile: the epilogue warps' sums in fixed order
__device__ __forceinline__ void oz_store_tile_eps(const OzParams& P, const double2* te, int t) {
  double e0 = 0.0, e1 = 0.0;
  for (int w = 0; w < EPW; ++w) e0 += te[w].x, e1 += te[w].y;
  reinterpret_cast<double2*>(P.tile_eps)[t] = make_double2(e0, e1);
}

template <bool FUSED, bool CORR>
__global__ void __launch_bounds__(THREADS, 1) oz_vgemm_kernel(OzParams P) {
  using Sh = OzShape<FUSED, CORR>;
  constexpr int NB = Sh::NB, PW = Sh::PW, STAGE = Sh::STAGE, CPW = Sh::CPW;
  constexpr int A_CP = Sh::A_CP, B_CP = Sh::B_CP, B_KSM = Sh::B_KSM, NST = Sh::NSTAGE;
  constexpr int NACC = Sh::NACC, NSLOT = Sh::NSLOT, PB = Sh::PB;
  static_assert(!CORR || FUSED, "the refinement pass serves the fused literal path");
  pdl_wait();
  pdl_trigger();
  if constexpr (CORR)  // nothing to refine unless the main pass rejected this step
    if (*reinterpret_cast<volatile const int*>(&P.st->oz_trip) != 1) return;
  extern __shared__ __align__(1024) int8_t sm[];
  // Measured and rejected: eight rotating 64-column accumulator slots (tile i's diagonal d in slot
  // (6 i + d) % 8, drained and freed diagonal by diagonal so the next tile starts early): V-GEMM
  // 1.733 vs 1.571 ms on the same box; the next tile's k-step 0 waits on the drain diagonal by
  // diagonal anyway, and TMEM reads under running MMAs are slower. Also rejected: A from TMEM
  // (tcgen05.cp 128x256b per slice and k-step, MMA with [a_tmem]): exact, but 1.89 vs 1.59 ms
  // (tools/oz_gemm.cu -DA_TMEM). At N = 80 (same-box A/B, V-GEMM ms): 3 / 4 / 5 ring stages
  // 1.333 / 1.335 / 1.335; 4 epilogue warps 1.482 vs 8 warps 1.335 (the drain is the epilogue
  // warps' instruction latency while the MMA waits for TMEM). Round 2: a diagonal-major drain
  // releasing each diagonal at once, with the next tile's first k-step issued diagonal by
  // diagonal, 1.475 vs 1.35 ms (tile period 30.5k vs 28.75k cycles: TMEM reads under the
  // restarted MMAs slow both).
  __shared__ __align__(8) uint64_t full[NST], empty[NST], tfull[NSLOT], tempty[NSLOT], ofull[2], oempty[2];
  constexpr bool OSM = Sh::OT_BYTES > 0;  // o values through shared memory
  __shared__ uint32_t tmem_base;
  __shared__ double s_red[EPW][6];
  __shared__ bool s_last;
  // FUSED: the f values of the last two tiles, [q 16][p PW] each (written before, read after the
  // epilogue warps' named barrier; two buffers so one barrier per tile suffices)
  __shared__ __align__(32) double4 s_f[2][FUSED ? 16 * PW : 1];
  // main pass with a refinement pass behind it: each epilogue warp's estimate of the last two tiles
  __shared__ double2 s_te[2][EPW];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KS = P.ks;
  // active k-steps of each Q block (32 points) and P block (NB / 4 points) from the slice
  // kernel's per-point-pair records: a tile runs min(Q block's, P blocks') k-steps (at least one)
  __shared__ uint8_t s_ka[KA_MAX], s_kb[KB_MAX];
  const int nqa = P.npts_oz / 32, npb = (P.npts_oz + NB / 4 - 1) / (NB / 4);
  const bool trunc = P.ks_cnt != nullptr && nqa <= KA_MAX && npb <= KB_MAX;
  if (trunc) {
    const int ncnt = P.npts_oz / 2;
    for (int i = tid; i < nqa; i += THREADS) {
      const uint4 v = *reinterpret_cast<const uint4*>(P.ks_cnt + 16 * i);
      uint32_t mx = __vmaxu4(__vmaxu4(v.x, v.y), __vmaxu4(v.z, v.w));
      mx = __vmaxu4(mx, mx >> 16);
      s_ka[i] = uint8_t(max(mx & 0xFFu, (mx >> 8) & 0xFFu));
    }
    constexpr int BC = NB / 8;  // records per P block
    for (int i = tid; i < npb; i += THREADS) {
      int mx = 0;
      for (int j = 0; j < BC; ++j)
        if (BC * i + j < ncnt) mx = max(mx, int(P.ks_cnt[BC * i + j]));
      s_kb[i] = uint8_t(mx);
    }
  }
  // main pass: the tile's k-step plan from the slice kernel's leading-zero records (OzParams::lz),
  // written by the producer warp (lane = k-step) before the tile's first copy and read by the
  // producer and MMA threads: a0 | b0 << 4 (issue the products s >= a0, t >= b0; copy only those
  // slices), or PLAN_SKIP when a0 + b0 >= S (every product of the k-step has a zero factor).
  // k-step 0 is always whole: it is every diagonal's first write. The producer is at most NST
  // stages, so at most NST + 1 tiles, ahead of the MMA thread: 8 plans rotate.
  constexpr int NPLAN = 8;
  constexpr uint8_t PLAN_SKIP = 0xFF;
  __shared__ uint8_t s_plan[NPLAN][OZ_LZ_STRIDE];
  const bool use_plan = !CORR && trunc && P.lz != nullptr && KS <= OZ_LZ_STRIDE;
  auto tile_ks = [&](int a, int b0, int nb) {
    if (!trunc) return KS;
    int kb = 0;
    for (int j = 0; j < nb; ++j) kb = max(kb, int(s_kb[b0 + j]));
    return max(1, min(min(int(s_ka[a]), kb), KS));
  };
  double acc_d = 0.0, acc_x = 0.0;  // FUSED: this thread's pair sums
  // FUSED, guard: sums of the squared per-pair error estimates and of |pair term|
  // (the estimates in FP32, in units of the model constant 2^-46: FP32 work costs nothing beside
  // the MMAs, FP64 instructions ~12x their usual time)
  float acc_ed = 0.0f, acc_ex = 0.0f;
  double acc_ad = 0.0, acc_ax = 0.0;
  constexpr double kSig2 = 0x1p-92;  // (2^-46)^2: the estimates' unit, applied with the CTA sums
  const bool guard = FUSED && P.pstat != nullptr;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int s = 0; s < NSLOT; ++s) mbar_init(&tfull[s], 1), mbar_init(&tempty[s], 32 * EPW);
    for (int s = 0; s < 2; ++s) mbar_init(&ofull[s], 1), mbar_init(&oempty[s], EPW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const int ntiles = CORR ? oz_group_tiles_dev(P.npts_oz / 32, PW, PB) : P.ntiles;
  const int my = int(blockIdx.x) < ntiles ? (ntiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;

  if (warp == EPW) {
    {  // producer (lane 0; the other lanes help with the tile's plan): one k-step of the tile's A and B slices per stage
      int stage = 0;
      uint32_t ph = 0;
      unsigned long long issued = 0;  // slice products of this CTA's tiles
      OzGroupWalk w(int(blockIdx.x), PW, PB);
      for (int it = 0; it < my; ++it, w.next(int(gridDim.x))) {
        if constexpr (CORR)
          if (P.tile_eps && !oz_refine_group(P, w)) continue;
        const int a = w.a, b0 = w.g * PB, nb = min(PB, w.row_blocks() - b0);
        const int8_t* ga = P.sa + size_t(a) * KS * A_KSM;
        const int8_t* gb = P.sb + size_t(b0) * KS * B_KSM;
        const int nk = tile_ks(a, b0, nb);
        if (use_plan) {  // lane = k-step: leading zero slices of the Q block's A rows and the P block's B rows
          uint8_t pl = 0;
          if (lane > 0 && lane < nk) {
            constexpr int BC = NB / 8;  // records per P block
            const int ncnt = P.npts_oz / 2;
            int la = S, lb = S;
            for (int i = 0; i < 16; ++i) la = min(la, int(P.lz[size_t(16 * a + i) * OZ_LZ_STRIDE + lane] >> 4));
            for (int j = 0; j < BC; ++j)
              if (BC * b0 + j < ncnt) lb = min(lb, int(P.lz[size_t(BC * b0 + j) * OZ_LZ_STRIDE + lane] & 15));
            pl = la + lb >= S ? PLAN_SKIP : uint8_t(la | (lb << 4));
          }
          s_plan[it % NPLAN][lane] = pl;
          __syncwarp();
        }
        if (lane != 0) continue;
        if constexpr (OSM) {  // the tile's o values: walkers PW b0 .. of Q block row a (up to the diagonal)
          const int ob = it & 1, np = min(PW, 16 * (a + 1) - PW * b0);
          mbar_wait(&oempty[ob], ((it >> 1) & 1) ^ 1u);
          mbar_expect_tx(&ofull[ob], np * 4096 + NB * 4);
          bulk_g2s(sm + NST * STAGE + ob * Sh::OT_BUF, P.otiles + size_t(a) * (a + 1) * 4096 + size_t(PW * b0) * 512,
                   np * 4096, &ofull[ob]);
          bulk_g2s(sm + NST * STAGE + ob * Sh::OT_BUF + Sh::OT_BYTES, P.sb_exp + size_t(b0) * NB, NB * 4, &ofull[ob]);
        }
        for (int ks = 0; ks < nk; ++ks) {
          int a0 = 0, sb0 = 0;
          if (use_plan) {
            const uint8_t pl = s_plan[it % NPLAN][ks];
            if (pl == PLAN_SKIP) continue;
            a0 = pl & 15, sb0 = pl >> 4;
          }
          if constexpr (!CORR) issued += oz_products(a0, sb0);
          mbar_wait(&empty[stage], ph ^ 1u);
          int8_t* dst = sm + stage * STAGE;
          if (a0 | sb0) {  // A slices a0 .. S-1-sb0 and B slices sb0 .. S-1-a0 take part
            const int ns = S - a0 - sb0;
            mbar_expect_tx(&full[stage], ns * (MA * 32 + NB * 32));
            bulk_g2s(dst + a0 * MA * 32, ga + size_t(ks) * A_KSM + a0 * MA * 32, ns * MA * 32, &full[stage]);
            bulk_g2s(dst + A_CP + sb0 * NB * 32, gb + size_t(ks) * B_KSM + sb0 * NB * 32, ns * NB * 32, &full[stage]);
          } else {
            mbar_expect_tx(&full[stage], A_CP + nb * B_CP);
            bulk_g2s(dst, ga + size_t(ks) * A_KSM, A_CP, &full[stage]);
            for (int j = 0; j < nb; ++j)
              bulk_g2s(dst + A_CP + j * B_CP, gb + (size_t(j) * KS + ks) * B_KSM, B_CP, &full[stage]);
          }
          if (++stage == NST) stage = 0, ph ^= 1u;
        }
      }
      if constexpr (!CORR)
        if (lane == 0 && P.ks_exec) atomicAdd(P.ks_exec, issued);
    }
  } else if (warp == EPW + 1) {
    if (lane == 0) {  // MMA issuer: the slice products of each k-step into the tile's accumulators
      int stage = 0, u = 0;  // u: tiles through TMEM (the refinement pass skips unrefined groups)
      uint32_t ph = 0;
      OzGroupWalk w(int(blockIdx.x), PW, PB);
      for (int it = 0; it < my; ++it, w.next(int(gridDim.x))) {
        if constexpr (CORR)
          if (P.tile_eps && !oz_refine_group(P, w)) continue;
        const int slot = u % NSLOT;
        const int nb = min(PB, w.row_blocks() - w.g * PB);
        TL(it, 0, clock64());
        mbar_wait(&tempty[slot], ((u / NSLOT) & 1) ^ 1u);  // the epilogue has drained this slot
        asm volatile("tcgen05.fence::after_thread_sync;");
        TL(it, 1, clock64());
        const int nk = tile_ks(w.a, w.g * PB, nb);
        for (int ks = 0; ks < nk; ++ks) {
          // the plan is read behind the wait for the tile's first stage (k-step 0 is always whole),
          // which orders it after the producer's writes
          int a0 = 0, sb0 = 0;
          if (use_plan && ks > 0) {
            const uint8_t pl = *reinterpret_cast<volatile const uint8_t*>(&s_plan[it % NPLAN][ks]);
            if (pl == PLAN_SKIP) continue;
            a0 = pl & 15, sb0 = pl >> 4;
          }
          mbar_wait(&full[stage], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const int8_t* sa = sm + stage * STAGE;
          const int8_t* sb = sa + A_CP;
          if constexpr (CORR) {
            for (int j = 0; j < nb; ++j)
#pragma unroll
              for (int s = 0; s < SL; ++s)  // diagonal 6: (s, 6 - s)
                umma_i8<Sh::IDESC>(tmem + uint32_t((slot * PB + j) * NB), umma_desc(sa + s * MA * 32),
                                   umma_desc(sb + j * B_CP + (SL - 1 - s) * NB * 32), ks > 0 || s > 0 ? 1u : 0u);
          } else if (a0 | sb0) {
            oz_issue_partial<NB>(tmem, sa, sb, a0, sb0);
          } else {
            oz_issue_diagonals<NB, 0>(tmem, sa, sb, ks > 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);  // the stage is free once these MMAs have read it
          if (++stage == NST) stage = 0, ph ^= 1u;
        }
        umma_commit(&tfull[slot]);
        TL(it, 2, clock64());
        ++u;
      }
    }
  } else {  // epilogue: TMEM lane = A row; this warp's columns [c_lo, c_lo + CPW)
    const int lq = warp & 3, c_lo = (warp >> 2) * CPW;
    const int row = lq * 32 + lane;
    const int q = row >> 3, plane = row & 1, exq = (row >> 1) & 3;
    OzGroupWalk w(int(blockIdx.x), PW, PB);
    int sub = 0;  // P blocks processed: the parity of the shared f buffer
    int u = 0;    // tiles through TMEM
    float te_d = 0.0f, te_x = 0.0f;  // main pass: this thread's estimate of the current tile
    // one pair's literal term (estimator.cpp:26-32) from its f values into the thread's sums.
    // Main pass: F is stored for a refinement pass. Refinement pass: F is this pass's correction
    // to the stored f values (refined groups) or zero (groups left unrefined).
    // Accuracy guard: the INT8 error of each f is modelled per element as a random sum over K' of
    // slice remainders and dropped products, sigma(u, v) = 2^-46 (A_u S_v + S_u A_v) with the row
    // stats of oz_slice_kernel (S = max row scale 2^e of the point, A = max of 2^e sqrt(|x 2^-e|^2 /
    // 3 + 0.6 #{|x 2^-e| > 2^-8})), propagated through the contraction with |o block|_F <=
    // |Phi_o(u)|_F |Phi_o(v)|_F: eps = |w| (sigma_f1 |f2| + |f1| sigma_f2) per pair, summed in
    // quadrature over the step (the last CTA compares sqrt(sum eps^2) with guard_tol |sum|). On the
    // oracle's cfg3/cfg4 steps this estimate is 3-250x the actual error
    // (tests/test_oz_guard_model.py), on 2000-step device chains 2.3-170x (tests/test_gpu_guard.py);
    // it is a model, not a bound. Pairs of refined groups (one more slice and diagonal): 2^-49.
    // Evaluated in FP32 from float point stats (a model needs no more; sums of squares far below
    // the largest terms may flush to zero).
    const float wdf = fabsf(float(P.w_direct)), wxf = fabsf(float(P.w_exchange));
    // the four points' stats of a pair (q walker's two points, p walker's two)
    struct PairStats { float4 c, d, a, b; };
    auto load_stats = [&](int qg, int pg) {
      const float4* ps = reinterpret_cast<const float4*>(P.pstat);
      return PairStats{ps[2 * qg], ps[2 * qg + 1], ps[2 * pg], ps[2 * pg + 1]};
    };
    auto pair_term = [&](double4 F, int qg, int pg, bool refined, const PairStats& st) {
      double4* fs = P.fstore ? reinterpret_cast<double4*>(P.fstore) + (size_t(qg) * (qg - 1) / 2 + pg) : nullptr;
      if constexpr (CORR) {
        const double4 f6 = *fs;
        F.x += f6.x, F.y += f6.y, F.z += f6.z, F.w += f6.w;
      } else if (fs) {
        *fs = F;
      }
      const double td = (-P.w_direct * F.x) * F.y;    // f1d f2d
      const double tx = (-P.w_exchange * F.z) * F.w;  // f1x f2x
      acc_d += td;
      acc_x += tx;
      if (guard) {
        const float kRef = CORR && refined ? 0.125f : 1.0f;  // refined pairs: 2^-49 against 2^-46
        const float4 Sc = st.c, Sd = st.d, Sa = st.a, Sb = st.b;
        const float nac = kRef * Sa.z * Sc.z, nbd = kRef * Sb.z * Sd.z;
        const float s1d = nac * (Sc.y * Sa.x + Sc.x * Sa.y), s2d = nbd * (Sd.y * Sb.x + Sd.x * Sb.y);
        const float s1x = nac * (Sd.y * Sa.x + Sd.x * Sa.y), s2x = nbd * (Sc.y * Sb.x + Sc.x * Sb.y);
        const float fx = fabsf(float(F.x)), fy = fabsf(float(F.y)), fz = fabsf(float(F.z)), fw = fabsf(float(F.w));
        const float ed = wdf * (s1d * fy + fx * s2d);
        const float ex = wxf * (s1x * fw + fz * s2x);
        acc_ed += ed * ed;
        acc_ex += ex * ex;
        acc_ad += fabs(td);
        acc_ax += fabs(tx);
        if constexpr (!CORR) te_d += ed * ed, te_x += ex * ex;
      }
    };
    for (int it = 0; it < my; ++it, w.next(int(gridDim.x))) {
      const int t = int(blockIdx.x) + it * int(gridDim.x);
      const int a = w.a, nbk = min(PB, w.row_blocks() - w.g * PB);
      if constexpr (CORR) {
        if (P.tile_eps && !oz_refine_group(P, w)) {  // the main pass's terms and estimates stand
          for (int j = 0; j < nbk; ++j)
            for (int id = warp * 32 + lane; id < 16 * PW; id += 32 * EPW) {
              const int qg = 16 * a + id / PW, pg = PW * (w.g * PB + j) + id % PW;
              if (qg < P.m && pg < P.m && qg > pg)
                pair_term(make_double4(0.0, 0.0, 0.0, 0.0), qg, pg, false, guard ? load_stats(qg, pg) : PairStats{});
            }
          continue;
        }
      }
      const int slot = u % NSLOT;
      // main pass: this thread's pair of the tile (16 x PW pairs over the epilogue threads); its
      // point stats are fetched now, behind the wait for the accumulators
      PairStats pst{};
      if constexpr (!CORR) {
        const int id = warp * 32 + lane, qg = 16 * a + id / PW, pg = PW * w.g + id % PW;
        if (guard && id < 16 * PW && qg < P.m && pg < P.m && qg > pg) pst = load_stats(qg, pg);
      }
      mbar_wait(&tfull[slot], (u / NSLOT) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) TL(it, 3 + 3 * warp, clock64());
      for (int j = 0; j < nbk; ++j, ++sub) {  // the tile's P blocks in turn (one in the main pass)
      const int b = w.g * PB + j;
      const uint32_t tbase = tmem + (uint32_t(lq * 32) << 16) + uint32_t((slot * PB + j) * NB + c_lo);
      long long X[CPW];
      auto merge = [&](const uint32_t (&v)[NACC][16], int c0, int n) {
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          if (c >= n) break;
          long long x = int32_t(v[0][c]);
#pragma unroll
          // (measured and rejected: the same sum from the low end with 32 x 32 + 64 multiply-adds,
          // IMAD.WIDE -- 272 instead of 459 instructions up to the release, but V-GEMM 1.03 vs 0.98 ms
          // at cfg4 and 6.6 vs 5.7 ms at cfg5-10: the wide multiply-adds issue at a lower rate.
          // Also rejected: each chunk's diagonals loaded in two halves, one half's tcgen05.ld in
          // flight while the other is merged, no more registers: step 1.661 / 1.657 / 1.676 vs
          // 1.656 / 1.658 / 1.665 ms in a same-box A/B -- the drain is TMEM-read-bound (~100 B/clk),
          // not merge-latency-bound)
          for (int d = 1; d < NACC; ++d)  // the last diagonal joins rounded to the one before it
            x = d < S - 1 ? x * 256 + int32_t(v[d][c]) : x + ((int32_t(v[d][c]) + 128) >> 8);
          X[c0 + c] = x;
        }
      };
#pragma unroll
      for (int c0 = 0; c0 + 16 <= CPW; c0 += 16) {
        uint32_t v[NACC][16];
#pragma unroll
        for (int d = 0; d < NACC; ++d) tmem_ld16(tbase + uint32_t(d * NB + c0), v[d]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        merge(v, c0, 16);
      }
      if constexpr (CPW % 16 != 0) {  // N = 80: a last 8-column chunk
        constexpr int c0 = CPW / 16 * 16;
        uint32_t v[NACC][16];
#pragma unroll
        for (int d = 0; d < NACC; ++d) tmem_ld8(tbase + uint32_t(d * NB + c0), v[d]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        merge(v, c0, 8);
      }
      if (j == nbk - 1) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive(&tempty[slot]);  // accumulators free: the next tile's MMAs overlap the work below
      }
      if (lane == 0) TL(it, 4 + 3 * warp, clock64());
      // main pass: V = X 2^(e_q + e_p - 46); refinement: dV = acc 2^(e_q + e_p - 62)
      const double sr = P.sa_scale[size_t(a) * MA + row] * (CORR ? 0x1p-16 : 1.0);
      const double* sbv = P.sb_scale + size_t(b) * NB + c_lo;
      if constexpr (!FUSED) {
        double* dst = P.v + size_t(t) * (MA * NB) + q * 512 + plane * 32 + exq * 8 + c_lo * 8;
#pragma unroll
        for (int p = 0; p < CPW / 8; ++p)
#pragma unroll
          for (int c = 0; c < 8; c += 2)
            __stcg(reinterpret_cast<double2*>(dst + p * 64 + c),
                   make_double2(double(X[8 * p + c]) * sr * sbv[8 * p + c],
                                double(X[8 * p + c + 1]) * sr * sbv[8 * p + c + 1]));
      } else {
        // literal contraction (estimator.cpp:26-32) on the Kramers alpha rows, as pair_kr's epilogue:
        // f(e_q, e_p) = 2 Re sum_{x_alpha, y} o_{e_p}(q, p; y, x_alpha) V(q e_q x_alpha; p e_p y),
        // o = conj O~ from pair_kr_kernel<false, 2>. This thread (q, e_q, x_alpha, re/im plane) holds
        // Re V (plane 0) or Im V (plane 1) for its (p, e_p, y): partial g = sum_y o_re Re V, or
        // -sum_y o_im Im V, then the four lanes of (x_alpha, plane) add up.
        // o blocks are in pair_kr's 16 x 8 tiles: walker p of this tile is p_g = PW b + p, in pair_kr
        // tile a (a + 1) + p_g / 8 (none past the triangle row: those pairs are masked below).
        // FP64 SIMT work runs ~12x slower while tcgen05 MMAs occupy the SM (tools/fp64_vs_umma.cu).
        // An exact integer form of sum_y o_y V_y (53-bit mantissas aligned per quad, 128-bit
        // products) was measured slower, 1.60 vs 1.42 ms at cfg4 (1.26 vs 0.85 ms in the refinement
        // pass): its instruction stream competes with the MMA-issuing warp for issue slots. So the
        // FP64 form stays and the per-pair terms are packed into whole warps after the named barrier
        // (1.42 -> 1.35 ms with the guard's estimate; 1.29 ms with no contraction at all).
        // o values [p][q 16][quad (x_alpha, re/im, e_p) ^ (p & 3)][y 4] (pair_kr's O pass)
        const int row_o = q * 32, quad_o = ((row >> 1) & 1) * 4 + plane * 2;
        const double* so = nullptr;
        const int* se = nullptr;  // the P rows' scale exponents (e 2^20) of this warp's columns
        if constexpr (OSM) {
          mbar_wait(&ofull[u & 1], (u >> 1) & 1);
          so = reinterpret_cast<const double*>(sm + NST * STAGE + (u & 1) * Sh::OT_BUF);
          se = reinterpret_cast<const int*>(sm + NST * STAGE + (u & 1) * Sh::OT_BUF + Sh::OT_BYTES) + c_lo;
        }
        constexpr int NK = CPW / 4;  // (p, e_p) of this warp
        double g[NK];
        // the refinement pass has too few MMAs to hide the o-tile loads behind: load all of this
        // thread's o quads for the P block first (one latency instead of NK), then contract
        constexpr int NPF = CORR ? NK : 1;
        longlong2 opf[NPF][2];
        if constexpr (CORR) {
#pragma unroll
          for (int k = 0; k < NK; ++k) {
            const int pg = min(PW * b + (c_lo + 4 * k) / 8, 16 * (a + 1) - 1);
            const double* o = P.otiles + size_t(a) * (a + 1) * 4096 + size_t(pg) * 512 + row_o +
                              ((quad_o + (k & 1)) ^ (pg & 3)) * 4;
            opf[k][0] = __ldcs(reinterpret_cast<const longlong2*>(o));
            opf[k][1] = __ldcs(reinterpret_cast<const longlong2*>(o + 2));
          }
        }
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          const int pg = PW * b + (c_lo + 4 * k) / 8;
          double sgp = 0.0;
          if (pg < 16 * (a + 1)) {
            if constexpr (!CORR) {
              const double* o = so + ((c_lo + 4 * k) / 8) * 512 + row_o + ((quad_o + (k & 1)) ^ (pg & 3)) * 4;
              const double2 o01 = *reinterpret_cast<const double2*>(o);
              const double2 o23 = *reinterpret_cast<const double2*>(o + 2);
              // V 2^-(e_q - 46) = X 2^(e_p): the P row's power-of-two scale goes into the converted
              // sum's exponent field on the integer pipe (a nonzero X converts to a normal number; the
              // scales keep it one), the Q row's follows below: five FP64 operations per quad beside
              // the conversions
              const int4 eb = *reinterpret_cast<const int4*>(se + 4 * k);
              auto vx = [](long long x, int e20) {
                const double v = double(x);
                const int hi = __double2hiint(v);
                return __hiloint2double(hi ? hi + e20 : 0, __double2loint(v));
              };
              sgp = fma(o23.y, vx(X[4 * k + 3], eb.w),
                        fma(o23.x, vx(X[4 * k + 2], eb.z), fma(o01.y, vx(X[4 * k + 1], eb.y), o01.x * vx(X[4 * k], eb.x))));
            } else {
              // the refinement's correction df = sum o dV is ~2^-46 of f, so FP32 carries it with
              // room to spare (its rounding is ~2^-66 of f): o_y sb_y as a 24-bit float mantissa
              // with an integer exponent (read from the bits), terms aligned to the quad's largest
              // exponent, one conversion and scaling
              const long long ob[4] = {opf[CORR ? k : 0][0].x, opf[CORR ? k : 0][0].y, opf[CORR ? k : 0][1].x,
                                       opf[CORR ? k : 0][1].y};
              int E[4], emax = 0;
#pragma unroll
              for (int y = 0; y < 4; ++y) {
                const int ex = int((ob[y] >> 52) & 0x7FF);  // zero / subnormal o: dropped
                E[y] = ex ? ex + int((__double_as_longlong(sbv[4 * k + y]) >> 52) & 0x7FF) : 0;
                emax = max(emax, E[y]);
              }
              float acc = 0.0f;
#pragma unroll
              for (int y = 0; y < 4; ++y) {
                const int dsh = E[y] - emax;
                if (E[y] == 0 || dsh < -120) continue;
                const float mf = __int_as_float(0x3F800000 | int((ob[y] >> 29) & 0x7FFFFF)) *
                                 __int_as_float((127 + dsh) << 23);
                acc = fmaf(ob[y] < 0 ? -mf : mf, __int2float_rn(int(X[4 * k + y])), acc);
              }
              if (emax) {  // sum = acc 2^(emax - 2046) (the Q row's scale sr follows below)
                const int tt = emax - 2046;
                const double scale = (tt > -1023 && tt < 1024) ? __longlong_as_double((long long)(tt + 1023) << 52) : ldexp(1.0, tt);
                sgp = double(acc) * scale;
              }
            }
          }
          g[k] = sgp * (plane ? -sr : sr);
        }
        if constexpr (OSM) {  // this warp is done with the o buffer
          __syncwarp();
          if (lane == 0) mbar_arrive(&oempty[u & 1]);
        }
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          g[k] += __shfl_xor_sync(0xffffffffu, g[k], 1);
          g[k] += __shfl_xor_sync(0xffffffffu, g[k], 2);
        }
        // lanes row % 8 == 0 (e_q 0) take f(1, e_p) from row + 4 (e_q 1) and park the tile's f
        // values in shared memory; the per-pair terms are formed below by all epilogue lanes
        double4* sf = s_f[sub & 1];
#pragma unroll
        for (int p = 0; p < NK / 2; ++p) {
          const double f10 = __shfl_xor_sync(0xffffffffu, g[2 * p], 4);
          const double f11 = __shfl_xor_sync(0xffffffffu, g[2 * p + 1], 4);
          // f(0,0) = f1d, f(1,1) = f2d, f(1,0) = f1x, f(0,1) = f2x (the factor 2 of 2 Re here)
          if ((row & 7) == 0) sf[q * PW + c_lo / 8 + p] = make_double4(2.0 * g[2 * p], 2.0 * f11, 2.0 * f10, 2.0 * g[2 * p + 1]);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPW) : "memory");  // the tile's 16 x PW f values are parked
        if constexpr (!CORR)
          if (P.tile_eps && tid == 0 && sub > 0) oz_store_tile_eps(P, s_te[(sub - 1) & 1], t - int(gridDim.x));
        const int qg0 = 16 * a, pg0 = PW * b;
        for (int id = (warp * 32 + lane); id < 16 * PW; id += 32 * EPW) {
          const int q2 = id / PW, p2 = id % PW, qg = qg0 + q2, pg = pg0 + p2;
          if (!(qg < P.m && pg < P.m && qg > pg)) continue;
          pair_term(sf[id], qg, pg, true, CORR ? (guard ? load_stats(qg, pg) : PairStats{}) : pst);
        }
        if constexpr (!CORR)
          if (P.tile_eps) {  // this tile's estimate: warp sums now, the CTA's after the next barrier
            float e0 = te_d, e1 = te_x;
            te_d = te_x = 0.0f;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
              e0 += __shfl_down_sync(0xffffffffu, e0, o);
              e1 += __shfl_down_sync(0xffffffffu, e1, o);
            }
            if (lane == 0) s_te[sub & 1][warp] = make_double2(double(e0) * kSig2, double(e1) * kSig2);
          }
      }
      }  // P blocks of the tile
      if (lane == 0) TL(it, 5 + 3 * warp, clock64());
      ++u;
    }
    if constexpr (FUSED) {  // fixed-order CTA sums: warp shuffles, then the epilogue warps in order
      double r[6] = {acc_d, acc_x, double(acc_ed) * kSig2, double(acc_ex) * kSig2, acc_ad, acc_ax};
#pragma unroll
      for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int k = 0; k < 6; ++k) r[k] += __shfl_down_sync(0xffffffffu, r[k], o);
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < 6; ++k) s_red[warp][k] = r[k];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  if constexpr (FUSED && !CORR)
    if (P.tile_eps && tid == 0 && my > 0) oz_store_tile_eps(P, s_te[(my - 1) & 1], int(blockIdx.x) + (my - 1) * int(gridDim.x));
  if constexpr (FUSED) {  // per-CTA partials, then the last CTA's fixed-order sum (as pair_kr.cu)
    if (tid == 0) {
      const double cw = P.ng2 / P.st_ro->wtau;  // estimator.cpp:55
      double r[6] = {0, 0, 0, 0, 0, 0};
      for (int w = 0; w < EPW; ++w)
#pragma unroll
        for (int k = 0; k < 6; ++k) r[k] += s_red[w][k];
      double* pp = P.partials + size_t(blockIdx.x) * 8;
      pp[0] = r[0] * cw;
      pp[1] = 0.0;
      pp[2] = r[1] * cw;
      pp[3] = 0.0;
      pp[4] = r[2] * cw * cw;
      pp[5] = r[3] * cw * cw;
      pp[6] = r[4] * cw;
      pp[7] = r[5] * cw;
      __threadfence();
      s_last = atomicAdd(&P.st->done_pair, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || tid != 0) return;
    __threadfence();
    double r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (unsigned c = 0; c < gridDim.x; ++c)
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] += P.partials[size_t(c) * 8 + k];
    const double d = r[0], x = r[2];
    const double npairs = 0.5 * P.m * (P.m - 1);
    P.step_out[0] = (d + x) / npairs;
    P.step_out[1] = 0.0;
    P.step_out[2] = d;
    P.step_out[3] = 0.0;
    P.step_out[4] = x;
    P.step_out[5] = 0.0;
    // guard: estimated error of the direct and exchange sums and of the step value against
    // guard_tol; a failed (or non-finite) step goes to the refinement pass (oz_trip 1: when the
    // main pass stored the f values) or to the DMMA kernel (oz_trip 2)
    const double ed = sqrt(r[4]), ex = sqrt(r[5]), tol = P.guard_tol;
    const bool trip = guard && tol > 0.0 &&
                      (!(ed <= tol * fabs(d)) || !(ex <= tol * fabs(x)) || !(sqrt(r[4] + r[5]) <= tol * fabs(d + x)));
    P.step_out[6] = ed;
    P.step_out[7] = ex;
    P.step_out[8] = r[6];
    P.step_out[9] = r[7];
    P.step_out[10] = 1.0;
    if constexpr (CORR) {
      P.step_out[11] = trip ? 2.0 : 1.0;  // refined; DMMA next if the refined step still fails
      P.st->oz_trip = trip ? 2 : 0;
    } else {
      P.step_out[11] = trip && !P.fstore ? 2.0 : 0.0;
      if (trip) P.st->oz_trip = P.fstore ? 1 : 2;
      if (trip && P.fstore && P.tile_eps) {
        // the refinement pass refines the tile groups whose estimate exceeds 1 / groups of the
        // step's budget (tol |sum|)^2 -- those left carry at most the budget between them -- and
        // re-forms the others' terms from the stored f values (d, x carry cw, the estimates not)
        const double cw = P.ng2 / P.st_ro->wtau;
        const double ng = double(oz_group_tiles_dev(P.npts_oz / 32, OzShape<true, true>::PW, OzShape<true, true>::PB));
        const double t2 = tol * tol / (cw * cw) / ng;
        P.st->oz_thr[0] = t2 * d * d;
        P.st->oz_thr[1] = t2 * x * x;
        P.st->oz_thr[2] = t2 * (d + x) * (d + x);
      }
    }
    P.st->done_pair = 0;
  }
}

int g_sms_oz[64];
}  // namespace

void oz_layout(int n_vir, int& kh, int& ks) {
  kh = (n_vir + 15) / 16 * 16;
  ks = 2 * kh / 32;
}
size_t oz_slice_bytes_a(int npts_pad, int ks) { return size_t(npts_pad / 32) * ks * A_KSM; }
int oz_p_blocks(int npts_oz, int nb_rows) { return (npts_oz + nb_rows / 4 - 1) / (nb_rows / 4); }
size_t oz_slice_bytes_b(int npts_oz, int ks, int nb_rows) {
  return size_t(oz_p_blocks(npts_oz, nb_rows)) * ks * SL * nb_rows * 32;
}
int oz_nb_rows(bool fused) { return fused ? OzShape<true>::NB : OzShape<false>::NB; }
int oz_ntiles(int nbq, bool fused) { return oz_tiles(nbq, oz_nb_rows(fused) / 8); }

cudaError_t oz_kernel_setup() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_sms_oz[dev & 63], cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaFuncSetAttribute(oz_vgemm_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       OzShape<false>::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(oz_vgemm_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           OzShape<true>::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(oz_vgemm_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              OzShape<true, true>::SMEM_BYTES);
}

void launch_oz_slice(const OzParams& P, cudaStream_t s, bool pdl) {
  const dim3 grid((P.npts_oz + 1) / 2);
  const bool held = P.kh / 4 <= 96;
  if (!pdl) {  // on the side stream, behind an event: a plain launch (griddepcontrol.wait is a no-op)
    if (held) oz_slice_kernel<true><<<grid, 256, 0, s>>>(P);
    else oz_slice_kernel<false><<<grid, 256, 0, s>>>(P);
  } else if (held) {
    pdl_launch(oz_slice_kernel<true>, grid, dim3(256), 0, s, P);
  } else {
    pdl_launch(oz_slice_kernel<false>, grid, dim3(256), 0, s, P);
  }
}

double oz_int8_ops(const OzParams& P) {
  return double(P.ntiles) * (S * (S + 1) / 2) * 2.0 * MA * P.nb_rows * 32.0 * P.ks;
}

void launch_oz_vgemm(const OzParams& P, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = g_sms_oz[dev & 63] > 0 ? g_sms_oz[dev & 63] : 148;
  const int grid = P.ntiles < sms ? P.ntiles : sms;
  if (P.otiles)
    pdl_launch(oz_vgemm_kernel<true, false>, dim3(grid), dim3(THREADS), OzShape<true>::SMEM_BYTES, s, P);
  else
    pdl_launch(oz_vgemm_kernel<false, false>, dim3(grid), dim3(THREADS), OzShape<false>::SMEM_BYTES, s, P);
}

#ifdef OZ_TIMELINE
}  // namespace mcmp2dev
extern "C" int mcmp2dev_debug_oz_timeline(void* host, size_t bytes) {
  return int(cudaMemcpyFromSymbol(host, mcmp2dev::g_oz_tl, bytes < sizeof(mcmp2dev::g_oz_tl) ? bytes : sizeof(mcmp2dev::g_oz_tl)));
}
namespace mcmp2dev {
#endif

void launch_oz_refine(const OzParams& P, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = g_sms_oz[dev & 63] > 0 ? g_sms_oz[dev & 63] : 148;
  const int nt = oz_group_tiles(P.npts_oz / 32, OzShape<true, true>::PW, OzShape<true, true>::PB);
  const int grid = nt < sms ? nt : sms;
  pdl_launch(oz_vgemm_kernel<true, true>, dim3(grid), dim3(THREADS), OzShape<true, true>::SMEM_BYTES, s, P);
}

}  // namespace mcmp2dev
