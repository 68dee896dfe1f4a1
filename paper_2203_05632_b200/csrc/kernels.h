// kernels.h — launch parameters of the libmcmp2dev.so kernels (host + device).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace mcmp2dev {

enum WalkMode { WALK_PRODUCTION = 0, WALK_BURN = 1, WALK_INIT = 2 };

struct WalkParams {
  WalkerBuf in, out;   // sweep reads `in`, writes `out` (ping-pong)
  int m;
  DevSites sites;
  double ng, lambda;
  uint32_t k0, k1, stream;
  DevState* st;
  int mode;
  long long sweep;     // 1-based burn-in sweep index (adaptation every 100)
  int adapt;
  const double* energies;
  int n_occ, n_vir;
  double* sw;          // [n_occ + n_vir] sqrt(guarded_exp) weights of this step
  int* block_acc;      // per-CTA accept counts
  int nens;            // > 1: batched ensembles (walk_batch_kernel), m walkers each, st[nens]
  int sw_stride;       // doubles between the ensembles' spinor weight vectors
  int nactive;         // batched production sweep: ensembles >= nactive (if > 0) stay as they are
};

// spinor evaluation + MO transform (model.cpp:55-64, :166-178) into the Phi layout
struct SpinorParams {
  int npts;            // 2m valid points
  int npts_pad;        // points in the Phi layout (multiple of 2*WB)
  WalkerBuf walkers;
  int ncomp;
  // basis groups: one per channel, or one per Kramers channel pair (shared basis list)
  int ngroups;
  int grp_fn_off[4], grp_nfn[4], grp_k4[4], grp_nf[4];
  int grp_chan[8];             // (x_a, x_b) per group; x_b = -1 for a single channel
  long long grp_chi_off[4], grp_b_off[4];
  int max_nf;
  double* chi;                 // A fragments per group: [pt/8][mu/4][32]
  const double* bfrag;         // B fragments per group: [mu/4][nf][32]
  const double* fn_center;     // [nfunc][3]
  const int* fn_lm;          // [nfunc][2]
  const int* fn_prim_off;    // [nfunc + 1]
  const double* prim_coeff;  // [nprim]
  const int* prim_uniq;      // [nprim] index into the unique (centre, zeta) table
  int nuniq;
  const double* uniq_center; // [nuniq][3]
  const double* uniq_zeta;   // [nuniq]
  int n_occ, n_vir, n_p;
  int Go, Gv;                // occupied and virtual k-groups (PhiChunks)
  const double* sw;
  double* phi;
  double* hinv;              // [m] 1 / (g1 g2) per walker (chi_kernel), folded into Phi_v by mo_kernel
  // mo_kernel tiles (64 points x 8 n fragments), numbered group-major: group g owns tiles
  // [grp_tile0[g], grp_tile0[g] + ptiles * grp_nt[g]); handed out by the DevState counter
  int grp_nt[4], grp_tile0[4];
  int mo_ntiles, mo_slots;
  DevState* st;
  int ens_pts;               // > 0: batched ensembles of ens_pts points, spinor weights sw + e * sw_stride
  int sw_stride;
};

struct PairParams {
  const double* phi;
  int npts_pad, Go, Gv;      // Phi layout (PhiChunks)
  int ring, ring_doubles;    // pair_kr: stage ring depth and stage size for this layout
  int m, nb;                 // walkers, walker blocks of WB
  WalkerBuf walkers;         // g1 (row 6), g2 (row 7)
  const DevState* st_ro;
  DevState* st;
  double ng2, w_direct, w_exchange;
  int physical;              // 1: Tr(o1 va) Tr(o2 vb), Tr(o1 vd o2 vc) epilogue (opt-in)
  double* partials;          // [ntiles][4]; batched: [nens * ens_tiles][consumer warps][2]
  double* step_out;          // [6] of this step (single ensembles: a kStepDoubles record); batched: [nens][6]
  int nens, ens_tiles;       // batched ensembles: m walkers each, st_ro[nens]
  const double* vtiles;      // pair_kr only, single ensemble: V blocks of every tile from
                             // pair_oz.cu (INT8 Ozaki); null: the DMMA V phase
  double* otiles;            // pair_kr only, single ensemble, literal: write the o blocks of every
                             // tile for oz_vgemm_kernel<true> and skip the V phase and the sums
  int guard_fallback;        // pair_kr only: the INT8 path's guard launch -- exit at once unless
                             // st->oz_trip, else recompute the step on DMMA (writes step_out[0..5],
                             // clears oz_trip)
};

// INT8 (Ozaki) V blocks of the Kramers pair stage (pair_oz.cu)
#define OZ_SLICES 6
#define OZ_LZ_STRIDE 32  // k-steps per record of OzParams::lz (n_vir <= 512: at most 32)
struct OzParams {
  const double* phi;
  int npts_pad, Go, Gv;      // Phi layout (PhiChunks)
  int n_vir;
  int npts;                  // 2m points with data
  int npts_oz;               // points covered by the slice blocks (32 per Q block)
  int kh, ks;                // K' = 2 kh = 32 ks
  int ntiles;                // V-GEMM tile triangle (16 x nb_rows / 8 walkers)
  int nb_rows;               // B rows per tile: 64 (physical; pair_kr's 16 x 8 tiles) or 80 (fused)
  int8_t* sa;                // [npts_oz / 32][ks][slice][128 rows x 32] A slices (Q side)
  int8_t* sb;                // [P blocks][ks][slice][nb_rows x 32] B slices (P side, nb_rows / 4 points each)
  double* sa_scale;          // [npts_oz / 32][128]: 2^(e - 49)
  double* sb_scale;          // [P blocks][nb_rows]: 2^e
  int* sb_exp;               // [P blocks][nb_rows]: e 2^20 (the exponent-field increment of 2^e)
  double* v;                 // [ntiles][8192] V blocks in pair_kr's epilogue order (physical)
  // fused literal contraction (oz_vgemm_kernel<true>): o blocks in, the step's sums out
  const double* otiles;      // [ntiles][4096] from pair_kr_kernel<false, 2>
  int m;
  double ng2, w_direct, w_exchange;
  const DevState* st_ro;
  DevState* st;
  double* partials;          // [grid][8]: direct, 0, exchange, 0, sum eps_d^2, sum eps_x^2, sum |t_d|, sum |t_x|
  double* step_out;          // [kStepDoubles] (common.cuh)
  // accuracy guard (literal estimator): per-point stats from oz_slice_kernel, the step's
  // estimated INT8 error against guard_tol (<= 0: no guard)
  int n_occ;
  float* pstat;              // [npts_oz][4]: S = max_x 2^e_x, A = max_x 2^e_x a_x, N = |Phi_o(pt)|_F, 0
  double guard_tol;
  double* fstore;            // [C(m,2)][4] f(0,0), f(1,1), f(1,0), f(0,1) of each pair q > p (index
                             // q (q - 1) / 2 + p), written by the main pass for the refinement pass
  double* tile_eps;          // [ntiles][2] the main pass's sum eps_d^2, sum eps_x^2 per tile: the
                             // refinement pass refines only the tile groups that carry the error
  // active k-steps: K' is ordered by virtual energy (16 spinors' [re | im] per k-step), so the
  // spinors whose exp(-eps tau / 2) leaves no digit in any slice sit in the trailing k-steps;
  // oz_slice_kernel records each point pair's last k-step with a nonzero digit and the V-GEMM
  // runs a tile's k-steps only up to min(Q block's, P block's) -- the products beyond are exact
  // zeros, so the sums are bit-identical to the full K' loop. nullptr: every tile runs all ks.
  uint8_t* ks_cnt;           // [npts_oz / 2]
  // Per point pair and k-step, the first main slice with a nonzero digit (0 .. OZ_SLICES; low
  // nibble: all four channel rows = the pair's B rows, high nibble: its alpha rows = A rows). A
  // k-step whose A operand has `a` and B operand `b` leading zero slices needs only the products
  // (s, t) with s >= a, t >= b (none when a + b >= OZ_SLICES): the rest are exact zeros.
  uint8_t* lz;               // [npts_oz / 2][OZ_LZ_STRIDE]
  unsigned long long* ks_exec;  // slice products issued by the main-pass V-GEMM launches (cumulative; 21 per full k-step)
};
void oz_layout(int n_vir, int& kh, int& ks);
size_t oz_slice_bytes_a(int npts_oz, int ks);
size_t oz_slice_bytes_b(int npts_oz, int ks, int nb_rows);
int oz_p_blocks(int npts_oz, int nb_rows);
int oz_nb_rows(bool fused);
int oz_ntiles(int nbq, bool fused);
void launch_oz_slice(const OzParams& P, cudaStream_t s, bool pdl = true);  // pdl: programmatic launch after the stream's previous kernel
void launch_oz_vgemm(const OzParams& P, cudaStream_t s);
void launch_oz_refine(const OzParams& P, cudaStream_t s);  // exits at once unless st->oz_trip == 1
double oz_int8_ops(const OzParams& P);  // executed int8 tensor ops of one V-GEMM launch
cudaError_t oz_kernel_setup();

void launch_walk(const WalkParams& P, cudaStream_t s);
void launch_replay_load(const WalkParams& P, const double* walkers, double tau, cudaStream_t s);
void launch_spinor(const SpinorParams& P, cudaStream_t s);
int spinor_smem_bytes(const SpinorParams& P);
void launch_pair(const PairParams& P, cudaStream_t s);
cudaError_t pair_kernel_setup();
// Kramers-restricted variant (pair_kr.cu): half the DMMA work for time-reversal-paired columns
void launch_pair_kr(const PairParams& P, cudaStream_t s);
cudaError_t pair_kr_kernel_setup();
// QB = 1 build of pair_kr.cu (8 x 8 tiles, two CTAs per SM) for ensembles of fewer than 64 walkers
void launch_pair_kr_qb1(const PairParams& P, cudaStream_t s);
// PW = 4 build of pair_kr.cu (8 consumer warps) for the O-only pass of the INT8 V path
void launch_pair_kr_pw4(const PairParams& P, cudaStream_t s);
cudaError_t pair_kr_kernel_setup_pw4();
void pair_kr_ring_pw4(int max_width, int& ring, int& ring_doubles);
cudaError_t pair_kr_kernel_setup_qb1();
double pair_kr_block_tiles_qb1(int nb);
int pair_kr_tiles_qb1(int nb);
int pair_kr_consumers_qb1();
void pair_kr_ring_qb1(int max_width, int& ring, int& ring_doubles);
double pair_kr_block_tiles(int nb);
int pair_kr_tiles(int nb);      // tiles of one ensemble of nb walker blocks
int pair_kr_consumers();        // DMMA warps per pair_kr CTA (per-tile partials in batched mode)
int pair_consumers();           // DMMA warps per pair_kernel CTA
void pair_kr_ring(int max_width, int& ring, int& ring_doubles);  // stage ring for the widest chunk  // WB x WB walker blocks the Kramers launch computes
cudaError_t spinor_kernel_setup();
int mo_ctas_per_sm();

}  // namespace mcmp2dev
