// common.cuh — device-side layouts and helpers shared by the walker, spinor and pair
// kernels of libmcmp2dev.so (sm_100a).
//
// HBM layout of the per-step spinor values ("Phi", the output of the MO transform and the
// input of the pair kernel), chosen so the pair kernel's DMMA fragments are contiguous:
//   point pt = 2*walker + electron            (estimator.cpp:39-42: 2p <- r1, 2p+1 <- r2)
//   k-group g = 4 consecutive spinors; occupied groups [0, Go), virtual groups [Go, Go+Gv)
//   chunk c = up to KC4 consecutive groups of one kind (the smem stage of the pair kernel):
//     the occupied groups in chunks of KC4, the last one narrower, then the virtual ones
//   chunk c holding groups [first, first + width):
//     Phi[first * npts_pad + pt * width + (g - first)][plane re/im][x*4 + k%4]
//     (32 doubles per (point, group); 16 per plane, x = channel)
// so one half-fragment (4 channels x 4 spinors) of one point is 128 contiguous bytes and a
// stage (consecutive points x width groups) is one contiguous TMA bulk copy with no padding
// groups. Values are
// scaled by sqrt(guarded_exp(+-eps tau)) so O = Phi_o Phi_o^H and V = Phi_v Phi_v^H carry
// the full exp(+-eps tau) weight (greens.cpp:63-79).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

#include "philox.h"

namespace mcmp2dev {

#ifndef KC4_GROUPS
// cfg4 Kramers pair kernel (ms): KC4 4 -> 4.08, 5 -> 4.03, 6 -> 4.04, 7 -> 4.02 (2 stages of
// 86 KB); 8 does not fit two stages next to the o table. General kernel neutral, physical -2%.
#define KC4_GROUPS 7
#endif
constexpr int KC4 = KC4_GROUPS;  // k-groups per pair-kernel stage
constexpr int WB = 8;           // walkers per pair-kernel tile side
constexpr int NCH = 4;          // channels per point in the Phi layout (ncomp <= 4, zero padded)
// per-step record of a single ensemble (include/mcmp2dev.h mcmp2dev_step_ex): value, imag,
// direct re/im, exchange re/im, then the INT8 path's guard: estimated error of the direct and
// exchange sums, sums of |pair term|, INT8 flag, fallback level (0 main pass, 1 refined, 2 DMMA)
constexpr int kStepDoubles = 12;

// Bank swizzle of the Phi layout: element (x, k) of point pt sits at (x*4 + k) ^ phi_swz(pt).
// Points pt and pt^1, and pt and pt^2, land on different halves of the 32 banks, so the
// alpha-row fragment loads of pair_kr.cu (4 doubles from each of 4 points per half-warp) are
// conflict-free; whole half-fragment loads stay permutations of one 128-byte row.
__host__ __device__ __forceinline__ int phi_swz(int pt) { return ((pt ^ (pt >> 1)) & 1) << 2; }

// chunking of the k-groups (see the layout above); identical on host and device
struct PhiChunks {
  int Go, Gv;  // occupied and virtual k-groups
  __host__ __device__ int occ_chunks() const { return (Go + KC4 - 1) / KC4; }
  __host__ __device__ int count() const { return occ_chunks() + (Gv + KC4 - 1) / KC4; }
  __host__ __device__ int first(int c) const {
    const int co = occ_chunks();
    return c < co ? c * KC4 : Go + (c - co) * KC4;
  }
  __host__ __device__ int width(int c) const {
    const int co = occ_chunks(), r = c < co ? Go - c * KC4 : Gv - (c - co) * KC4;
    return r < KC4 ? r : KC4;
  }
  __host__ __device__ int chunk_of(int g) const { return g < Go ? g / KC4 : occ_chunks() + (g - Go) / KC4; }
  // offset in doubles of (group g, point pt)
  __host__ __device__ size_t offset(int g, int pt, int npts_pad) const {
    const int c = chunk_of(g), f = first(c);
    return (size_t(f) * npts_pad + size_t(pt) * width(c) + (g - f)) * 32;
  }
};

// ------------------------------------------------------------------ programmatic dependent launch
// Every kernel of a step is launched with programmatic stream serialization (pdl_launch) and
// starts with pdl_wait(): griddepcontrol.wait blocks until the preceding kernel has completed and
// its memory is visible (a no-op for a normal launch), so correctness is that of plain stream
// order, while the launch of a kernel overlaps the tail of the previous one. pdl_trigger()
// (griddepcontrol.launch_dependents) lets the next kernel launch once every CTA has passed it.
#ifndef MCMP2_PDL
#define MCMP2_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if MCMP2_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if MCMP2_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

#ifdef __CUDACC__
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = MCMP2_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
#endif

// ------------------------------------------------------------------ overlap timeline (debug)
// OZ_OVERLAP_TL build (tools/overlap_timeline.py): first CTA start and last CTA end of a kernel
// on the global nanosecond timer, in a per-translation-unit pair g_tl[2] (pair_oz.cu: the slice
// kernel, pair_kr.cu: the O pass)
#ifdef OZ_OVERLAP_TL
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define OVERLAP_TL_BEGIN(g) \
  if (threadIdx.x == 0) atomicMin(&(g)[0], global_ns())
#define OVERLAP_TL_END(g) \
  if (threadIdx.x == 0) atomicMax(&(g)[1], global_ns())
#define OVERLAP_TL_DEFINE(g, getter)                                                       \
  static __device__ unsigned long long g[2] = {~0ull, 0ull};                              \
  extern "C" int getter(unsigned long long* host2, int reset) {                          \
    int e = int(cudaMemcpyFromSymbol(host2, g, 16));                                      \
    const unsigned long long init[2] = {~0ull, 0ull};                                    \
    if (reset) e |= int(cudaMemcpyToSymbol(g, init, 16));                                 \
    return e;                                                                             \
  }
#else
#define OVERLAP_TL_BEGIN(g)
#define OVERLAP_TL_END(g)
#endif

// ------------------------------------------------------------------ device system
struct DevSites {
  int n;
  const double* pos;    // [n][3]
  const double* prim;   // [n][2][2] (coeff, zeta)
  const double* zeta1;  // [n]
};

// walker arrays, SoA: [9][mmax] = r1x r1y r1z r2x r2y r2z g1 g2 weight
struct WalkerBuf {
  double* w;
  int mmax;
  __device__ double& at(int k, int p) const { return w[size_t(k) * mmax + p]; }
};

// device-resident per-handle scalars
struct DevState {
  unsigned long long pos;     // next u32 of the reference stream
  double sigma;               // sigma_step
  double tau, wtau;           // this step's tau and its density (weights.cpp:109-111)
  long long proposed, accepted;
  long long win_prop, win_acc;  // burn-in adaptation window (sampler.cpp:82-90)
  int error;                  // 1: exponential overflow (greens.cpp:10-13)
  int error_idx;              // spinor index of the overflow
  int redo;                   // a coincident proposal needs the sequential path
  unsigned int done_ctas;     // last-CTA counters (walker kernel)
  unsigned int done_pair;     // (pair kernel)
  int spec_error_idx;         // overflow index from the speculative tau draw (INT_MAX: none)
  unsigned int mo_next;       // mo_kernel tile counter (dynamic scheduling)
  unsigned int mo_done;       // mo_kernel CTAs finished (the last one resets both)
  int oz_trip;                // INT8 V path: this step's error estimate failed the guard; 1: the
                              // refinement pass runs (oz_vgemm_kernel<true, true>), 2: the guarded
                              // DMMA pair launch recomputes the step; each clears it when done
  double oz_thr[3];           // the refinement pass's group thresholds on the main pass's error
                              // estimates (sum eps_d^2, sum eps_x^2, their sum), set with oz_trip 1
};

}  // namespace mcmp2dev
