// mcmp2dev.cu — handle management and the C ABI of libmcmp2dev.so (include/mcmp2dev.h).
//
// One handle = one reference "worker" (driver.cpp:200-205) resident on one device -- or, after
// mcmp2dev_init_batch, several workers as batched ensembles: the immutable system
// (SpinorSet/WeightSpec/TauSampler), the walker ensembles (ping-pong SoA buffers + a DevState
// per ensemble with its Philox stream position) and the per-step work buffers. Each MC step is
// four launches on the handle's stream (programmatic dependent launches, captured in CUDA
// graphs of 32 steps): walk (Metropolis sweep + tau), chi (basis values), mo (MO transform into
// the Phi layout), pair (O/V GEMMs + integrand + reduction). Per-step StepEstimates stay on the
// device until the end of a chunk, then one copy returns them.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/mcmp2dev.h"
#include "common.cuh"
#include "kernels.h"

using namespace mcmp2dev;

namespace {

constexpr int kChunk = 1024;  // steps per device->host copy of StepEstimates
constexpr int kGraphSteps = 32;  // production steps per captured CUDA graph (even)
constexpr int kBatchMaxWalkers = 480;  // per batched ensemble (2m + 32 threads <= 1024, m % 16 == 0)
// default guard tolerance of the INT8 V path: the estimated error must stay below 2e-10 of
// |direct|, |exchange| and |value|. Measured on 2000-step chains (profiles/r07_guard_*): the
// estimate is 2.3-170x the actual error; at 3e-10 the steps kept on the main pass stay within
// 6e-11 of FP64 (the unguarded path exceeds the 1e-10 gate on 0.6-0.8% of the steps, by up to
// 3e-7 on the value); 2e-10 keeps a 2x margin at the smallest measured estimate/error ratio.
// Cost at cfg4 (profiles/r07_guard_cost_cfg4.json): estimate 0.09 ms/step, each refined step
// ~0.9 ms (10-15% of the steps at 3e-10)
constexpr double kGuardTol = 2e-10;
thread_local std::string g_create_error;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct RtError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
T* dalloc(size_t n, std::vector<void*>& owned) {
  void* p = nullptr;
  ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
  owned.push_back(p);
  return static_cast<T*>(p);
}

// copies ordered on the handle's (non-blocking) stream, then waited for: a plain cudaMemcpy
// runs on the legacy stream, which does not order against cudaStreamNonBlocking streams
cudaError_t scopy(cudaStream_t s, void* dst, const void* src, size_t n, cudaMemcpyKind kind) {
  cudaError_t e = cudaMemcpyAsync(dst, src, n, kind, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

template <class T>
T* dupload(const T* src, size_t n, std::vector<void*>& owned) {
  T* d = dalloc<T>(n, owned);
  if (n) ck(cudaMemcpy(d, src, n * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  return d;
}

}  // namespace

#ifndef OZ_O_PW4
#define OZ_O_PW4 1  // O-only pass of the INT8 path on the PW = 4 build of pair_kr (8 consumer warps):
                    // 0.443 -> 0.392 ms at cfg4 (same-box A/B), more independent DMMA chains per warp
#endif

struct mcmp2dev_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  // INT8 V path: oz_slice_kernel runs here, next to the O pass on `stream`
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool oz_overlap = true;
  std::vector<void*> owned;
  std::string err;

  // system
  int ncomp = 0, n_occ = 0, n_vir = 0, n_p = 0, nfunc = 0, rows = 0;
  int Go = 0, Gv = 0;
  double ng = 0, lambda = 0, w_direct = 0, w_exchange = 0;
  int estimator = 0;
  bool kramers_eligible = false, kramers = false;  // pair_kr.cu path
  double kramers_dev = 0.0;                         // deviation from exact time-reversal pairing
  // V blocks of the Kramers pair stage on the INT8 tensor cores (pair_oz.cu), single ensembles
  // of QB = 2 tiles; buffers sized for oz_m walkers, grown outside graph capture (ensure_oz)
  bool oz = true;
  // Selected by default only above 16 virtual spinors (more than one 32-wide k-step of K'): with
  // a single k-step the V-GEMM is bound by its per-tile epilogue, not by MMAs, and the DMMA pair
  // kernel is faster (cfg5-2, n_vir 10, m 8192: 5.3 vs 6.6 ms per step; cfg5-10, n_vir 30: 10.0
  // vs 8.0). mcmp2dev_pair_path(h, 1) selects it regardless.
  static constexpr int kOzAutoMinVir = 16;
  bool oz_forced = false;
  int oz_m = 0;
  OzParams ozp{};
  double* oz_otiles = nullptr;
  // accuracy guard of the INT8 path (literal estimator): a step whose estimated INT8 error of
  // the direct sum, the exchange sum or the step value exceeds guard_tol of that quantity is
  // recomputed on the DMMA pair kernel (pair_oz.cu, pair_kr.cu guard_fallback); <= 0: off
  double guard_tol = kGuardTol;
  float* d_pstat = nullptr;   // [npts_oz][4] point stats (oz_slice_kernel)
  double* d_fstore = nullptr; // [C(oz_m, 2)][4] f values of the main pass for the refinement pass
  // per-tile k-step truncation of the INT8 V-GEMM (OzParams::ks_cnt): on by default, exact
  bool oz_trunc = true;
  bool oz_trunc_slices = true;  // with oz_trunc: also the leading zero slices of each k-step (OzParams::lz)
  uint8_t* d_ks_cnt = nullptr;             // [npts_oz / 2]
  uint8_t* d_lz = nullptr;                 // [npts_oz / 2][OZ_LZ_STRIDE] leading zero slices (OzParams::lz)
  unsigned long long* d_ks_exec = nullptr; // k-steps issued by the main-pass V-GEMM launches
  double oz_ks_full = 0;                   // k-steps of one untruncated launch (last launch's sizes)
  double* d_tile_eps = nullptr;  // [main tiles][2] the main pass's error estimate per tile
  long long guard_steps = 0, guard_refined = 0, guard_dmma = 0;
  double guard_max_est = 0.0;  // largest estimated relative error of a step kept on INT8
  SpinorParams sp{}, sp_kr{};  // general / Kramers-pair MO transform groups
  DevSites sites{};
  double* d_energies = nullptr;
  double* d_sw = nullptr;

  // ensemble
  int mmax = 0, nbmax = 0, npts_pad = 0;
  int m = 0;
  uint32_t k0 = 0, k1 = 0, rstream = 0;
  bool have_ensemble = false;
  WalkerBuf buf[2]{}, rbuf{};
  int cur = 0;
  DevState* d_state = nullptr;  // [nens_cap]: ensemble e of a batched handle uses d_state[e]
  int nens = 1, nens_cap = 1;   // batched ensembles (mcmp2dev_init_batch): walkers [e m, (e+1) m)
  double* d_bpart = nullptr;    // batched: per-tile pair partials
  size_t bpart_cap = 0;
  double* d_bsteps = nullptr;   // batched: [kGraphSteps][nens][6] step results
  double* h_bsteps = nullptr;   // pinned
  size_t bsteps_cap = 0;
  int* d_block_acc = nullptr;
  double* d_phi = nullptr;
  double* d_hinv = nullptr;
  double* d_partials = nullptr;
  double* d_steps = nullptr;
  double* d_replay = nullptr;
  double* h_steps = nullptr;  // pinned
  double* h_replay = nullptr; // pinned [mmax][8]

  // profiling
  bool prof = false;
  cudaEvent_t ev[4]{};
  cudaEvent_t ev_oz[3]{};                   // after oz_slice_kernel, before / after oz_vgemm_kernel
  double prof_oz[5] = {0, 0, 0, 0, 0};       // ms of slice, V-GEMM, pair_kr (INT8 V path), launches,
                                             // the guard's refinement + DMMA launches
  double oz_ops = 0;                         // int8 ops of the last V-GEMM launch
  double prof_ms[4] = {0, 0, 0, 0};
  double prof_n[4] = {0, 0, 0, 0};

  // captured production steps, one per walker-buffer parity; valid for one (m, RNG key/stream,
  // kernel path)
  cudaGraphExec_t graphs[2] = {nullptr, nullptr};
  double* d_gsteps = nullptr;  // [kGraphSteps][kStepDoubles] step results written by the graph
  struct GraphKey {
    int m = -1, kramers = -1, nens = 1, oz = -1, trunc = -1, overlap = -1;
    uint32_t k0 = 0, k1 = 0, stream = 0;
    double guard_tol = -1.0;
    bool operator==(const GraphKey&) const = default;
  } graph_keys[2];

  cudaGraphExec_t ensure_graph() {
    const GraphKey key{m, kramers ? 1 : 0, nens, oz_active(m, nens) ? 1 : 0, oz_trunc ? (oz_trunc_slices ? 2 : 1) : 0, oz_overlap ? 1 : 0, k0, k1, rstream, guard_tol};
    cudaGraphExec_t& graph_exec = graphs[cur];
    if (graph_exec && key == graph_keys[cur]) return graph_exec;
    if (graph_exec) cudaGraphExecDestroy(graph_exec), graph_exec = nullptr;
    cudaGraph_t g = nullptr;
    ck(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "graph capture");
    const int c0 = cur;
    for (int s = 0; s < kGraphSteps; ++s) {  // even count: the walker parity returns to c0
      launch_walk(walk_params(WALK_PRODUCTION, 0, 0), stream);
      cur ^= 1;
      if (nens > 1) launch_estimate(buf[cur], m, d_bsteps + size_t(6) * nens * s, nens);
      else launch_estimate(buf[cur], m, d_gsteps + kStepDoubles * s);
    }
    cur = c0;
    ck(cudaStreamEndCapture(stream, &g), "graph capture end");
    ck(cudaGraphInstantiate(&graph_exec, g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    graph_keys[cur] = key;
    return graph_exec;
  }

  WalkParams walk_params(int mode, long long sweep, int adapt) {
    WalkParams P{};
    P.in = buf[cur];
    P.out = buf[cur ^ 1];
    P.m = m;
    P.sites = sites;
    P.ng = ng;
    P.lambda = lambda;
    P.k0 = k0;
    P.k1 = k1;
    P.stream = rstream;
    P.st = d_state;
    P.mode = mode;
    P.sweep = sweep;
    P.adapt = adapt;
    P.energies = d_energies;
    P.n_occ = n_occ;
    P.n_vir = n_vir;
    P.sw = d_sw;
    P.block_acc = d_block_acc;
    P.nens = nens;
    P.sw_stride = n_p;
    return P;
  }

  // the QB = 1 build of pair_kr.cu (8 x 8 tiles, 2 CTAs/SM) for small ensembles (m < 64) and when
  // the QB = 2 tiles would not cover the SMs (single cfg2, m = 128: 72 tiles; 197 -> 211 M samples/s);
  // measured slower for batched cfg2 (x4: 370 vs 354 M) and cfg3 (0.171 vs 0.191 ms)
  int sms = 148;
  bool kr_qb1(int mm, int ne = 1) const {
    return mm < 64 || double(ne) * pair_kr_tiles((mm + WB - 1) / WB) < sms;
  }

  bool oz_active(int mm, int ne) const {
    return oz && kramers && ne == 1 && mm >= 2 && !kr_qb1(mm, ne) && n_vir > 0 && n_vir <= 512 &&
           (oz_forced || n_vir > kOzAutoMinVir);
  }
  void oz_free() {
    for (void* p : {(void*)ozp.sa, (void*)ozp.sb, (void*)ozp.sa_scale, (void*)ozp.sb_scale, (void*)ozp.sb_exp, (void*)ozp.v,
                    (void*)oz_otiles, (void*)d_pstat, (void*)d_fstore, (void*)d_tile_eps, (void*)d_ks_cnt,
                    (void*)d_ks_exec, (void*)d_lz})
      if (p) cudaFree(p);
    d_ks_cnt = nullptr;
    d_ks_exec = nullptr;
    d_lz = nullptr;
    ozp.sa = ozp.sb = nullptr;
    ozp.sa_scale = ozp.sb_scale = ozp.v = nullptr;
    ozp.sb_exp = nullptr;
    oz_otiles = nullptr;
    d_pstat = nullptr;
    d_fstore = nullptr;
    d_tile_eps = nullptr;
    oz_m = 0;
  }
  // captured steps hold the addresses of every work buffer: any reallocation drops them first
  void drop_graphs() {
    ck(cudaStreamSynchronize(stream), "graph drop sync");
    for (auto& g : graphs)
      if (g) cudaGraphExecDestroy(g), g = nullptr;
  }
  // buffers of the INT8 V path for mm walkers (no-op when inactive or already large enough)
  void ensure_oz(int mm) {
    if (!oz_active(mm, 1) || mm <= oz_m) return;
    drop_graphs();
    oz_free();
    const int nbq = (mm + 15) / 16, npts_oz = 32 * nbq;
    int kh = 0, ks = 0;
    oz_layout(n_vir, kh, ks);
    const size_t ntiles = size_t(nbq) * (nbq + 1);
    ck(cudaStreamSynchronize(stream), "oz sync");
    ck(cudaMalloc(&ozp.sa, oz_slice_bytes_a(npts_oz, ks)), "cudaMalloc oz slices");
    // B blocks: 8 walkers (physical) or 10 (literal, fused); rows past the last point stay zero
    const int nbr = oz_nb_rows(estimator != MCMP2DEV_ESTIMATOR_PHYSICAL);
    const size_t sb_bytes = oz_slice_bytes_b(npts_oz, ks, nbr);
    const size_t sbs_bytes = sizeof(double) * oz_p_blocks(npts_oz, nbr) * nbr;
    ck(cudaMalloc(&ozp.sb, sb_bytes), "cudaMalloc oz slices");
    ck(cudaMemset(ozp.sb, 0, sb_bytes), "memset oz slices");
    ck(cudaMalloc(&ozp.sa_scale, sizeof(double) * npts_oz * 4), "cudaMalloc oz scales");
    ck(cudaMalloc(&ozp.sb_scale, sbs_bytes), "cudaMalloc oz scales");
    ck(cudaMemset(ozp.sb_scale, 0, sbs_bytes), "memset oz scales");
    ck(cudaMalloc(&ozp.sb_exp, sbs_bytes / 2), "cudaMalloc oz scale exponents");
    ck(cudaMemset(ozp.sb_exp, 0, sbs_bytes / 2), "memset oz scale exponents");
    // physical estimator: V tiles for pair_kr's trace epilogue; literal: o tiles for the fused
    // contraction in the V-GEMM epilogue
    if (estimator == MCMP2DEV_ESTIMATOR_PHYSICAL)
      ck(cudaMalloc(&ozp.v, sizeof(double) * 8192 * ntiles), "cudaMalloc oz V blocks");
    else {
      ck(cudaMalloc(&oz_otiles, sizeof(double) * 4096 * ntiles), "cudaMalloc oz o blocks");
      const size_t mq = size_t(16) * nbq;
      ck(cudaMalloc(&d_fstore, sizeof(double) * 4 * (mq * (mq - 1) / 2)), "cudaMalloc oz pair f values");
      ck(cudaMalloc(&d_tile_eps, sizeof(double) * 2 * oz_ntiles(nbq, true)), "cudaMalloc oz tile estimates");
    }
    ck(cudaMalloc(&d_pstat, sizeof(float) * 4 * npts_oz), "cudaMalloc oz point stats");
    ck(cudaMemset(d_pstat, 0, sizeof(float) * 4 * npts_oz), "memset oz point stats");
    ck(cudaMalloc(&d_ks_cnt, npts_oz / 2), "cudaMalloc oz k-step counts");
    ck(cudaMemset(d_ks_cnt, 0, npts_oz / 2), "memset oz k-step counts");
    ck(cudaMalloc(&d_lz, size_t(npts_oz / 2) * OZ_LZ_STRIDE), "cudaMalloc oz leading-zero slices");
    ck(cudaMemset(d_lz, 0, size_t(npts_oz / 2) * OZ_LZ_STRIDE), "memset oz leading-zero slices");
    ck(cudaMalloc(&d_ks_exec, sizeof(unsigned long long)), "cudaMalloc oz k-step counter");
    ck(cudaMemset(d_ks_exec, 0, sizeof(unsigned long long)), "memset oz k-step counter");
    oz_m = 16 * nbq;
  }

  void launch_estimate(const WalkerBuf& wb, int mm, double* step_out, int ne = 1) {
    SpinorParams s = kramers ? sp_kr : sp;
    s.npts = 2 * mm * ne;
    s.ens_pts = ne > 1 ? 2 * mm : 0;
    s.sw_stride = n_p;
    s.walkers = wb;
    if (prof) ck(cudaEventRecord(ev[1], stream), "event");
    launch_spinor(s, stream);
    if (prof) ck(cudaEventRecord(ev[2], stream), "event");
    PairParams p{};
    p.phi = d_phi;
    p.npts_pad = npts_pad;
    p.Go = Go;
    p.Gv = Gv;
    const bool qb1 = kr_qb1(mm, ne);
    {
      const int wmax = std::min(KC4, std::max(Go, Gv));
      if (qb1) pair_kr_ring_qb1(wmax > 0 ? wmax : 1, p.ring, p.ring_doubles);
      else pair_kr_ring(wmax > 0 ? wmax : 1, p.ring, p.ring_doubles);
    }
    p.m = mm;
    p.nb = (mm + WB - 1) / WB;
    p.walkers = wb;
    p.st_ro = d_state;
    p.st = d_state;
    p.ng2 = ng * ng;
    p.w_direct = w_direct;
    p.w_exchange = w_exchange;
    p.physical = estimator == MCMP2DEV_ESTIMATOR_PHYSICAL;
    p.partials = ne > 1 ? d_bpart : d_partials;
    p.step_out = step_out;
    p.nens = ne;
    p.ens_tiles = ne > 1 ? (kramers ? (qb1 ? pair_kr_tiles_qb1(p.nb) : pair_kr_tiles(p.nb)) : p.nb * (p.nb + 1) / 2) : 0;
    p.vtiles = nullptr;
    p.otiles = nullptr;
    const bool oz_path = oz_active(mm, ne);
    const bool fused = oz_path && !p.physical;
    const bool guarded = fused && guard_tol > 0.0;
    const PairParams p_full = p;  // the DMMA pair stage (the guard's fallback launch)
    if (oz_path) {
      if (mm > oz_m) throw RtError("mcmp2dev: INT8 V buffers not prepared for this ensemble size");
      OzParams o = ozp;
      o.phi = d_phi;
      o.npts_pad = npts_pad;
      o.Go = Go;
      o.Gv = Gv;
      o.n_vir = n_vir;
      o.npts = 2 * mm;
      const int nbq = (mm + 15) / 16;
      o.npts_oz = 32 * nbq;
      oz_layout(n_vir, o.kh, o.ks);
      o.ntiles = oz_ntiles(nbq, fused);
      o.nb_rows = oz_nb_rows(fused);
      o.otiles = fused ? oz_otiles : nullptr;
      o.m = mm;
      o.ng2 = p.ng2;
      o.w_direct = w_direct;
      o.w_exchange = w_exchange;
      o.st_ro = d_state;
      o.st = d_state;
      o.partials = d_partials;
      o.step_out = step_out;
      o.n_occ = n_occ;
      o.pstat = guarded ? d_pstat : nullptr;
      o.guard_tol = guard_tol;
      o.fstore = guarded ? d_fstore : nullptr;
      o.tile_eps = guarded ? d_tile_eps : nullptr;
      o.ks_cnt = oz_trunc ? d_ks_cnt : nullptr;
      o.lz = oz_trunc && oz_trunc_slices && o.ks <= OZ_LZ_STRIDE ? d_lz : nullptr;
      o.ks_exec = d_ks_exec;
      // Literal estimator: the slice kernel (integer / load-store work, 1 KB of shared memory) and
      // the O pass (DMMA, one CTA per SM) need only Phi, so the slices are cut on a side stream
      // next to the O pass and the V-GEMM waits for both (the fork and join are captured into
      // the step graphs like any other dependency). Profiling runs keep them in series so each
      // kernel's events time it alone.
      const bool fork = fused && !prof && oz_overlap;
      if (fork) ck(cudaEventRecord(ev_fork, stream), "fork event");
      else launch_oz_slice(o, stream, true);
      if (prof) ck(cudaEventRecord(ev_oz[0], stream), "event");
      if (fused) {  // o blocks first, then V blocks with the contraction and the step's sums
        p.otiles = oz_otiles;
        if (OZ_O_PW4) {
          const int wmax = std::min(KC4, std::max(Go, 1));
          pair_kr_ring_pw4(wmax, p.ring, p.ring_doubles);
          launch_pair_kr_pw4(p, stream);
        } else {
          launch_pair_kr(p, stream);
        }
        if (prof) ck(cudaEventRecord(ev_oz[1], stream), "event");
        if (fork) {  // the O pass is in flight (its CTAs take their SMs first); the slices beside it
          ck(cudaStreamWaitEvent(side, ev_fork, 0), "fork wait");
          launch_oz_slice(o, side, false);
          ck(cudaEventRecord(ev_join, side), "join event");
          ck(cudaStreamWaitEvent(stream, ev_join, 0), "join wait");
        }
        launch_oz_vgemm(o, stream);
        if (prof) ck(cudaEventRecord(ev_oz[2], stream), "event");
        if (guarded) {  // each exits at once unless the step failed the check before it
          launch_oz_refine(o, stream);
          PairParams f = p_full;
          f.guard_fallback = 1;
          launch_pair_kr(f, stream);
        }
      } else {
        launch_oz_vgemm(o, stream);
        if (prof) ck(cudaEventRecord(ev_oz[1], stream), "event");
        if (prof) ck(cudaEventRecord(ev_oz[2], stream), "event");
        p.vtiles = o.v;
        launch_pair_kr(p, stream);
      }
      oz_ops = oz_int8_ops(o);
      oz_ks_full = double(o.ntiles) * o.ks;
    } else if (kramers && qb1) {
      launch_pair_kr_qb1(p, stream);
    } else if (kramers) {
      launch_pair_kr(p, stream);
    } else {
      launch_pair(p, stream);
    }
    if (prof) {
      ck(cudaEventRecord(ev[3], stream), "event");
      ck(cudaEventSynchronize(ev[3]), "event sync");
      float a = 0, b = 0, c = 0;
      ck(cudaEventElapsedTime(&a, ev[0], ev[1]), "elapsed");
      ck(cudaEventElapsedTime(&b, ev[1], ev[2]), "elapsed");
      ck(cudaEventElapsedTime(&c, ev[2], ev[3]), "elapsed");
      prof_ms[0] += a;
      prof_ms[1] += b;
      prof_ms[2] += c;
      prof_ms[3] += a + b + c;
      if (oz_path) {  // slice, then V-GEMM and pair_kr in launch order (fused: pair_kr first)
        float x = 0, y = 0, z = 0, gz = 0;
        ck(cudaEventElapsedTime(&x, ev[2], ev_oz[0]), "elapsed");
        ck(cudaEventElapsedTime(&y, ev_oz[0], ev_oz[1]), "elapsed");
        ck(cudaEventElapsedTime(&z, ev_oz[1], ev_oz[2]), "elapsed");
        ck(cudaEventElapsedTime(&gz, ev_oz[2], ev[3]), "elapsed");
        prof_oz[0] += x;
        prof_oz[1] += fused ? z : y;
        prof_oz[2] += fused ? y : z + gz;
        prof_oz[3] += 1;
        prof_oz[4] += fused ? gz : 0.0;
      }
      prof_n[0] += 1;
      prof_n[1] += 1;
      prof_n[2] += 1;
      prof_n[3] += 1;
    }
    ck(cudaGetLastError(), "kernel launch");
  }

  void check_state_errors() {
    std::vector<DevState> all(nens);
    ck(cudaMemcpyAsync(all.data(), d_state, sizeof(DevState) * nens, cudaMemcpyDeviceToHost, stream), "state D2H");
    ck(cudaStreamSynchronize(stream), "stream sync");
    DevState st = all[0];
    for (const DevState& x : all)
      if (x.error && (!st.error || x.error_idx < st.error_idx)) st = x;
    if (st.error) {
      reset_errors();
      // greens.cpp:10-13
      throw RtError("greens: exponential overflow for spinor " + std::to_string(st.error_idx) +
                    " (positive occupied or negative virtual energy with large tau?)");
    }
  }

  void reset_errors() {
    std::vector<DevState> all(nens);
    ck(scopy(stream, all.data(), d_state, sizeof(DevState) * nens, cudaMemcpyDeviceToHost), "state D2H");
    for (DevState& st : all) {
      st.error = 0;
      st.error_idx = INT_MAX;
      st.spec_error_idx = INT_MAX;
    }
    ck(scopy(stream, d_state, all.data(), sizeof(DevState) * nens, cudaMemcpyHostToDevice), "state H2D");
  }

  // read-modify-write of every ensemble's DevState
  template <class F>
  void each_state(F&& f) {
    std::vector<DevState> all(nens);
    ck(scopy(stream, all.data(), d_state, sizeof(DevState) * nens, cudaMemcpyDeviceToHost), "state D2H");
    for (DevState& st : all) f(st);
    ck(scopy(stream, d_state, all.data(), sizeof(DevState) * nens, cudaMemcpyHostToDevice), "state H2D");
  }
};

namespace {

template <class F>
int guard(mcmp2dev_t* h, F&& f) {
  std::string* err = h ? &h->err : &g_create_error;
  try {
    if (h) ck(cudaSetDevice(h->device), "cudaSetDevice");
    f();
    return MCMP2DEV_OK;
  } catch (const ArgError& e) {
    *err = e.what();
    return MCMP2DEV_INVALID_ARGUMENT;
  } catch (const RtError& e) {
    *err = e.what();
    return MCMP2DEV_RUNTIME;
  } catch (const CudaError& e) {
    *err = e.what();
    return MCMP2DEV_CUDA;
  } catch (const std::exception& e) {
    *err = e.what();
    return MCMP2DEV_RUNTIME;
  }
}

// Time-reversal pairing of the spinor columns (oracle.cpp:346-355 generalised): channel pairs
// (0,1) [and (2,3)] carry identical basis lists, columns (2k, 2k+1) satisfy (a, b) -> (-b*, a*)
// per channel pair and pair energies are equal. Returns the largest deviation from exact pairing
// relative to max |C| (coefficients) and max |eps| (energies), or +inf when the structure does
// not pair (odd counts, basis lists that differ). The Kramers path derives every odd column
// from its even partner, so a deviation d changes the results by O(d) relative: inputs within
// kKramersTol use it (a Dirac-Hartree-Fock set paired to rounding, not bit for bit).
constexpr double kKramersTol = 1e-12;
double kramers_deviation(const mcmp2dev_system* s, const std::vector<int>& ch_off) {
  const double inf = HUGE_VAL;
  if (s->ncomp == 1 || s->n_occ % 2 || s->n_vir % 2) return inf;
  const int np = s->n_occ + s->n_vir;
  double emax = 0.0, cmax = 0.0, de = 0.0, dc = 0.0;
  for (int k = 0; k < np; ++k) emax = std::max(emax, std::fabs(s->energies[k]));
  for (int k = 0; k < np; k += 2) de = std::max(de, std::fabs(s->energies[k] - s->energies[k + 1]));
  for (int i = 0; i < 2 * ch_off[s->ncomp] * np; ++i) cmax = std::max(cmax, std::fabs(s->coeff[i]));
  for (int pr = 0; pr < s->ncomp / 2; ++pr) {
    const int a0 = ch_off[2 * pr], b0 = ch_off[2 * pr + 1], n = ch_off[2 * pr + 1] - ch_off[2 * pr];
    if (ch_off[2 * pr + 2] - b0 != n) return inf;
    for (int i = 0; i < n; ++i) {
      const int fa = a0 + i, fb = b0 + i;
      for (int d = 0; d < 3; ++d)
        if (s->fn_center[3 * fa + d] != s->fn_center[3 * fb + d]) return inf;
      if (s->fn_lm[2 * fa] != s->fn_lm[2 * fb] || s->fn_lm[2 * fa + 1] != s->fn_lm[2 * fb + 1]) return inf;
      const int pa = s->fn_prim_offset[fa], pb = s->fn_prim_offset[fb];
      const int na = s->fn_prim_offset[fa + 1] - pa;
      if (s->fn_prim_offset[fb + 1] - pb != na) return inf;
      for (int q = 0; q < na; ++q)
        if (s->prim_zeta[pa + q] != s->prim_zeta[pb + q] || s->prim_coeff[pa + q] != s->prim_coeff[pb + q])
          return inf;
      for (int k = 0; k < np; k += 2) {
        const double* ca = s->coeff + 2 * (size_t(fa) * np + k);  // (a re, a im) of column k
        const double* cb = s->coeff + 2 * (size_t(fb) * np + k);
        // partner column k+1: alpha = -conj(beta_k), beta = conj(alpha_k)
        dc = std::max({dc, std::fabs(ca[2] + cb[0]), std::fabs(ca[3] - cb[1]), std::fabs(cb[2] - ca[0]),
                       std::fabs(cb[3] + ca[1])});
      }
    }
  }
  return std::max(cmax > 0 ? dc / cmax : dc, emax > 0 ? de / emax : de);
}

// Basis groups of the MO transform and the coefficient matrix in DMMA B-fragment order
// B[mu/4][nf][lane] (lane: mu%4 = lane%4, real column = lane/4 of fragment nf).
//  general: one group per channel; per unit of 8 columns two fragments (re, im).
//  kramers: one group per channel pair (a, b) sharing a basis list; per unit of 8 even
//           columns 2j four fragments (a re, a im, b re, b im); odd columns follow exactly.
void build_groups(SpinorParams& sp, const mcmp2dev_system* s, const std::vector<int>& ch_off, bool kramers,
                  int ptf_max, std::vector<void*>& owned) {
  const int np = s->n_occ + s->n_vir;
  sp.ngroups = kramers ? s->ncomp / 2 : s->ncomp;
  std::vector<double> bfrag;
  long long chi_doubles = 0;
  sp.max_nf = 0;
  // groups ordered by decreasing basis size: mo_kernel's blockIdx.z = group, so the longest
  // tiles are dispatched first and the last wave holds the short ones
  std::vector<int> order(sp.ngroups);
  for (int g = 0; g < sp.ngroups; ++g) order[g] = g;
  auto size_of = [&](int g) { const int x = kramers ? 2 * g : g; return ch_off[x + 1] - ch_off[x]; };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return size_of(a) > size_of(b); });
  for (int g = 0; g < sp.ngroups; ++g) {
    const int src = order[g];
    const int xa = kramers ? 2 * src : src, xb = kramers ? 2 * src + 1 : -1;
    const int nfn = ch_off[xa + 1] - ch_off[xa], k4n = (nfn + 3) / 4;
    int units = kramers ? (np / 2 + 7) / 8 : (np + 7) / 8;
    if (!kramers) units += units & 1;  // warps take 4 fragments
    const int nf = units * (kramers ? 4 : 2);
    sp.grp_fn_off[g] = ch_off[xa];
    sp.grp_nfn[g] = nfn;
    sp.grp_k4[g] = k4n;
    sp.grp_nf[g] = nf;
    sp.grp_chan[2 * g] = xa;
    sp.grp_chan[2 * g + 1] = xb;
    sp.grp_chi_off[g] = chi_doubles;
    sp.grp_b_off[g] = (long long)bfrag.size();
    sp.max_nf = std::max(sp.max_nf, nf);
    sp.grp_nt[g] = (nf + 7) / 8;
    chi_doubles += (long long)ptf_max * k4n * 32;
    const size_t base = bfrag.size();
    // [nf / 8][k4][nf % 8][lane]: one k-slice of an 8-fragment n tile is contiguous
    bfrag.resize(base + size_t(sp.grp_nt[g]) * k4n * 8 * 32, 0.0);
    for (int k4 = 0; k4 < k4n; ++k4)
      for (int f = 0; f < nf; ++f)
        for (int lane = 0; lane < 32; ++lane) {
          const int mu = k4 * 4 + (lane & 3), r8 = lane >> 2;
          if (mu >= nfn) continue;
          double v = 0.0;
          if (!kramers) {
            const int col = (f >> 1) * 8 + r8, plane = f & 1;
            if (col < np) v = s->coeff[2 * (size_t(ch_off[xa] + mu) * np + col) + plane];
          } else {
            const int col = 2 * ((f >> 2) * 8 + r8), sub = f & 3;
            const int x = sub < 2 ? xa : xb, plane = sub & 1;
            if (col < np) v = s->coeff[2 * (size_t(ch_off[x] + mu) * np + col) + plane];
          }
          bfrag[base + ((size_t(f >> 3) * k4n + k4) * 8 + (f & 7)) * 32 + lane] = v;
        }
  }
  sp.bfrag = dupload(bfrag.data(), bfrag.size(), owned);
  sp.chi = dalloc<double>(size_t(chi_doubles), owned);
  ck(cudaMemset(sp.chi, 0, size_t(chi_doubles) * sizeof(double)), "memset chi");
}

void build(mcmp2dev_t* h, const mcmp2dev_system* s, int device, int max_walkers) {
  if (!s) throw ArgError("mcmp2dev_create: null system");
  if (s->ncomp != 1 && s->ncomp != 2 && s->ncomp != 4)
    throw ArgError("SpinorSet: component count must be 1, 2 or 4");
  if (s->n_occ < 0 || s->n_vir < 0 || s->n_occ + s->n_vir == 0)
    throw ArgError("SpinorSet: invalid occupied/virtual counts");
  if (max_walkers < 2) throw ArgError("init_ensemble: at least two electron-pair walkers");
  if (s->nsites < 1) throw ArgError("Molecule: at least one nucleus required");
  if (!(s->lambda > 0.0)) throw ArgError("TauSampler: lambda must be positive");
  h->device = device;
  ck(cudaSetDevice(device), "cudaSetDevice");
  {  // the side stream's kernels fill what the main stream's leave (lower priority)
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priority range");
    ck(cudaStreamCreateWithPriority(&h->stream, cudaStreamNonBlocking, hi), "cudaStreamCreate");
    ck(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, lo), "cudaStreamCreate");
  }
  ck(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming), "cudaEventCreate");
  ck(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming), "cudaEventCreate");
  ck(pair_kernel_setup(), "pair kernel attributes");
  ck(spinor_kernel_setup(), "spinor kernel attributes");
  ck(pair_kr_kernel_setup(), "pair_kr kernel attributes");
  ck(pair_kr_kernel_setup_qb1(), "pair_kr (QB 1) kernel attributes");
  ck(oz_kernel_setup(), "pair_oz kernel attributes");
  ck(pair_kr_kernel_setup_pw4(), "pair_kr (PW 4) kernel attributes");
  for (auto& e : h->ev) ck(cudaEventCreate(&e), "cudaEventCreate");
  for (auto& e : h->ev_oz) ck(cudaEventCreate(&e), "cudaEventCreate");

  h->ncomp = s->ncomp;
  h->n_occ = s->n_occ;
  h->n_vir = s->n_vir;
  h->n_p = s->n_occ + s->n_vir;
  h->ng = s->ng;
  h->lambda = s->lambda;
  h->w_direct = s->w_direct;
  h->w_exchange = s->w_exchange;
  h->estimator = s->estimator;
  // the INT8 V path is the default of the literal estimator, where its accuracy guard runs; the
  // opt-in physical estimator keeps the FP64 DMMA pair stage unless mcmp2dev_pair_path selects it
  h->oz = s->estimator == MCMP2DEV_ESTIMATOR_LITERAL;
  if (s->estimator != MCMP2DEV_ESTIMATOR_LITERAL && s->estimator != MCMP2DEV_ESTIMATOR_PHYSICAL)
    throw ArgError("mcmp2dev_create: unknown estimator");

  // ---- basis: flatten, dedupe exp(-zeta r^2) by (centre, zeta) ----
  std::vector<int> ch_off(s->ncomp + 1, 0);
  for (int x = 0; x < s->ncomp; ++x) {
    if (s->channel_count[x] < 1) throw ArgError("SpinorSet: empty basis list for a component");
    ch_off[x + 1] = ch_off[x] + s->channel_count[x];
  }
  const int nfunc = ch_off[s->ncomp];
  h->nfunc = nfunc;
  h->rows = nfunc;
  const int nprim = s->fn_prim_offset[nfunc];
  std::map<std::tuple<double, double, double, double>, int> uniq;
  std::vector<double> uc, uz;
  std::vector<int> prim_uniq(nprim);
  for (int f = 0; f < nfunc; ++f) {
    const int l = s->fn_lm[2 * f], mm = s->fn_lm[2 * f + 1];
    if (l < 0 || l > 3) throw ArgError("BasisFunction: l must be in [0,3]");
    if (mm < -l || mm > l) throw ArgError("BasisFunction: m out of range");
    if (s->fn_prim_offset[f + 1] <= s->fn_prim_offset[f])
      throw ArgError("BasisFunction: needs at least one primitive");
    for (int k = s->fn_prim_offset[f]; k < s->fn_prim_offset[f + 1]; ++k) {
      if (!(s->prim_zeta[k] > 0.0)) throw ArgError("BasisFunction: exponents must be strictly positive");
      const auto key = std::make_tuple(s->fn_center[3 * f], s->fn_center[3 * f + 1],
                                       s->fn_center[3 * f + 2], s->prim_zeta[k]);
      auto it = uniq.find(key);
      if (it == uniq.end()) {
        it = uniq.emplace(key, int(uz.size())).first;
        uc.insert(uc.end(), {s->fn_center[3 * f], s->fn_center[3 * f + 1], s->fn_center[3 * f + 2]});
        uz.push_back(s->prim_zeta[k]);
      }
      prim_uniq[k] = it->second;
    }
  }
  for (int p = 1; p < h->n_occ; ++p)
    if (s->energies[p] < s->energies[p - 1]) throw RtError("SpinorSet: occupied energies not ascending");
  for (int p = h->n_occ + 1; p < h->n_p; ++p)
    if (s->energies[p] < s->energies[p - 1]) throw RtError("SpinorSet: virtual energies not ascending");

  auto& o = h->owned;
  SpinorParams& sp = h->sp;
  sp.ncomp = s->ncomp;
  sp.fn_center = dupload(s->fn_center, size_t(3) * nfunc, o);
  sp.fn_lm = dupload(s->fn_lm, size_t(2) * nfunc, o);
  sp.fn_prim_off = dupload(s->fn_prim_offset, size_t(nfunc) + 1, o);
  sp.prim_coeff = dupload(s->prim_coeff, size_t(nprim), o);
  sp.prim_uniq = dupload(prim_uniq.data(), prim_uniq.size(), o);
  sp.nuniq = int(uz.size());
  sp.uniq_center = dupload(uc.data(), uc.size(), o);
  sp.uniq_zeta = dupload(uz.data(), uz.size(), o);
  h->kramers_dev = kramers_deviation(s, ch_off);
  h->kramers_eligible = h->kramers_dev <= kKramersTol;  // literal and physical epilogues both exist
  h->kramers = h->kramers_eligible;
  sp.n_occ = h->n_occ;
  sp.n_vir = h->n_vir;
  sp.n_p = h->n_p;
  // k-groups of 4 spinors; chunked per kind (PhiChunks), so O and V phases never share a stage
  h->Go = (h->n_occ + 3) / 4;
  h->Gv = (h->n_vir + 3) / 4;
  sp.Go = h->Go;
  sp.Gv = h->Gv;
  h->d_energies = dupload(s->energies, size_t(h->n_p), o);
  h->nens_cap = std::max(1, max_walkers / 16);  // batched ensembles hold >= 16 walkers each
  h->d_sw = dalloc<double>(size_t(h->n_p) * h->nens_cap, o);
  sp.sw = h->d_sw;

  h->sites.n = s->nsites;
  h->sites.pos = dupload(s->site_pos, size_t(3) * s->nsites, o);
  h->sites.prim = dupload(s->site_prim, size_t(4) * s->nsites, o);
  h->sites.zeta1 = dupload(s->site_zeta1, size_t(s->nsites), o);

  // ---- ensemble and work buffers ----
  h->mmax = max_walkers;
  h->nbmax = (max_walkers + WB - 1) / WB;
  h->npts_pad = 2 * WB * ((h->nbmax + 1) / 2 * 2);  // whole 16-walker Q rows for pair_kr tiles
  for (auto& b : h->buf) {
    b.mmax = h->nbmax * WB;
    b.w = dalloc<double>(size_t(9) * b.mmax, o);
    ck(cudaMemset(b.w, 0, sizeof(double) * 9 * b.mmax), "memset");
  }
  h->rbuf.mmax = h->nbmax * WB;
  h->rbuf.w = dalloc<double>(size_t(9) * h->rbuf.mmax, o);
  ck(cudaMemset(h->rbuf.w, 0, sizeof(double) * 9 * h->rbuf.mmax), "memset");
  h->d_state = dalloc<DevState>(h->nens_cap, o);
  ck(cudaMemset(h->d_state, 0, sizeof(DevState) * h->nens_cap), "memset state");
  DevState st{};
  st.sigma = 1.0;  // sampler.hpp:45
  st.error_idx = INT_MAX;
  st.spec_error_idx = INT_MAX;
  ck(scopy(h->stream, h->d_state, &st, sizeof st, cudaMemcpyHostToDevice), "state H2D");
  h->d_block_acc = dalloc<int>((max_walkers + 63) / 64 + 2, o);  // 64 walkers per walk CTA + tau CTA
  const size_t phi_doubles = size_t(h->Go + h->Gv) * h->npts_pad * 32;
  h->d_phi = dalloc<double>(phi_doubles, o);
  ck(cudaMemset(h->d_phi, 0, phi_doubles * sizeof(double)), "memset phi");
  sp.phi = h->d_phi;
  sp.npts_pad = h->npts_pad;
  h->d_hinv = dalloc<double>(size_t(h->npts_pad) / 2, o);
  ck(cudaMemset(h->d_hinv, 0, sizeof(double) * h->npts_pad / 2), "memset hinv");
  sp.hinv = h->d_hinv;
  // MO-transform operands: basis groups, B fragments of C, A-fragment buffer for chi
  const int ptf_max = (h->npts_pad + 255) / 256 * 32;  // point fragments, padded to any mo_kernel tile (<= 256 points)
  {
    int sms = 0;
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "SM count");
    sp.mo_slots = sms * mo_ctas_per_sm();
    h->sms = sms;
  }
  sp.st = h->d_state;
  h->sp_kr = sp;
  build_groups(h->sp, s, ch_off, false, ptf_max, o);
  if (h->kramers_eligible) build_groups(h->sp_kr, s, ch_off, true, ptf_max, o);
  // per-CTA partials: the grid of any pair kernel is at most its tile count
  const size_t ntiles = std::max({size_t(h->nbmax) * (h->nbmax + 1) / 2, size_t(pair_kr_tiles(h->nbmax)),
                                  size_t(pair_kr_tiles_qb1(h->nbmax))});
  // (oz_vgemm_kernel: one CTA per SM, 8 doubles each)
  h->d_partials = dalloc<double>(std::max(ntiles * 4, size_t(h->sms) * 8), o);
  h->d_steps = dalloc<double>(size_t(kChunk) * kStepDoubles, o);
  h->d_gsteps = dalloc<double>(size_t(kGraphSteps) * kStepDoubles, o);
  ck(cudaMemset(h->d_steps, 0, sizeof(double) * kChunk * kStepDoubles), "memset steps");
  ck(cudaMemset(h->d_gsteps, 0, sizeof(double) * kGraphSteps * kStepDoubles), "memset steps");
  h->d_replay = dalloc<double>(size_t(h->mmax) * 8, o);
  ck(cudaMallocHost(&h->h_steps, sizeof(double) * kChunk * kStepDoubles), "cudaMallocHost");
  ck(cudaMallocHost(&h->h_replay, sizeof(double) * h->mmax * 8), "cudaMallocHost");
  ck(cudaDeviceSynchronize(), "setup sync");
}

void require_ensemble(mcmp2dev_t* h) {
  if (!h->have_ensemble) throw ArgError("mcmp2dev: no walker ensemble (call init_ensemble or set_ensemble)");
}

}  // namespace

extern "C" {

int mcmp2dev_abi_version(void) { return MCMP2DEV_ABI_VERSION; }

const char* mcmp2dev_last_error(const mcmp2dev_t* h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

int mcmp2dev_create(const mcmp2dev_system* sys, int device, int max_walkers, mcmp2dev_t** out) {
  if (!out) {
    g_create_error = "mcmp2dev_create: null output pointer";
    return MCMP2DEV_INVALID_ARGUMENT;
  }
  *out = nullptr;
  auto* h = new mcmp2dev_handle();
  const int rc = guard(nullptr, [&] { build(h, sys, device, max_walkers); });
  if (rc != MCMP2DEV_OK) {
    mcmp2dev_destroy(h);
    return rc;
  }
  *out = h;
  return MCMP2DEV_OK;
}

int mcmp2dev_destroy(mcmp2dev_t* h) {
  if (!h) return MCMP2DEV_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->owned) cudaFree(p);
  if (h->h_steps) cudaFreeHost(h->h_steps);
  if (h->h_replay) cudaFreeHost(h->h_replay);
  if (h->d_bpart) cudaFree(h->d_bpart);
  h->oz_free();
  if (h->d_bsteps) cudaFree(h->d_bsteps);
  if (h->h_bsteps) cudaFreeHost(h->h_bsteps);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->ev_oz)
    if (e) cudaEventDestroy(e);
  for (auto& g : h->graphs)
    if (g) cudaGraphExecDestroy(g);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return MCMP2DEV_OK;
}

int mcmp2dev_init_ensemble(mcmp2dev_t* h, int m, uint64_t seed, uint32_t stream) {
  return guard(h, [&] {
    if (m < 2) throw ArgError("init_ensemble: at least two electron-pair walkers");
    if (m > h->mmax) throw ArgError("init_ensemble: more walkers than the handle was sized for");
    h->m = m;
    h->nens = 1;
    h->k0 = uint32_t(seed);
    h->k1 = uint32_t(seed >> 32);
    h->rstream = stream;
    DevState st{};
    st.pos = 0;
    st.sigma = 1.0;  // sampler.hpp:45
    st.error_idx = INT_MAX;
    st.spec_error_idx = INT_MAX;
    ck(cudaMemcpyAsync(h->d_state, &st, sizeof st, cudaMemcpyHostToDevice, h->stream), "state H2D");
    launch_walk(h->walk_params(WALK_INIT, 0, 0), h->stream);
    h->cur ^= 1;
    ck(cudaGetLastError(), "walk launch");
    ck(cudaStreamSynchronize(h->stream), "stream sync");
    h->have_ensemble = true;
  });
}

int mcmp2dev_set_sigma_step(mcmp2dev_t* h, double sigma) {
  return guard(h, [&] { h->each_state([&](DevState& st) { st.sigma = sigma; }); });
}

int mcmp2dev_burn_in(mcmp2dev_t* h, long n_burn, int adapt) {
  return guard(h, [&] {
    require_ensemble(h);
    h->each_state([](DevState& st) { st.win_acc = st.win_prop = 0; });
    for (long s = 1; s <= n_burn; ++s) {
      launch_walk(h->walk_params(WALK_BURN, s, adapt), h->stream);
      h->cur ^= 1;
    }
    ck(cudaGetLastError(), "walk launch");
    h->each_state([](DevState& st) {
      st.proposed = st.accepted = 0;  // sampler.cpp:92
      st.win_acc = st.win_prop = 0;
    });
  });
}

int mcmp2dev_set_ensemble(mcmp2dev_t* h, const mcmp2dev_ensemble* e) {
  return guard(h, [&] {
    if (!e || !e->walkers) throw ArgError("set_ensemble: null ensemble");
    if (e->m < 2) throw RtError("checkpoint: malformed ensemble record");
    if (e->m > h->mmax) throw ArgError("set_ensemble: more walkers than the handle was sized for");
    // stream position of PhiloxRng state (rng.cpp:46-51, :83-94)
    if (e->rng_counter[2] != 0) throw ArgError("set_ensemble: rng counter beyond 2^64 blocks");
    const uint64_t B = uint64_t(e->rng_counter[0]) | (uint64_t(e->rng_counter[1]) << 32);
    uint64_t pos;
    if (e->rng_idx >= 4) pos = 4 * B;
    else {
      if (B == 0) throw ArgError("set_ensemble: partially consumed block before the first refill");
      pos = 4 * (B - 1) + e->rng_idx;
    }
    h->m = e->m;
    h->nens = 1;
    h->k0 = e->rng_key[0];
    h->k1 = e->rng_key[1];
    h->rstream = e->rng_counter[3];
    std::vector<double> soa(size_t(9) * h->buf[0].mmax, 0.0);
    for (int p = 0; p < e->m; ++p)
      for (int k = 0; k < 9; ++k) soa[size_t(k) * h->buf[0].mmax + p] = e->walkers[size_t(p) * 9 + k];
    ck(scopy(h->stream, h->buf[h->cur].w, soa.data(), soa.size() * sizeof(double), cudaMemcpyHostToDevice),
       "walkers H2D");
    DevState st{};
    st.pos = pos;
    st.sigma = e->sigma_step;
    st.proposed = e->proposed;
    st.accepted = e->accepted;
    st.error_idx = INT_MAX;
    st.spec_error_idx = INT_MAX;
    ck(scopy(h->stream, h->d_state, &st, sizeof st, cudaMemcpyHostToDevice), "state H2D");
    h->have_ensemble = true;
  });
}

int mcmp2dev_get_ensemble(mcmp2dev_t* h, mcmp2dev_ensemble* e) {
  return guard(h, [&] {
    require_ensemble(h);
    if (!e || !e->walkers) throw ArgError("get_ensemble: null ensemble");
    if (h->nens > 1) throw ArgError("get_ensemble: batched handle (use mcmp2dev_get_ensemble_at)");
    ck(cudaStreamSynchronize(h->stream), "stream sync");
    DevState st;
    ck(scopy(h->stream, &st, h->d_state, sizeof st, cudaMemcpyDeviceToHost), "state D2H");
    std::vector<double> soa(size_t(9) * h->buf[0].mmax);
    ck(scopy(h->stream, soa.data(), h->buf[h->cur].w, soa.size() * sizeof(double), cudaMemcpyDeviceToHost),
       "walkers D2H");
    e->m = h->m;
    for (int p = 0; p < h->m; ++p)
      for (int k = 0; k < 9; ++k) e->walkers[size_t(p) * 9 + k] = soa[size_t(k) * h->buf[0].mmax + p];
    e->sigma_step = st.sigma;
    e->proposed = st.proposed;
    e->accepted = st.accepted;
    e->rng_key[0] = h->k0;
    e->rng_key[1] = h->k1;
    const uint64_t pos = st.pos;
    uint64_t B;
    if (pos % 4 == 0) {
      B = pos / 4;
      e->rng_idx = 4;
    } else {
      B = pos / 4 + 1;
      e->rng_idx = uint32_t(pos % 4);
    }
    e->rng_counter[0] = uint32_t(B);
    e->rng_counter[1] = uint32_t(B >> 32);
    e->rng_counter[2] = 0;
    e->rng_counter[3] = h->rstream;
  });
}

namespace {
// advance of a batched handle: chunks of kGraphSteps steps (one graph replay when possible),
// results [nsteps][nens]
void advance_batched(mcmp2dev_t* h, long nsteps, int nactive, double* values, double* imags) {
  const int ne = h->nens;
  for (long done = 0; done < nsteps;) {
    const long n = std::min<long>(kGraphSteps, nsteps - done);
    if (!h->prof && n == kGraphSteps && nactive == ne) {
      ck(cudaGraphLaunch(h->ensure_graph(), h->stream), "cudaGraphLaunch");
    } else {
      for (long s = 0; s < n; ++s) {
        if (h->prof) ck(cudaEventRecord(h->ev[0], h->stream), "event");
        WalkParams P = h->walk_params(WALK_PRODUCTION, 0, 0);
        P.nactive = nactive;
        launch_walk(P, h->stream);
        h->cur ^= 1;
        h->launch_estimate(h->buf[h->cur], h->m, h->d_bsteps + size_t(6) * ne * s, ne);
      }
    }
    if (values || imags)
      ck(cudaMemcpyAsync(h->h_bsteps, h->d_bsteps, sizeof(double) * 6 * ne * n, cudaMemcpyDeviceToHost, h->stream),
         "steps D2H");
    h->check_state_errors();  // synchronises
    for (long s = 0; s < n; ++s)
      for (int e = 0; e < ne; ++e) {
        const double* r = h->h_bsteps + (size_t(s) * ne + e) * 6;
        if (values) values[size_t(done + s) * ne + e] = r[0];
        if (imags) imags[size_t(done + s) * ne + e] = r[1];
      }
    done += n;
  }
}
}  // namespace

namespace {
// the guard's bookkeeping over one step record (kStepDoubles) of the INT8 path
void guard_account(mcmp2dev_t* h, const double* r) {
  if (r[10] == 0.0) return;
  ++h->guard_steps;
  if (r[11] == 2.0) {
    ++h->guard_dmma;
    return;
  }
  if (r[11] == 1.0) ++h->guard_refined;
  const double d = std::fabs(r[2]), x = std::fabs(r[4]), v = std::fabs(r[2] + r[4]);
  double est = 0.0;
  if (d > 0) est = std::max(est, r[6] / d);
  if (x > 0) est = std::max(est, r[7] / x);
  if (v > 0) est = std::max(est, std::sqrt(r[6] * r[6] + r[7] * r[7]) / v);
  h->guard_max_est = std::max(h->guard_max_est, est);
}

void fill_ex(const double* r, mcmp2dev_step_ex* o) {
  o->value = r[0];
  o->imag = r[1];
  o->direct_re = r[2];
  o->direct_im = r[3];
  o->exchange_re = r[4];
  o->exchange_im = r[5];
  o->est_err_direct = r[6];
  o->est_err_exchange = r[7];
  o->abs_direct = r[8];
  o->abs_exchange = r[9];
  o->int8_v = r[10] != 0.0 ? 1 : 0;
  o->fallback = int(r[11]);
}

// single-ensemble advance: chunks of kChunk steps, whole graphs of kGraphSteps where possible
void advance_single(mcmp2dev_t* h, long nsteps, double* values, double* imags, mcmp2dev_step_ex* ex) {
  h->ensure_oz(h->m);
  const bool oz = h->oz_active(h->m, 1);
  constexpr int R = kStepDoubles;
  long done = 0;
  while (done < nsteps) {
    const long n = std::min<long>(kChunk, nsteps - done);
    long s = 0;
    // whole blocks of kGraphSteps steps replay one captured CUDA graph
    if (!h->prof && n >= kGraphSteps) {
      cudaGraphExec_t graph = h->ensure_graph();
      for (; s + kGraphSteps <= n; s += kGraphSteps) {
        ck(cudaGraphLaunch(graph, h->stream), "cudaGraphLaunch");
        ck(cudaMemcpyAsync(h->h_steps + R * s, h->d_gsteps, sizeof(double) * R * kGraphSteps,
                           cudaMemcpyDeviceToHost, h->stream),
           "steps D2H");
      }
    }
    const long s0 = s;
    for (; s < n; ++s) {
      if (h->prof) ck(cudaEventRecord(h->ev[0], h->stream), "event");
      launch_walk(h->walk_params(WALK_PRODUCTION, 0, 0), h->stream);
      h->cur ^= 1;
      h->launch_estimate(h->buf[h->cur], h->m, h->d_steps + R * s);
    }
    if (n > s0)
      ck(cudaMemcpyAsync(h->h_steps + R * s0, h->d_steps + R * s0, sizeof(double) * R * (n - s0),
                         cudaMemcpyDeviceToHost, h->stream),
         "steps D2H");
    h->check_state_errors();  // synchronises
    for (long k = 0; k < n; ++k) {
      double* r = h->h_steps + R * k;
      if (!oz) std::fill(r + 6, r + R, 0.0);  // the guard fields exist on the INT8 path only
      guard_account(h, r);
      if (values) values[done + k] = r[0];
      if (imags) imags[done + k] = r[1];
      if (ex) fill_ex(r, ex + done + k);
    }
    done += n;
  }
}
}  // namespace

int mcmp2dev_advance(mcmp2dev_t* h, long nsteps, double* values, double* imags) {
  return guard(h, [&] {
    require_ensemble(h);
    if (nsteps < 0) throw ArgError("advance: negative step count");
    if (h->nens > 1) {
      advance_batched(h, nsteps, h->nens, values, imags);
      return;
    }
    advance_single(h, nsteps, values, imags, nullptr);
  });
}

int mcmp2dev_advance_ex(mcmp2dev_t* h, long nsteps, mcmp2dev_step_ex* out) {
  return guard(h, [&] {
    require_ensemble(h);
    if (nsteps < 0) throw ArgError("advance: negative step count");
    if (h->nens > 1) throw ArgError("advance_ex: batched handle (use mcmp2dev_advance_batch)");
    if (!out && nsteps > 0) throw ArgError("advance_ex: null output");
    advance_single(h, nsteps, nullptr, nullptr, out);
  });
}

namespace {
void replay_steps(mcmp2dev_t* h, int m, long nsteps, const double* walkers, const double* tau, mcmp2dev_step* out,
                  mcmp2dev_step_ex* ex) {
  if (m < 2) throw ArgError("replay: at least two electron-pair walkers");
  if (m > h->mmax) throw ArgError("replay: more walkers than the handle was sized for");
  h->ensure_oz(m);
  const bool oz = h->oz_active(m, 1);
  for (long st = 0; st < nsteps; ++st) {
    if (tau[st] < 0) throw ArgError("sample_term: tau must be non-negative");
    std::memcpy(h->h_replay, walkers + size_t(st) * m * 8, sizeof(double) * 8 * m);
    ck(cudaMemcpyAsync(h->d_replay, h->h_replay, sizeof(double) * 8 * m, cudaMemcpyHostToDevice, h->stream),
       "replay H2D");
    if (h->prof) ck(cudaEventRecord(h->ev[0], h->stream), "event");
    WalkParams P = h->walk_params(WALK_PRODUCTION, 0, 0);
    P.out = h->rbuf;
    P.m = m;
    launch_replay_load(P, h->d_replay, tau[st], h->stream);
    h->launch_estimate(h->rbuf, m, h->d_steps);
    ck(cudaMemcpyAsync(h->h_steps, h->d_steps, sizeof(double) * kStepDoubles, cudaMemcpyDeviceToHost, h->stream),
       "steps D2H");
    h->check_state_errors();
    double* r = h->h_steps;
    if (!oz) std::fill(r + 6, r + kStepDoubles, 0.0);
    guard_account(h, r);
    if (out) {
      out[st].value = r[0];
      out[st].imag = r[1];
      out[st].direct_re = r[2];
      out[st].direct_im = r[3];
      out[st].exchange_re = r[4];
      out[st].exchange_im = r[5];
    }
    if (ex) fill_ex(r, ex + st);
  }
}
}  // namespace

int mcmp2dev_replay(mcmp2dev_t* h, int m, long nsteps, const double* walkers, const double* tau,
                    mcmp2dev_step* out) {
  return guard(h, [&] { replay_steps(h, m, nsteps, walkers, tau, out, nullptr); });
}

int mcmp2dev_replay_ex(mcmp2dev_t* h, int m, long nsteps, const double* walkers, const double* tau,
                       mcmp2dev_step_ex* out) {
  return guard(h, [&] { replay_steps(h, m, nsteps, walkers, tau, nullptr, out); });
}

int mcmp2dev_guard(mcmp2dev_t* h, double tol, double* previous) {
  return guard(h, [&] {
    if (previous) *previous = h->guard_tol;
    if (!(tol == tol)) return;  // NaN: query only
    h->guard_tol = tol > 0.0 ? tol : 0.0;  // a different value re-captures the graphs (GraphKey)
  });
}

int mcmp2dev_guard_stats(mcmp2dev_t* h, double* out5) {
  return guard(h, [&] {
    if (!out5) throw ArgError("guard_stats: null output");
    out5[0] = double(h->guard_steps);
    out5[1] = double(h->guard_refined);
    out5[2] = double(h->guard_dmma);
    out5[3] = h->guard_max_est;
    out5[4] = h->guard_tol;
    h->guard_steps = h->guard_refined = h->guard_dmma = 0;
    h->guard_max_est = 0.0;
  });
}

int mcmp2dev_profile(mcmp2dev_t* h, int enable, int reset, double* out) {
  return guard(h, [&] {
    if (out)
      for (int i = 0; i < 4; ++i) {
        out[i] = h->prof_ms[i];
        out[4 + i] = h->prof_n[i];
      }
    if (reset)
      for (int i = 0; i < 4; ++i) h->prof_ms[i] = h->prof_n[i] = 0;
      for (double& x : h->prof_oz) x = 0;
    h->prof = enable != 0;
  });
}

int mcmp2dev_work(mcmp2dev_t* h, double* pair_flop, double* spinor_flop, double* phi_bytes) {
  return guard(h, [&] {
    const double m = h->m, nc = h->ncomp, ne = h->nens;  // per step, all ensembles of the handle
    const double fpair = 8.0 * nc * nc * (2.0 * h->n_occ + 4.0 * h->n_vir) + 4.0 * 8.0 * nc * nc;
    if (pair_flop) *pair_flop = ne * 0.5 * m * (m - 1) * fpair;
    if (spinor_flop) *spinor_flop = ne * 2.0 * m * 4.0 * h->rows * h->n_p;
    if (phi_bytes) *phi_bytes = ne * 2.0 * m * nc * h->n_p * 16.0;
  });
}

void* mcmp2dev_stream(mcmp2dev_t* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

int mcmp2dev_prepare(mcmp2dev_t* h) {
  return guard(h, [&] {
    require_ensemble(h);
    h->ensure_oz(h->m);
    for (int k = 0; k < 2; ++k) {  // both walker-buffer parities; nothing is executed
      h->ensure_graph();
      h->cur ^= 1;
    }
  });
}

int mcmp2dev_work_executed(mcmp2dev_t* h, double* pair_dmma_flop) {
  return guard(h, [&] {
    const int nb = (h->m + WB - 1) / WB;
    const double ntiles = h->kramers ? (h->kr_qb1(h->m, h->nens) ? pair_kr_block_tiles_qb1(nb) : pair_kr_block_tiles(nb))
                                     : 0.5 * nb * (nb + 1);
    // DMMAs per WB x WB block per k-group (all warps): O phase and V phase, 3 per complex product
    const double per_o = h->kramers ? 4 * 2 * 2 * 3 : 8 * 2 * 2 * 3;
    const double per_v = h->oz_active(h->m, h->nens) ? 0.0 : h->kramers ? 4 * 2 * 4 * 3 : 8 * 2 * 4 * 3;
    *pair_dmma_flop = h->nens * ntiles * 512.0 * (h->Go * per_o + h->Gv * per_v);
  });
}

int mcmp2dev_init_batch(mcmp2dev_t* h, int nens, int m, uint64_t seed, uint32_t stream0) {
  return guard(h, [&] {
    if (nens < 1) throw ArgError("init_batch: at least one ensemble");
    if (m < 2) throw ArgError("init_ensemble: at least two electron-pair walkers");
    if (nens > 1 && m % 16) throw ArgError("init_batch: batched ensembles need a multiple of 16 walkers each");
    if (nens > 1 && m > kBatchMaxWalkers)  // walk_batch_kernel: one CTA of 2m + 32 threads per ensemble
      throw ArgError("init_batch: batched ensembles hold at most " + std::to_string(kBatchMaxWalkers) + " walkers each");
    if (size_t(nens) * m > size_t(h->mmax)) throw ArgError("init_batch: more walkers than the handle was sized for");
    if (nens > h->nens_cap) throw ArgError("init_batch: more ensembles than the handle was sized for");
    h->m = m;
    h->nens = nens;
    h->k0 = uint32_t(seed);
    h->k1 = uint32_t(seed >> 32);
    h->rstream = stream0;
    if (nens > 1) {
      const int nb = (m + WB - 1) / WB;  // per-tile partials of either pair kernel
      const size_t part = size_t(nens) * std::max({size_t(pair_kr_tiles(nb)) * pair_kr_consumers() * 2,
                                                   size_t(pair_kr_tiles_qb1(nb)) * pair_kr_consumers_qb1() * 2,
                                                   size_t(nb) * (nb + 1) / 2 * pair_consumers() * 4});
      if (part > h->bpart_cap) {
        h->drop_graphs();
        if (h->d_bpart) cudaFree(h->d_bpart);
        h->d_bpart = nullptr;
        ck(cudaMalloc(&h->d_bpart, part * sizeof(double)), "cudaMalloc");
        h->bpart_cap = part;
      }
      const size_t steps = size_t(kGraphSteps) * nens * 6;
      if (steps > h->bsteps_cap) {
        h->drop_graphs();
        if (h->d_bsteps) cudaFree(h->d_bsteps);
        if (h->h_bsteps) cudaFreeHost(h->h_bsteps);
        h->d_bsteps = nullptr;
        h->h_bsteps = nullptr;
        ck(cudaMalloc(&h->d_bsteps, steps * sizeof(double)), "cudaMalloc");
        ck(cudaMallocHost(&h->h_bsteps, steps * sizeof(double)), "cudaMallocHost");
        h->bsteps_cap = steps;
      }
    }
    std::vector<DevState> all(nens);
    for (DevState& st : all) {
      st = DevState{};
      st.sigma = 1.0;  // sampler.hpp:45
      st.error_idx = INT_MAX;
      st.spec_error_idx = INT_MAX;
    }
    ck(cudaMemcpyAsync(h->d_state, all.data(), sizeof(DevState) * nens, cudaMemcpyHostToDevice, h->stream),
       "state H2D");
    launch_walk(h->walk_params(WALK_INIT, 0, 0), h->stream);
    h->cur ^= 1;
    ck(cudaGetLastError(), "walk launch");
    ck(cudaStreamSynchronize(h->stream), "stream sync");
    h->have_ensemble = true;
  });
}

int mcmp2dev_batch_size(const mcmp2dev_t* h) { return h ? h->nens : 0; }

int mcmp2dev_advance_batch(mcmp2dev_t* h, long nsteps, int nactive, double* values, double* imags) {
  if (h && h->nens == 1 && nactive == 1) return mcmp2dev_advance(h, nsteps, values, imags);
  return guard(h, [&] {
    require_ensemble(h);
    if (nsteps < 0) throw ArgError("advance: negative step count");
    if (nactive < 1 || nactive > h->nens) throw ArgError("advance_batch: active ensembles out of range");
    advance_batched(h, nsteps, nactive, values, imags);
  });
}

int mcmp2dev_get_ensemble_at(mcmp2dev_t* h, int ens, mcmp2dev_ensemble* e) {
  return guard(h, [&] {
    require_ensemble(h);
    if (!e || !e->walkers) throw ArgError("get_ensemble: null ensemble");
    if (ens < 0 || ens >= h->nens) throw ArgError("get_ensemble_at: no such ensemble");
    DevState st;
    ck(scopy(h->stream, &st, h->d_state + ens, sizeof st, cudaMemcpyDeviceToHost), "state D2H");
    const int m = h->m, mmax = h->buf[0].mmax;
    std::vector<double> rows(size_t(9) * m);
    for (int k = 0; k < 9; ++k)
      ck(cudaMemcpyAsync(rows.data() + size_t(k) * m, h->buf[h->cur].w + size_t(k) * mmax + size_t(ens) * m,
                         sizeof(double) * m, cudaMemcpyDeviceToHost, h->stream),
         "walkers D2H");
    ck(cudaStreamSynchronize(h->stream), "stream sync");
    e->m = m;
    for (int p = 0; p < m; ++p)
      for (int k = 0; k < 9; ++k) e->walkers[size_t(p) * 9 + k] = rows[size_t(k) * m + p];
    e->sigma_step = st.sigma;
    e->proposed = st.proposed;
    e->accepted = st.accepted;
    e->rng_key[0] = h->k0;
    e->rng_key[1] = h->k1;
    const uint64_t pos = st.pos;  // PhiloxRng state at stream position pos (rng.cpp:46-51, :83-94)
    const uint64_t B = pos % 4 == 0 ? pos / 4 : pos / 4 + 1;
    e->rng_idx = pos % 4 == 0 ? 4 : uint32_t(pos % 4);
    e->rng_counter[0] = uint32_t(B);
    e->rng_counter[1] = uint32_t(B >> 32);
    e->rng_counter[2] = 0;
    e->rng_counter[3] = h->rstream + uint32_t(ens);
  });
}

int mcmp2dev_get_ensembles(mcmp2dev_t* h, mcmp2dev_ensemble* es) {
  return guard(h, [&] {
    require_ensemble(h);
    if (!es) throw ArgError("get_ensembles: null array");
    const int ne = h->nens, m = h->m, mmax = h->buf[0].mmax;
    std::vector<DevState> all(ne);
    std::vector<double> soa(size_t(9) * mmax);
    ck(cudaMemcpyAsync(all.data(), h->d_state, sizeof(DevState) * ne, cudaMemcpyDeviceToHost, h->stream), "state D2H");
    ck(cudaMemcpyAsync(soa.data(), h->buf[h->cur].w, soa.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream),
       "walkers D2H");
    ck(cudaStreamSynchronize(h->stream), "stream sync");
    for (int k = 0; k < ne; ++k) {
      mcmp2dev_ensemble* e = es + k;
      if (!e->walkers) throw ArgError("get_ensembles: null walker buffer");
      e->m = m;
      for (int p = 0; p < m; ++p)
        for (int c = 0; c < 9; ++c) e->walkers[size_t(p) * 9 + c] = soa[size_t(c) * mmax + size_t(k) * m + p];
      const DevState& st = all[k];
      e->sigma_step = st.sigma;
      e->proposed = st.proposed;
      e->accepted = st.accepted;
      e->rng_key[0] = h->k0;
      e->rng_key[1] = h->k1;
      const uint64_t B = st.pos % 4 == 0 ? st.pos / 4 : st.pos / 4 + 1;
      e->rng_idx = st.pos % 4 == 0 ? 4 : uint32_t(st.pos % 4);
      e->rng_counter[0] = uint32_t(B);
      e->rng_counter[1] = uint32_t(B >> 32);
      e->rng_counter[2] = 0;
      e->rng_counter[3] = h->rstream + uint32_t(k);
    }
  });
}

int mcmp2dev_set_ensembles(mcmp2dev_t* h, const mcmp2dev_ensemble* es) {
  return guard(h, [&] {
    require_ensemble(h);
    if (!es) throw ArgError("set_ensembles: null array");
    const int ne = h->nens, m = h->m, mmax = h->buf[0].mmax;
    std::vector<DevState> all(ne);
    std::vector<double> soa(size_t(9) * mmax, 0.0);
    for (int k = 0; k < ne; ++k) {
      const mcmp2dev_ensemble* e = es + k;
      if (!e->walkers) throw ArgError("set_ensemble: null ensemble");
      if (e->m != m) throw ArgError("set_ensemble_at: every ensemble of a batch has the same walker count");
      if (e->rng_key[0] != h->k0 || e->rng_key[1] != h->k1 || e->rng_counter[3] != h->rstream + uint32_t(k))
        throw ArgError("set_ensemble_at: ensemble e of a batch runs on the batch seed and stream stream0 + e");
      if (e->rng_counter[2] != 0) throw ArgError("set_ensemble: rng counter beyond 2^64 blocks");
      const uint64_t B = uint64_t(e->rng_counter[0]) | (uint64_t(e->rng_counter[1]) << 32);
      uint64_t pos;
      if (e->rng_idx >= 4) pos = 4 * B;
      else {
        if (B == 0) throw ArgError("set_ensemble: partially consumed block before the first refill");
        pos = 4 * (B - 1) + e->rng_idx;
      }
      for (int p = 0; p < m; ++p)
        for (int c = 0; c < 9; ++c) soa[size_t(c) * mmax + size_t(k) * m + p] = e->walkers[size_t(p) * 9 + c];
      DevState& st = all[k];
      st = DevState{};
      st.pos = pos;
      st.sigma = e->sigma_step;
      st.proposed = e->proposed;
      st.accepted = e->accepted;
      st.error_idx = INT_MAX;
      st.spec_error_idx = INT_MAX;
    }
    ck(cudaMemcpyAsync(h->buf[h->cur].w, soa.data(), soa.size() * sizeof(double), cudaMemcpyHostToDevice, h->stream),
       "walkers H2D");
    ck(scopy(h->stream, h->d_state, all.data(), sizeof(DevState) * ne, cudaMemcpyHostToDevice), "state H2D");
  });
}

int mcmp2dev_set_ensemble_at(mcmp2dev_t* h, int ens, const mcmp2dev_ensemble* e) {
  return guard(h, [&] {
    require_ensemble(h);
    if (!e || !e->walkers) throw ArgError("set_ensemble: null ensemble");
    if (ens < 0 || ens >= h->nens) throw ArgError("set_ensemble_at: no such ensemble");
    if (e->m != h->m) throw ArgError("set_ensemble_at: every ensemble of a batch has the same walker count");
    if (e->rng_key[0] != h->k0 || e->rng_key[1] != h->k1 || e->rng_counter[3] != h->rstream + uint32_t(ens))
      throw ArgError("set_ensemble_at: ensemble e of a batch runs on the batch seed and stream stream0 + e");
    if (e->rng_counter[2] != 0) throw ArgError("set_ensemble: rng counter beyond 2^64 blocks");
    const uint64_t B = uint64_t(e->rng_counter[0]) | (uint64_t(e->rng_counter[1]) << 32);
    uint64_t pos;
    if (e->rng_idx >= 4) pos = 4 * B;
    else {
      if (B == 0) throw ArgError("set_ensemble: partially consumed block before the first refill");
      pos = 4 * (B - 1) + e->rng_idx;
    }
    const int m = h->m, mmax = h->buf[0].mmax;
    std::vector<double> rows(size_t(9) * m);
    for (int p = 0; p < m; ++p)
      for (int k = 0; k < 9; ++k) rows[size_t(k) * m + p] = e->walkers[size_t(p) * 9 + k];
    for (int k = 0; k < 9; ++k)
      ck(cudaMemcpyAsync(h->buf[h->cur].w + size_t(k) * mmax + size_t(ens) * m, rows.data() + size_t(k) * m,
                         sizeof(double) * m, cudaMemcpyHostToDevice, h->stream),
         "walkers H2D");
    DevState st{};
    st.pos = pos;
    st.sigma = e->sigma_step;
    st.proposed = e->proposed;
    st.accepted = e->accepted;
    st.error_idx = INT_MAX;
    st.spec_error_idx = INT_MAX;
    ck(scopy(h->stream, h->d_state + ens, &st, sizeof st, cudaMemcpyHostToDevice), "state H2D");
  });
}

int mcmp2dev_kramers_deviation(const mcmp2dev_t* h, double* deviation) {
  if (!h || !deviation) return MCMP2DEV_INVALID_ARGUMENT;
  *deviation = h->kramers_dev;
  return MCMP2DEV_OK;
}

int mcmp2dev_kramers(mcmp2dev_t* h, int mode) {
  if (!h) return -1;
  if (mode == 0) h->kramers = false;
  if (mode == 1) h->kramers = h->kramers_eligible;
  return h->kramers ? 1 : 0;
}

int mcmp2dev_profile_pair(mcmp2dev_t* h, double* out) {
  return guard(h, [&] {
    for (int i = 0; i < 4; ++i) out[i] = h->prof_oz[i];
    out[4] = h->oz_ops;
    out[5] = h->prof_oz[4];
  });
}

int mcmp2dev_pair_path(mcmp2dev_t* h, int mode) {
  if (!h) return -1;
  if (mode == 0) h->oz = false, h->oz_forced = false;
  if (mode == 1) h->oz = true, h->oz_forced = true;
  return h->oz && h->kramers && h->n_vir > 0 && h->n_vir <= 512 &&
                 (h->oz_forced || h->n_vir > mcmp2dev_handle::kOzAutoMinVir)
             ? 1
             : 0;
}

int mcmp2dev_oz_truncation(mcmp2dev_t* h, int mode) {
  if (!h) return -1;
  if (mode == 0) h->oz_trunc = false;
  if (mode == 1) h->oz_trunc = true, h->oz_trunc_slices = true;
  if (mode == 2) h->oz_trunc = true, h->oz_trunc_slices = false;
  return h->oz_trunc ? (h->oz_trunc_slices ? 1 : 2) : 0;
}

int mcmp2dev_oz_overlap(mcmp2dev_t* h, int mode) {
  if (!h) return -1;
  if (mode == 0) h->oz_overlap = false;
  if (mode == 1) h->oz_overlap = true;
  return h->oz_overlap ? 1 : 0;
}

int mcmp2dev_oz_ksteps(mcmp2dev_t* h, double* out2) {
  return guard(h, [&] {
    out2[0] = out2[1] = 0.0;
    if (!h->d_ks_exec) return;
    unsigned long long n = 0;
    ck(cudaStreamSynchronize(h->stream), "stream sync");
    ck(cudaMemcpy(&n, h->d_ks_exec, sizeof n, cudaMemcpyDeviceToHost), "k-step counter D2H");
    out2[0] = double(n) / 21.0;  // products -> k-steps (a partly empty k-step counts its share)
    out2[1] = h->oz_ks_full;
  });
}

int mcmp2dev_synchronize(mcmp2dev_t* h) {
  return guard(h, [&] { ck(cudaStreamSynchronize(h->stream), "stream sync"); });
}

}  // extern "C"
