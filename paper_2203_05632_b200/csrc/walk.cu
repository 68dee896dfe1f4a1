// walk.cu — Metropolis walker-pair update, ensemble initialisation and the tau draw
// (reference proj/core/src/sampler.cpp:21-93, weights.cpp:92-111, driver.cpp:444-445).
//
// Compiled with --fmad=false so that the proposal/weight arithmetic rounds like the
// reference's (non-contracted) C++ and device chains track the CPU chain.
//
// RNG: the reference consumes ONE sequential Philox stream per worker: 18 u32 per pair
// proposal (two gaussian3 = 2 x 4 uniforms x 2 u32, then one uniform), 2 u32 for tau, 10
// u32 per electron at initialisation. Because those counts are fixed, walker p's draws
// start at a computable offset (pos + 18 p), so each thread evaluates its own Philox
// counters independently (counter-based, per walker) and reproduces the reference chain.
// The only data-dependent consumption is the reference's redraw of an exactly coincident
// proposal (sampler.cpp:57-62) / placement (sampler.cpp:38-40); when that happens the last
// CTA replays the whole sweep sequentially, so the stream stays exact.
#include <cuda_runtime.h>

#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace mcmp2dev {

namespace {

__device__ __forceinline__ double g_of(const DevSites& s, double x, double y, double z) {
  // WeightSpec::g (weights.cpp:92-99): sites in order, two primitives each
  double v = 0.0;
  for (int i = 0; i < s.n; ++i) {
    const double dx = x - s.pos[3 * i], dy = y - s.pos[3 * i + 1], dz = z - s.pos[3 * i + 2];
    const double d2 = dx * dx + dy * dy + dz * dz;
    v += s.prim[4 * i + 0] * exp(-s.prim[4 * i + 1] * d2);
    v += s.prim[4 * i + 2] * exp(-s.prim[4 * i + 3] * d2);
  }
  return v;
}

__device__ __forceinline__ void gaussian3(StreamReader& r, double g[3]) {
  // PhiloxRng::gaussian3 (rng.cpp:66-74): four uniforms, fourth variate discarded
  const double u1 = r.uniform();
  const double u2 = r.uniform();
  const double u3 = r.uniform();
  const double u4 = r.uniform();
  const double r1 = sqrt(-2.0 * log1p(-u1));
  const double r2 = sqrt(-2.0 * log1p(-u2));
  const double a1 = 2.0 * 3.141592653589793 * u3;
  const double a2 = 2.0 * 3.141592653589793 * u4;
  double s1, c1;
  sincos(a1, &s1, &c1);
  g[0] = r1 * c1;
  g[1] = r1 * s1;
  g[2] = r2 * cos(a2);
}

struct Walker {
  double r1[3], r2[3], g1, g2, w;
};

__device__ __forceinline__ Walker load_walker(const WalkerBuf& b, int p) {
  Walker x;
  for (int k = 0; k < 3; ++k) {
    x.r1[k] = b.at(k, p);
    x.r2[k] = b.at(3 + k, p);
  }
  x.g1 = b.at(6, p);
  x.g2 = b.at(7, p);
  x.w = b.at(8, p);
  return x;
}

__device__ __forceinline__ void store_walker(const WalkerBuf& b, int p, const Walker& x) {
  for (int k = 0; k < 3; ++k) {
    b.at(k, p) = x.r1[k];
    b.at(3 + k, p) = x.r2[k];
  }
  b.at(6, p) = x.g1;
  b.at(7, p) = x.g2;
  b.at(8, p) = x.w;
}

// one proposal attempt for a pair (sampler.cpp:55-62); returns r12
__device__ __forceinline__ double propose(StreamReader& rd, const Walker& x, double sigma,
                                          double n1[3], double n2[3]) {
  double g[3];
  gaussian3(rd, g);
  for (int k = 0; k < 3; ++k) n1[k] = x.r1[k] + g[k] * sigma;
  gaussian3(rd, g);
  for (int k = 0; k < 3; ++k) n2[k] = x.r2[k] + g[k] * sigma;
  const double dx = n1[0] - n2[0], dy = n1[1] - n2[1], dz = n1[2] - n2[2];
  return sqrt(dx * dx + dy * dy + dz * dz);
}

// accept/reject of metropolis_step (sampler.cpp:63-77); returns 1 when accepted
__device__ __forceinline__ int decide(StreamReader& rd, const WalkParams& P, Walker& x,
                                      const double n1[3], const double n2[3], double r12) {
  const double g1 = g_of(P.sites, n1[0], n1[1], n1[2]);
  const double g2 = g_of(P.sites, n2[0], n2[1], n2[2]);
  const double wnew = g1 * g2 / (P.ng * r12);
  const double u = rd.uniform();
  if (u * x.w < wnew) {
    for (int k = 0; k < 3; ++k) {
      x.r1[k] = n1[k];
      x.r2[k] = n2[k];
    }
    x.g1 = g1;
    x.g2 = g2;
    x.w = wnew;
    return 1;
  }
  return 0;
}

// electron placement of init_ensemble (sampler.cpp:30-36)
__device__ __forceinline__ void place(StreamReader& rd, const DevSites& s, double r[3]) {
  const double u = rd.uniform();
  unsigned idx = unsigned(u * double(s.n));
  if (idx > unsigned(s.n - 1)) idx = unsigned(s.n - 1);
  const double spread = 1.0 / sqrt(2.0 * s.zeta1[idx]);
  double g[3];
  gaussian3(rd, g);
  for (int k = 0; k < 3; ++k) r[k] = s.pos[3 * idx + k] + g[k] * spread;
}

__device__ __forceinline__ double dist2(const double a[3], const double b[3]) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return dx * dx + dy * dy + dz * dz;
}

__device__ __forceinline__ void finish_init(const WalkParams& P, Walker& x) {
  x.g1 = g_of(P.sites, x.r1[0], x.r1[1], x.r1[2]);
  x.g2 = g_of(P.sites, x.r2[0], x.r2[1], x.r2[2]);
  x.w = x.g1 * x.g2 / (P.ng * sqrt(dist2(x.r1, x.r2)));
}

}  // namespace

// sqrt of guarded_exp (greens.cpp:9-16) for every spinor at the step's tau; overflow is
// flagged with the first offending spinor index, as the reference throws at set_tau.
__device__ void tau_weights(const WalkParams& P, double tau, bool speculative = false, DevState* st = nullptr,
                            double* swout = nullptr, int tid0 = -1, int nthr = 0) {
  const int np = P.n_occ + P.n_vir;
  if (!st) st = P.st;
  if (!swout) swout = P.sw;
  if (tid0 < 0) tid0 = threadIdx.x, nthr = blockDim.x;
  for (int k = tid0; k < np; k += nthr) {
    const double e = k < P.n_occ ? P.energies[k] * tau : -P.energies[k] * tau;
    double sw;
    if (e > 700.0) {
      if (speculative) {  // confirmed by the last CTA unless the sweep redrew a proposal
        atomicMin(&st->spec_error_idx, k);
      } else {
        atomicMin(&st->error_idx, k);
        st->error = 1;
      }
      sw = 0.0;
    } else if (e < -700.0) {
      sw = 0.0;
    } else {
      sw = exp(0.5 * e);
    }
    swout[k] = sw;
  }
}

// Two threads per walker (lane pair = electrons 1 and 2): each draws its electron's proposal
// from its own offset of the walker's 18 u32 (gaussian3 of electron 1 at +0, electron 2 at +8,
// the acceptance uniform at +16) and evaluates g at it; electron 1's thread then decides.
constexpr int WALK_THREADS = 128;

// tau = TauSampler::sample(rng.uniform()) after the sweep (driver.cpp:445), u32 at `pos`
__device__ double draw_tau(const WalkParams& P, unsigned long long pos, DevState* st = nullptr,
                           uint32_t stream = 0xffffffffu) {
  if (!st) st = P.st;
  StreamReader rd(P.k0, P.k1, stream == 0xffffffffu ? P.stream : stream, pos);
  const double u = rd.uniform();
  const double tau = -log1p(-u) / P.lambda;
  st->tau = tau;
  st->wtau = P.lambda * exp(-P.lambda * tau);
  return tau;
}

__global__ void __launch_bounds__(WALK_THREADS) walk_kernel(WalkParams P) {
  pdl_wait();     // the previous kernel's walkers / state are visible
  pdl_trigger();  // one wave: the next kernel may launch and wait for this one
  __shared__ int s_acc[WALK_THREADS / 32];
  __shared__ bool s_last;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = gt >> 1, e = gt & 1;
  // PRODUCTION launches one extra CTA that draws tau and the spinor weights speculatively at
  // the stream position the sweep ends at when no proposal is redrawn (pos + 18 m); the last
  // CTA redraws them in the rare redo case.
  const bool tau_cta = P.mode == WALK_PRODUCTION && blockIdx.x == gridDim.x - 1;
  const bool valid = p < P.m && !tau_cta;
  const unsigned long long pos0 = P.st->pos;
  int acc = 0;
  double n[3] = {0.0, 0.0, 0.0}, gn = 1.0;
  if (tau_cta) {
    __shared__ double s_tau;
    if (threadIdx.x == 0) s_tau = draw_tau(P, pos0 + 18ull * unsigned(P.m));
    __syncthreads();
    tau_weights(P, s_tau, true);
  } else if (P.mode == WALK_INIT) {
    if (valid) {  // placement of electron e: 10 u32 (sampler.cpp:30-36)
      StreamReader rd(P.k0, P.k1, P.stream, pos0 + 20ull * p + 10ull * e);
      place(rd, P.sites, n);
      gn = g_of(P.sites, n[0], n[1], n[2]);
    }
  } else if (valid) {  // proposal of electron e (sampler.cpp:55-56)
    StreamReader rd(P.k0, P.k1, P.stream, pos0 + 18ull * p + 8ull * e);
    double g[3];
    gaussian3(rd, g);
    const double sigma = P.st->sigma;
    for (int k = 0; k < 3; ++k) n[k] = P.in.at(3 * e + k, p) + g[k] * sigma;
    gn = g_of(P.sites, n[0], n[1], n[2]);
  }
  double m2[3];
  for (int k = 0; k < 3; ++k) m2[k] = __shfl_xor_sync(0xffffffffu, n[k], 1);
  const double g2n = __shfl_xor_sync(0xffffffffu, gn, 1);
  if (valid && e == 0) {
    if (P.mode == WALK_INIT) {
      Walker x;
      for (int k = 0; k < 3; ++k) {
        x.r1[k] = n[k];
        x.r2[k] = m2[k];
      }
      if (dist2(x.r1, x.r2) == 0.0) P.st->redo = 1;
      x.g1 = gn;
      x.g2 = g2n;
      x.w = x.g1 * x.g2 / (P.ng * sqrt(dist2(x.r1, x.r2)));
      store_walker(P.out, p, x);
    } else {
      Walker x = load_walker(P.in, p);
      const double dx = n[0] - m2[0], dy = n[1] - m2[1], dz = n[2] - m2[2];
      const double r12 = sqrt(dx * dx + dy * dy + dz * dz);
      if (r12 == 0.0) {
        P.st->redo = 1;
      } else {  // sampler.cpp:63-77
        StreamReader rd(P.k0, P.k1, P.stream, pos0 + 18ull * p + 16ull);
        const double wnew = gn * g2n / (P.ng * r12);
        const double u = rd.uniform();
        if (u * x.w < wnew) {
          for (int k = 0; k < 3; ++k) {
            x.r1[k] = n[k];
            x.r2[k] = m2[k];
          }
          x.g1 = gn;
          x.g2 = g2n;
          x.w = wnew;
          acc = 1;
        }
      }
      store_walker(P.out, p, x);
    }
  }
  // per-CTA accept count (integer: order independent)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) s_acc[wid] = acc;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < WALK_THREADS / 32; ++w) t += s_acc[w];
    P.block_acc[blockIdx.x] = t;
    __threadfence();
    const unsigned done = atomicAdd(&P.st->done_ctas, 1u);
    s_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ long long s_sum;
  if (threadIdx.x < 32) {  // sum of the per-CTA counts, one warp
    long long t = 0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) t += P.block_acc[b];
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) s_sum = t;
  }
  __syncthreads();

  // ---- last CTA: sequential redo if needed, stream advance, counters, tau ----
  __shared__ long long s_total;
  __shared__ unsigned long long s_consumed;
  __shared__ int s_redo;
  if (threadIdx.x == 0) {
    long long total = 0;
    unsigned long long consumed;
    s_redo = P.st->redo;
    if (s_redo) {
      // replay the whole sweep exactly as the reference's sequential loop
      StreamReader rd(P.k0, P.k1, P.stream, pos0);
      for (int q = 0; q < P.m; ++q) {
        if (P.mode == WALK_INIT) {
          Walker x;
          place(rd, P.sites, x.r1);
          do {
            place(rd, P.sites, x.r2);
          } while (dist2(x.r1, x.r2) == 0.0);
          finish_init(P, x);
          store_walker(P.out, q, x);
        } else {
          Walker x = load_walker(P.in, q);
          double n1[3], n2[3], r12;
          do {
            r12 = propose(rd, x, P.st->sigma, n1, n2);
          } while (r12 == 0.0);
          total += decide(rd, P, x, n1, n2, r12);
          store_walker(P.out, q, x);
        }
      }
      consumed = rd.pos - pos0;
      P.st->redo = 0;
    } else {
      total = s_sum;
      consumed = (P.mode == WALK_INIT ? 20ull : 18ull) * unsigned(P.m);
    }
    s_total = total;
    s_consumed = consumed;
    P.st->pos = pos0 + consumed;
    P.st->done_ctas = 0;
    if (P.mode == WALK_PRODUCTION) {
      P.st->proposed += P.m;
      P.st->accepted += total;
      if (s_redo) {
        draw_tau(P, P.st->pos);  // the speculative draw used the wrong position
      } else if (P.st->spec_error_idx != INT_MAX) {
        P.st->error = 1;
        P.st->error_idx = min(P.st->error_idx, P.st->spec_error_idx);
      }
      P.st->spec_error_idx = INT_MAX;
      P.st->pos += 2;
    } else if (P.mode == WALK_BURN) {
      // burn_in window and sigma adaptation (sampler.cpp:82-90)
      P.st->win_acc += total;
      P.st->win_prop += P.m;
      if (P.adapt && P.sweep % 100 == 0) {
        const double rate = double(P.st->win_acc) / double(P.st->win_prop);
        P.st->sigma = P.st->sigma * (rate > 0.5 ? 1.1 : 1.0 / 1.1);
        P.st->win_acc = 0;
        P.st->win_prop = 0;
      }
    }
  }
  __syncthreads();
  if (P.mode == WALK_PRODUCTION && s_redo) tau_weights(P, P.st->tau);
}

// Batched ensembles (several reference workers in one handle): one CTA per ensemble e, walkers
// [e m, (e+1) m) of the SoA buffers, Philox stream P.stream + e, state P.st[e], spinor weights
// P.sw + e * sw_stride. Threads 2p, 2p+1 take walker p's electrons exactly as walk_kernel; the
// last warp draws tau speculatively; the CTA itself does the bookkeeping that walk_kernel's last
// CTA does (sampler.cpp:49-93, driver.cpp:444-445), including the sequential redo.
__global__ void walk_batch_kernel(WalkParams P) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_acc;
  __shared__ int s_redo;
  __shared__ double s_tau;
  const int e = blockIdx.x, m = P.m;
  DevState* const st = P.st + e;
  const uint32_t stream = P.stream + uint32_t(e);
  double* const swe = P.sw + size_t(e) * P.sw_stride;
  const int base = e * m;
  const int tid = threadIdx.x, nwalk = 2 * m;
  const int p = tid >> 1, el = tid & 1;
  const bool walker_thread = tid < nwalk;
  const int tau_tid0 = (nwalk + 31) / 32 * 32;  // the tau warp follows the walker warps
  if (P.nactive > 0 && e >= P.nactive) {  // inactive this step: state and walkers unchanged
    for (int i = tid; i < 9 * m; i += blockDim.x) {
      const int k = i / m, q = i % m;
      P.out.at(k, base + q) = P.in.at(k, base + q);
    }
    return;
  }
  const unsigned long long pos0 = st->pos;
  if (tid == 0) {
    s_acc = 0;
    s_redo = 0;
  }
  __syncthreads();
  if (!walker_thread) {  // the tau warp (idle lanes of the last walker warp do nothing)
    if (P.mode == WALK_PRODUCTION && tid >= tau_tid0) {
      if (tid == tau_tid0) s_tau = draw_tau(P, pos0 + 18ull * unsigned(m), st, stream);
      __syncwarp();
      tau_weights(P, s_tau, true, st, swe, tid - tau_tid0, 32);
    }
  } else {
    double n[3], gn;
    if (P.mode == WALK_INIT) {
      StreamReader rd(P.k0, P.k1, stream, pos0 + 20ull * p + 10ull * el);
      place(rd, P.sites, n);
    } else {
      StreamReader rd(P.k0, P.k1, stream, pos0 + 18ull * p + 8ull * el);
      double g[3];
      gaussian3(rd, g);
      const double sigma = st->sigma;
      for (int k = 0; k < 3; ++k) n[k] = P.in.at(3 * el + k, base + p) + g[k] * sigma;
    }
    gn = g_of(P.sites, n[0], n[1], n[2]);
    const unsigned mask = __activemask();
    double m2[3];
    for (int k = 0; k < 3; ++k) m2[k] = __shfl_xor_sync(mask, n[k], 1);
    const double g2n = __shfl_xor_sync(mask, gn, 1);
    if (el == 0) {
      Walker x;
      if (P.mode == WALK_INIT) {
        for (int k = 0; k < 3; ++k) {
          x.r1[k] = n[k];
          x.r2[k] = m2[k];
        }
        if (dist2(x.r1, x.r2) == 0.0) s_redo = 1;
        x.g1 = gn;
        x.g2 = g2n;
        x.w = x.g1 * x.g2 / (P.ng * sqrt(dist2(x.r1, x.r2)));
      } else {
        x = load_walker(P.in, base + p);
        const double dx = n[0] - m2[0], dy = n[1] - m2[1], dz = n[2] - m2[2];
        const double r12 = sqrt(dx * dx + dy * dy + dz * dz);
        if (r12 == 0.0) {
          s_redo = 1;
        } else {  // sampler.cpp:63-77
          StreamReader rd(P.k0, P.k1, stream, pos0 + 18ull * p + 16ull);
          const double wnew = gn * g2n / (P.ng * r12);
          const double u = rd.uniform();
          if (u * x.w < wnew) {
            for (int k = 0; k < 3; ++k) {
              x.r1[k] = n[k];
              x.r2[k] = m2[k];
            }
            x.g1 = gn;
            x.g2 = g2n;
            x.w = wnew;
            atomicAdd(&s_acc, 1);  // integer count: order independent
          }
        }
      }
      store_walker(P.out, base + p, x);
    }
  }
  __syncthreads();
  if (tid == 0) {
    long long total = s_acc;
    unsigned long long consumed = (P.mode == WALK_INIT ? 20ull : 18ull) * unsigned(m);
    if (s_redo) {  // replay this ensemble's sweep exactly as the reference's sequential loop
      StreamReader rd(P.k0, P.k1, stream, pos0);
      total = 0;
      for (int q = 0; q < m; ++q) {
        if (P.mode == WALK_INIT) {
          Walker x;
          place(rd, P.sites, x.r1);
          do {
            place(rd, P.sites, x.r2);
          } while (dist2(x.r1, x.r2) == 0.0);
          finish_init(P, x);
          store_walker(P.out, base + q, x);
        } else {
          Walker x = load_walker(P.in, base + q);
          double n1[3], n2[3], r12;
          do {
            r12 = propose(rd, x, st->sigma, n1, n2);
          } while (r12 == 0.0);
          total += decide(rd, P, x, n1, n2, r12);
          store_walker(P.out, base + q, x);
        }
      }
      consumed = rd.pos - pos0;
    }
    st->pos = pos0 + consumed;
    if (P.mode == WALK_PRODUCTION) {
      st->proposed += m;
      st->accepted += total;
      if (s_redo) {
        s_tau = draw_tau(P, st->pos, st, stream);  // the speculative draw used the wrong position
        st->spec_error_idx = INT_MAX;
      } else if (st->spec_error_idx != INT_MAX) {
        st->error = 1;
        st->error_idx = min(st->error_idx, st->spec_error_idx);
        st->spec_error_idx = INT_MAX;
      }
      st->pos += 2;
    } else if (P.mode == WALK_BURN) {  // sampler.cpp:82-90
      st->win_acc += total;
      st->win_prop += m;
      if (P.adapt && P.sweep % 100 == 0) {
        const double rate = double(st->win_acc) / double(st->win_prop);
        st->sigma = st->sigma * (rate > 0.5 ? 1.1 : 1.0 / 1.1);
        st->win_acc = 0;
        st->win_prop = 0;
      }
    }
  }
  __syncthreads();
  if (P.mode == WALK_PRODUCTION && s_redo) tau_weights(P, s_tau, false, st, swe);
}

// replay: positions/g from the caller, tau given (estimator input of mc_step_estimate)
__global__ void replay_load_kernel(WalkParams P, const double* walkers, double tau) {
  pdl_wait();
  pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P.m) {
    for (int k = 0; k < 8; ++k) P.out.at(k, p) = walkers[size_t(p) * 8 + k];
  }
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      P.st->tau = tau;
      P.st->wtau = P.lambda * exp(-P.lambda * tau);
    }
    tau_weights(P, tau);
  }
}

void launch_walk(const WalkParams& P, cudaStream_t s) {
  // one CTA per ensemble (2m walker threads + one tau warp) for batches and for single ensembles
  // that fit one CTA: no cross-CTA last-CTA round trip
  if (P.nens > 1 || P.m <= 496) {
    const int threads = (2 * P.m + 31) / 32 * 32 + 32;
    pdl_launch(walk_batch_kernel, dim3(P.nens), dim3(threads), 0, s, P);
    return;
  }
  const int blocks = (2 * P.m + WALK_THREADS - 1) / WALK_THREADS + (P.mode == WALK_PRODUCTION ? 1 : 0);
  pdl_launch(walk_kernel, dim3(blocks), dim3(WALK_THREADS), 0, s, P);
}

void launch_replay_load(const WalkParams& P, const double* walkers, double tau, cudaStream_t s) {
  const int threads = 128;
  const int blocks = (P.m + threads - 1) / threads;
  pdl_launch(replay_load_kernel, dim3(blocks), dim3(threads), 0, s, P, walkers, tau);
}

}  // namespace mcmp2dev
