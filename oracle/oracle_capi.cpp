// oracle_capi.cpp — TEST INFRASTRUCTURE ONLY: C entry points of the CPU oracle for
// the pytest parity suite and bench.py's CPU-baseline leg (ctypes). Nothing in the
// product path loads liboracle.so.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <thread>

#include "mcmp2_oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

struct System {
  SpinorSet spinors;
  WeightSpec spec;
  TauSampler tau;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return 2;
  }
}

void walker_to(const WalkerPair& p, double* o) {
  const double v[9] = {p.r1.x, p.r1.y, p.r1.z, p.r2.x, p.r2.y, p.r2.z, p.g1, p.g2, p.weight};
  std::memcpy(o, v, sizeof v);
}

void est_to(const StepEstimate& e, double* o) {
  o[0] = e.value;
  o[1] = e.imag;
  o[2] = e.direct_sum.real();
  o[3] = e.direct_sum.imag();
  o[4] = e.exchange_sum.real();
  o[5] = e.exchange_sum.imag();
}

WalkerEnsemble from_walkers(const double* w, int m) {
  WalkerEnsemble ens;
  ens.pairs.resize(m);
  for (int p = 0; p < m; ++p) {
    const double* v = w + 8 * std::size_t(p);
    ens.pairs[p].r1 = {v[0], v[1], v[2]};
    ens.pairs[p].r2 = {v[3], v[4], v[5]};
    ens.pairs[p].g1 = v[6];
    ens.pairs[p].g2 = v[7];
  }
  return ens;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_philox_block(const std::uint32_t* ctr, const std::uint32_t* key, std::uint32_t* out) {
  const auto o = Philox::block({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = o[i];
  return 0;
}

// n sequential draws of kind 0: next_u32, 1: uniform, 2: gaussian3 (3 values each)
int orc_philox_stream(std::uint64_t seed, std::uint32_t stream, int kind, int n, double* out) {
  Philox r(seed, stream);
  for (int i = 0; i < n; ++i) {
    if (kind == 0) out[i] = double(r.next_u32());
    else if (kind == 1) out[i] = r.uniform();
    else {
      const auto g = r.gaussian3();
      out[3 * i] = g[0];
      out[3 * i + 1] = g[1];
      out[3 * i + 2] = g[2];
    }
  }
  return 0;
}

std::uint64_t orc_fnv1a64(const char* bytes, long n) { return fnv1a64(std::string(bytes, n)); }

double orc_boys_f0(double t) { return boys_f0(t); }
double orc_primitive_norm(int l, double z) { return primitive_norm(l, z); }
double orc_solid_harmonic(int l, int m, double x, double y, double z) {
  return solid_harmonic(l, m, Vec3{x, y, z});
}
int orc_guarded_exp(double e, int idx, double* out) {
  return guard([&] { *out = guarded_exp(e, idx); });
}

// spinor file + optional run-config text (only `weight` lines are used)
void* orc_system_load(const char* spinor_path, const char* config_text) {
  System* s = nullptr;
  const int rc = guard([&] {
    SpinorSet sp = load_spinor_set(spinor_path);
    if (!sp.nuclei) throw std::runtime_error("spinor file has no nuclei record; the sampling weight needs it");
    RunConfig cfg = parse_config_text(config_text ? config_text : "");
    WeightSpec spec(*sp.nuclei, cfg.weight_overrides);
    TauSampler ts(lambda_from_gap(sp));
    s = new System{std::move(sp), std::move(spec), ts};
  });
  return rc == 0 ? s : nullptr;
}

void orc_system_free(void* h) { delete static_cast<System*>(h); }

// ints: ncomp, n_occ, n_vir, rows, nsites; dbls: ng, lambda
int orc_system_info(void* h, int* ints, double* dbls) {
  auto* s = static_cast<System*>(h);
  ints[0] = s->spinors.ncomp;
  ints[1] = s->spinors.n_occ;
  ints[2] = s->spinors.n_vir;
  ints[3] = s->spinors.rows;
  ints[4] = int(s->spec.sites.size());
  dbls[0] = s->spec.ng();
  dbls[1] = s->tau.lambda();
  return 0;
}

int orc_g(void* h, const double* pts, int n, double* out) {
  auto* s = static_cast<System*>(h);
  for (int i = 0; i < n; ++i) out[i] = s->spec.g(Vec3{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
  return 0;
}

// spinor values at n points: occ [n][nc][n_occ] complex, vir [n][nc][n_vir] complex (re,im)
int orc_evaluate(void* h, const double* pts, int n, double* occ, double* vir) {
  auto* s = static_cast<System*>(h);
  const auto& sp = s->spinors;
  std::vector<double> chi(sp.max_channel_size());
  for (int i = 0; i < n; ++i)
    sp.evaluate_into(Vec3{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]},
                     reinterpret_cast<Complex*>(occ) + std::size_t(i) * sp.ncomp * sp.n_occ,
                     reinterpret_cast<Complex*>(vir) + std::size_t(i) * sp.ncomp * sp.n_vir, chi.data());
  return 0;
}

// Chain of the reference worker loop (driver.cpp:440-450): init_ensemble + burn_in, then
// nsteps x (metropolis_step, tau draw, estimate). Outputs:
//   init_state: post-burn-in ensemble, m x 9 (r1, r2, g1, g2, w) then sigma, 7 rng words
//   walkers: nsteps x m x 8 (r1, r2, g1, g2 used by the step), tau: nsteps,
//   est: nsteps x 6 (value, imag, direct re/im, exchange re/im), final_state like init_state
//   counters: proposed, accepted (production)
int orc_trajectory(void* h, std::uint64_t seed, std::uint32_t stream, int m, long burn,
                   double step_size, int adapt, long nsteps, int physical, double* init_state,
                   double* walkers, double* tau_out, double* est, double* final_state,
                   long long* counters) {
  auto* s = static_cast<System*>(h);
  return guard([&] {
    WalkerEnsemble ens = init_ensemble(m, *s->spinors.nuclei, s->spec, seed, stream);
    if (step_size > 0) ens.sigma_step = step_size;
    burn_in(ens, s->spec, burn, adapt != 0);
    auto dump_state = [&](double* o) {
      if (!o) return;
      for (int p = 0; p < m; ++p) walker_to(ens.pairs[p], o + 9 * std::size_t(p));
      double* t = o + 9 * std::size_t(m);
      t[0] = ens.sigma_step;
      t[1] = ens.rng.key[0];
      t[2] = ens.rng.key[1];
      for (int k = 0; k < 4; ++k) t[3 + k] = ens.rng.counter[k];
      t[7] = ens.rng.idx;
    };
    dump_state(init_state);
    EstimatorWorkspace ws(s->spinors, m);
    ws.physical = physical != 0;
    for (long st = 0; st < nsteps; ++st) {
      metropolis_step(ens, s->spec);
      const double tau = s->tau.sample(ens.rng.uniform());
      const StepEstimate e = mc_step_estimate(s->spinors, ens, tau, s->spec, s->tau, ws);
      if (walkers)
        for (int p = 0; p < m; ++p) {
          const auto& pr = ens.pairs[p];
          double* o = walkers + (std::size_t(st) * m + p) * 8;
          const double v[8] = {pr.r1.x, pr.r1.y, pr.r1.z, pr.r2.x, pr.r2.y, pr.r2.z, pr.g1, pr.g2};
          std::memcpy(o, v, sizeof v);
        }
      if (tau_out) tau_out[st] = tau;
      if (est) est_to(e, est + 6 * std::size_t(st));
    }
    dump_state(final_state);
    if (counters) {
      counters[0] = ens.proposed;
      counters[1] = ens.accepted;
    }
  });
}

// Metropolis-only chain (sampler.cpp:49-93): init_ensemble + burn_in(burn, adapt), then
// nsteps sweeps; every `thin`-th sweep the electron separations |r1 - r2| of all walkers are
// written to u_out (nsteps / thin x m). Returns the production acceptance in *acceptance.
int orc_chain_r12(void* h, std::uint64_t seed, int m, long burn, long nsteps, long thin, double* u_out,
                  double* acceptance) {
  auto* s = static_cast<System*>(h);
  return guard([&] {
    WalkerEnsemble ens = init_ensemble(m, *s->spinors.nuclei, s->spec, seed, 0);
    burn_in(ens, s->spec, burn, true);
    long k = 0;
    for (long st = 0; st < nsteps; ++st) {
      metropolis_step(ens, s->spec);
      if (st % thin != 0) continue;
      for (int p = 0; p < m; ++p) {
        const auto& w = ens.pairs[p];
        const double dx = w.r1.x - w.r2.x, dy = w.r1.y - w.r2.y, dz = w.r1.z - w.r2.z;
        u_out[k++] = std::sqrt(dx * dx + dy * dy + dz * dz);
      }
    }
    *acceptance = double(ens.accepted) / double(ens.proposed);
  });
}

// estimate at given positions (m x 8 per step) and tau: the replay oracle
int orc_replay(void* h, int m, long nsteps, const double* walkers, const double* tau, int physical,
               double* est) {
  auto* s = static_cast<System*>(h);
  return guard([&] {
    EstimatorWorkspace ws(s->spinors, m);
    ws.physical = physical != 0;
    for (long st = 0; st < nsteps; ++st) {
      const WalkerEnsemble ens = from_walkers(walkers + std::size_t(st) * m * 8, m);
      const StepEstimate e = mc_step_estimate(s->spinors, ens, tau[st], s->spec, s->tau, ws);
      est_to(e, est + 6 * std::size_t(st));
    }
  });
}

// One replay step at full size with `threads` std::threads, each summing the pair terms of a
// contiguous band of walker rows (bands balanced by pair count), partial results added in
// band order: the full-size parity check (association differs from the sequential loop only
// in the band split).
int orc_replay_parallel(void* h, int m, const double* walkers, double tau, int threads, int physical,
                        double* est) {
  auto* s = static_cast<System*>(h);
  return guard([&] {
    const WalkerEnsemble ens = from_walkers(walkers, m);
    const double total = 0.5 * double(m) * (m - 1);
    std::vector<int> cut(threads + 1, m);
    cut[0] = 0;
    double acc = 0.0;
    int t = 1;
    for (int p = 0; p < m && t < threads; ++p) {  // row p holds m - 1 - p pairs
      acc += m - 1 - p;
      if (acc >= total * t / threads) cut[t++] = p + 1;
    }
    std::vector<StepEstimate> part(threads);
    std::vector<std::thread> pool;
    for (int k = 0; k < threads; ++k)
      pool.emplace_back([&, k] {
        EstimatorWorkspace ws(s->spinors, m);
        ws.physical = physical != 0;
        part[k] = mc_step_estimate_rows(s->spinors, ens, tau, s->spec, s->tau, ws, cut[k], cut[k + 1], nullptr);
      });
    for (auto& th : pool) th.join();
    StepEstimate e;
    e.value = 0.0;
    e.imag = 0.0;
    for (const auto& q : part) {
      e.value += q.value;
      e.imag += q.imag;
      e.direct_sum += q.direct_sum;
      e.exchange_sum += q.exchange_sum;
    }
    est_to(e, est);
  });
}

// sample_term (estimator.cpp:65-75): p, q = 8 doubles each; out: direct re/im, exchange re/im
int orc_sample_term(void* h, const double* p, const double* q, double tau, int physical, double* out) {
  auto* s = static_cast<System*>(h);
  return guard([&] {
    const WalkerEnsemble e = from_walkers(p, 1), f = from_walkers(q, 1);
    const SampleTerm t = sample_term(s->spinors, e.pairs[0], f.pairs[0], tau, s->spec, s->tau, physical != 0);
    out[0] = t.direct.real();
    out[1] = t.direct.imag();
    out[2] = t.exchange.real();
    out[3] = t.exchange.imag();
  });
}

// driver run on config text; report text copied into buf
int orc_run_config(const char* config_text, char* buf, int cap) {
  return guard([&] {
    RunConfig cfg = parse_config_text(config_text);
    const std::string rep = format_report(run(cfg));
    std::snprintf(buf, cap, "%s", rep.c_str());
  });
}

int orc_resume(const char* ckpt, char* buf, int cap) {
  return guard([&] {
    const std::string rep = format_report(resume(ckpt));
    std::snprintf(buf, cap, "%s", rep.c_str());
  });
}

// CPU baseline (bench.py): `threads` independent workers (std::thread, as driver.cpp:423-438),
// each: init_ensemble(stream = worker), burn_in(burn), then `steps` x (metropolis_step, tau,
// estimate restricted to walker rows [0, rows)), i.e. a bounded sample of the step's C(m,2)
// pair loop. Returns the wall seconds of the timed production loop and the samples done.
int orc_cpu_baseline(void* h, std::uint64_t seed, int m, int rows, long burn, double step_size,
                     long steps, int threads, double* seconds, long long* samples) {
  auto* s = static_cast<System*>(h);
  return guard([&] {
    std::vector<WalkerEnsemble> ens(threads);
    for (int t = 0; t < threads; ++t) {
      ens[t] = init_ensemble(m, *s->spinors.nuclei, s->spec, seed, std::uint32_t(t));
      if (step_size > 0) ens[t].sigma_step = step_size;
      burn_in(ens[t], s->spec, burn, step_size <= 0);
    }
    std::vector<long long> done(threads, 0);
    std::vector<double> sink(threads, 0.0);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        EstimatorWorkspace ws(s->spinors, m);
        for (long st = 0; st < steps; ++st) {
          metropolis_step(ens[t], s->spec);
          const double tau = s->tau.sample(ens[t].rng.uniform());
          long long np = 0;
          const StepEstimate e =
              mc_step_estimate_rows(s->spinors, ens[t], tau, s->spec, s->tau, ws, 0, rows, &np);
          sink[t] += e.value;
          done[t] += np;
        }
      });
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    long long tot = 0;
    for (auto d : done) tot += d;
    *samples = tot;
  });
}

}  // extern "C"

extern "C" {
double orc_tau_sample(double lambda, double u) { return TauSampler(lambda).sample(u); }
double orc_tau_pdf(double lambda, double tau) { return TauSampler(lambda).pdf(tau); }

// BlockingAccumulator over a value stream: out = mean, sigma, sigma_bar, nblocks
int orc_blocking(const double* v, long n, long nb, double* out) {
  return guard([&] {
    BlockingAccumulator a(nb);
    for (long i = 0; i < n; ++i) a.add(v[i]);
    out[0] = a.mean();
    out[1] = a.sigma();
    out[2] = a.sigma_bar();
    out[3] = double(a.block_means().size());
  });
}
}
