// capi.cpp — C entry points of libmcmp2host.so (include/mcmp2host.h).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mcmp2host.h"
#include "../csrc/philox.h"
#include "mcmp2.hpp"

using namespace mcmp2;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

void copy_out(const std::string& s, char* buf, int cap) {
  if (buf && cap > 0) std::snprintf(buf, std::size_t(cap), "%s", s.c_str());
}
}  // namespace

struct mcmp2h_system {
  SpinorSet spinors;
  WeightSpec spec;
  DeviceSystem dev;
};

struct mcmp2h_worker {
  RunConfig cfg;
  std::unique_ptr<SpinorSet> spinors;
  std::unique_ptr<WeightSpec> spec;
  std::unique_ptr<DeviceWorker> worker;
};

// the workers one process hosts on one device (distributed.py): one batched handle when the
// walker count allows it (as the Engine does per device), else one handle per worker
struct mcmp2h_group {
  RunConfig cfg;
  std::unique_ptr<SpinorSet> spinors;
  std::unique_ptr<WeightSpec> spec;
  std::shared_ptr<DeviceBatch> batch;
  std::vector<std::unique_ptr<DeviceWorker>> workers;
};

extern "C" {

const char* mcmp2h_last_error(void) { return g_err.c_str(); }

namespace {
// workers [first, first + count) on one device; restored from `resume_path` when given, else
// init + burn-in (driver.cpp:354-373)
mcmp2h_group* make_group(const RunConfig& cfg, int first_index, int count, int device, const char* resume_path) {
  if (count < 1) throw std::invalid_argument("group: at least one worker");
  auto g = std::make_unique<mcmp2h_group>();
  g->cfg = cfg;
  g->cfg.validate();
  g->spinors = std::make_unique<SpinorSet>(load_spinor_set(g->cfg.spinor_path));
  if (!g->spinors->nuclei) throw std::runtime_error("spinor file has no nuclei record; the sampling weight needs it");
  g->spec = std::make_unique<WeightSpec>(*g->spinors->nuclei, g->cfg.weight_overrides);
  if (count > 1 && g->cfg.walkers % 16 == 0 && g->cfg.walkers <= 480) {
    DeviceSystem sys = make_device_system(*g->spinors, *g->spec,
                                          g->cfg.physical ? MCMP2DEV_ESTIMATOR_PHYSICAL : MCMP2DEV_ESTIMATOR_LITERAL);
    g->batch = std::make_shared<DeviceBatch>();
    check_dev(mcmp2dev_create(&sys.view, device, count * g->cfg.walkers, &g->batch->h), nullptr);
    g->batch->first = first_index;
    g->batch->nens = count;
    g->batch->m = g->cfg.walkers;
  }
  for (int k = 0; k < count; ++k) {
    if (g->batch) g->workers.push_back(std::make_unique<DeviceWorker>(g->batch, k, g->cfg, first_index + k));
    else g->workers.push_back(std::make_unique<DeviceWorker>(*g->spinors, *g->spec, g->cfg, first_index + k, device));
  }
  if (resume_path) {
    std::vector<DeviceWorker*> ws;
    for (auto& w : g->workers) ws.push_back(w.get());
    restore_workers(resume_path, *g->spec, g->cfg, ws);
  } else {
    for (auto& w : g->workers) w->init_and_burn_in();
  }
  return g.release();
}

int copy_sized(const std::string& s, char* buf, long cap, long* need) {
  if (need) *need = long(s.size()) + 1;
  if (buf && cap > long(s.size())) std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}
}  // namespace

mcmp2h_group* mcmp2h_group_create(const char* config_text, int first_index, int count, int device) {
  mcmp2h_group* out = nullptr;
  guard([&] { out = make_group(parse_config_text(config_text), first_index, count, device, nullptr); });
  return out;
}

mcmp2h_group* mcmp2h_group_resume(const char* checkpoint_path, int first_index, int count, int device) {
  mcmp2h_group* out = nullptr;
  guard([&] { out = make_group(checkpoint_config(checkpoint_path), first_index, count, device, checkpoint_path); });
  return out;
}

int mcmp2h_checkpoint_config(const char* checkpoint_path, char* canonical, int cap, int* nworkers) {
  return guard([&] {
    std::vector<int> idx;
    const RunConfig c = checkpoint_config(checkpoint_path, &idx);
    for (std::size_t k = 0; k < idx.size(); ++k)
      if (idx[k] != int(k)) throw std::runtime_error("checkpoint: worker records are not 0 .. workers - 1");
    if (nworkers) *nworkers = int(idx.size());
    copy_out(canonical_config_text(c), canonical, cap);
  });
}

int mcmp2h_checkpoint_header(const char* config_text, int nworkers, char* buf, long cap, long* need) {
  return guard([&] {
    const RunConfig c = parse_config_text(config_text);
    c.validate();
    copy_sized(checkpoint_header_text(c, std::size_t(nworkers)), buf, cap, need);
  });
}

int mcmp2h_group_record(mcmp2h_group* g, int k, char* buf, long cap, long* need) {
  return guard([&] {
    if (k < 0 || k >= int(g->workers.size())) throw std::invalid_argument("group: no such worker");
    copy_sized(worker_record_text(*g->workers[k]), buf, cap, need);
  });
}

int mcmp2h_group_trace(mcmp2h_group* g, int k, char* buf, long cap, long* need) {
  return guard([&] {
    if (k < 0 || k >= int(g->workers.size())) throw std::invalid_argument("group: no such worker");
    copy_sized(worker_trace_text(*g->workers[k]), buf, cap, need);
  });
}

void mcmp2h_group_free(mcmp2h_group* g) { delete g; }

int mcmp2h_group_size(const mcmp2h_group* g) { return g ? int(g->workers.size()) : 0; }

int mcmp2h_group_advance(mcmp2h_group* g, const long long* nsteps) {
  return guard([&] {
    std::vector<long long> n(nsteps, nsteps + g->workers.size());
    for (auto& x : n) x = std::max<long long>(x, 0);
    if (g->batch) {
      std::vector<DeviceWorker*> ws;
      for (auto& w : g->workers) ws.push_back(w.get());
      DeviceWorker::advance_batch(*g->batch, ws, n);
    } else {
      for (std::size_t k = 0; k < g->workers.size(); ++k) g->workers[k]->advance(n[k]);
    }
  });
}

int mcmp2h_group_stats(mcmp2h_group* g, int k, double* o) {
  return guard([&] {
    if (k < 0 || k >= int(g->workers.size())) throw std::invalid_argument("group: no such worker");
    const DeviceWorker& w = *g->workers[k];
    const auto& a = w.acc;
    o[0] = double(a.count());
    o[1] = a.real_sum();
    o[2] = a.imag_sum();
    o[3] = a.mean();
    o[4] = a.sigma_bar();
    o[5] = double(a.in_block());
    o[6] = a.partial();
    o[7] = double(a.block_means().size());
    const WorkerSummary s = w.summary();  // driver.cpp:207-216
    o[8] = s.acceptance;
    o[9] = s.imag_ratio;
  });
}

int mcmp2h_run(const char* config_text, char* report, int cap) {
  return guard([&] { copy_out(format_report(run(parse_config_text(config_text))), report, cap); });
}

int mcmp2h_run_hooked(const char* config_text, long abort_after, char* report, int cap) {
  return guard([&] {
    RunHooks h;
    h.abort_after_intervals = abort_after;
    copy_out(format_report(run(parse_config_text(config_text), h)), report, cap);
  });
}

int mcmp2h_resume(const char* path, char* report, int cap) {
  return guard([&] { copy_out(format_report(resume(path)), report, cap); });
}

int mcmp2h_merge(const char* const* paths, int n, double* value, double* sigma_bar, long long* steps) {
  return guard([&] {
    std::vector<std::string> p(paths, paths + n);
    const MergedEstimate m = merge_checkpoint_files(p);
    *value = m.value;
    *sigma_bar = m.sigma_bar;
    *steps = m.total_steps;
  });
}

int mcmp2h_parse_config(const char* text, char* canonical, int cap) {
  return guard([&] {
    const RunConfig c = parse_config_text(text);
    c.validate();
    copy_out(canonical_config_text(c), canonical, cap);
  });
}

uint64_t mcmp2h_fnv1a64(const char* bytes, long n) { return fnv1a64(std::string(bytes, std::size_t(n))); }

mcmp2h_system* mcmp2h_system_load(const char* spinor_path, const char* config_text) {
  mcmp2h_system* out = nullptr;
  guard([&] {
    SpinorSet s = load_spinor_set(spinor_path);
    if (!s.nuclei) throw std::runtime_error("spinor file has no nuclei record; the sampling weight needs it");
    const RunConfig c = parse_config_text(config_text ? config_text : "");
    WeightSpec w(*s.nuclei, c.weight_overrides);
    DeviceSystem d = make_device_system(s, w, c.physical ? MCMP2DEV_ESTIMATOR_PHYSICAL : MCMP2DEV_ESTIMATOR_LITERAL);
    out = new mcmp2h_system{std::move(s), std::move(w), std::move(d)};
  });
  return out;
}

void mcmp2h_system_free(mcmp2h_system* s) { delete s; }

const mcmp2dev_system* mcmp2h_system_view(const mcmp2h_system* s) { return &s->dev.view; }

int mcmp2h_system_info(const mcmp2h_system* s, int* ints, double* dbls) {
  return guard([&] {
    ints[0] = s->spinors.ncomp;
    ints[1] = s->spinors.n_occ;
    ints[2] = s->spinors.n_vir;
    ints[3] = s->spinors.rows();
    dbls[0] = s->spec.ng;
    dbls[1] = s->dev.view.lambda;
    dbls[2] = s->spinors.orthonormality_deviation();
  });
}

int mcmp2h_system_g(const mcmp2h_system* s, const double* pts, int n, double* out) {
  return guard([&] {
    for (int i = 0; i < n; ++i) out[i] = s->spec.g({pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
  });
}

int mcmp2h_save_spinor_set(const char* in_path, const char* out_path) {
  return guard([&] { save_spinor_set(load_spinor_set(in_path), out_path); });
}

mcmp2h_worker* mcmp2h_worker_create(const char* config_text, int worker_index, int device) {
  mcmp2h_worker* out = nullptr;
  guard([&] {
    auto w = std::make_unique<mcmp2h_worker>();
    w->cfg = parse_config_text(config_text);
    w->cfg.validate();
    w->spinors = std::make_unique<SpinorSet>(load_spinor_set(w->cfg.spinor_path));
    if (!w->spinors->nuclei) throw std::runtime_error("spinor file has no nuclei record; the sampling weight needs it");
    w->spec = std::make_unique<WeightSpec>(*w->spinors->nuclei, w->cfg.weight_overrides);
    w->worker = std::make_unique<DeviceWorker>(*w->spinors, *w->spec, w->cfg, worker_index, device);
    w->worker->init_and_burn_in();
    out = w.release();
  });
  return out;
}

void mcmp2h_worker_free(mcmp2h_worker* w) { delete w; }

int mcmp2h_worker_advance(mcmp2h_worker* w, long nsteps, double* values, double* imags) {
  return guard([&] {
    w->worker->advance(nsteps);
    for (long s = 0; s < nsteps; ++s) {
      if (values) values[s] = w->worker->last_values()[s];
      if (imags) imags[s] = w->worker->last_imags()[s];
    }
  });
}

int mcmp2h_worker_stats(mcmp2h_worker* w, double* o) {
  return guard([&] {
    const auto& a = w->worker->acc;
    o[0] = double(a.count());
    o[1] = a.real_sum();
    o[2] = a.imag_sum();
    o[3] = a.mean();
    o[4] = a.sigma_bar();
    o[5] = double(a.in_block());
    o[6] = a.partial();
    o[7] = double(a.block_means().size());
    const WorkerSummary s = w->worker->summary();  // driver.cpp:207-216
    o[8] = s.acceptance;
    o[9] = s.imag_ratio;
  });
}

int mcmp2h_worker_block_means(mcmp2h_worker* w, double* out, int cap) {
  return guard([&] {
    const auto& m = w->worker->acc.block_means();
    for (int i = 0; i < cap && i < int(m.size()); ++i) out[i] = m[i];
  });
}

mcmp2dev_t* mcmp2h_worker_device(mcmp2h_worker* w) { return w->worker->handle(); }

int mcmp2h_generate(const char* name, const char* dir) {
  return guard([&] { write_generated(name, dir); });
}

}  // extern "C"

extern "C" {

// BlockingAccumulator (estimator.cpp:77-121) over a value stream: mean, sigma, sigma_bar, nblocks
int mcmp2h_blocking(const double* v, long n, long nb, double* out) {
  return guard([&] {
    BlockingAccumulator a(nb);
    for (long i = 0; i < n; ++i) a.add(v[i]);
    out[0] = a.mean();
    out[1] = a.sigma();
    out[2] = a.sigma_bar();
    out[3] = double(a.block_means().size());
  });
}

// merge_estimates (driver.cpp:183-196): parts as {steps, mean, sigma_bar} rows
int mcmp2h_merge_estimates(const double* parts, int n, double* out3) {
  return guard([&] {
    std::vector<WorkerSummary> v;
    for (int i = 0; i < n; ++i)
      v.push_back(WorkerSummary{i, (long long)parts[3 * i], parts[3 * i + 1], parts[3 * i + 2], 0.0, 0.0});
    const MergedEstimate m = merge_estimates(v);
    out3[0] = m.value;
    out3[1] = m.sigma_bar;
    out3[2] = double(m.total_steps);
  });
}

uint64_t mcmp2h_config_hash(const char* config_text, uint64_t spinor_hash) {
  uint64_t h = 0;
  guard([&] { h = config_hash(parse_config_text(config_text), spinor_hash); });
  return h;
}

// u32 draws [pos, pos + n) of the reference stream PhiloxRng(seed, stream), addressed by
// position exactly as the device kernels do (csrc/philox.h)
int mcmp2h_philox_stream(uint64_t seed, uint32_t stream, uint64_t pos, int n, uint32_t* out) {
  mcmp2dev::StreamReader r(uint32_t(seed), uint32_t(seed >> 32), stream, pos);
  for (int i = 0; i < n; ++i) out[i] = r.next_u32();
  return 0;
}

}  // extern "C"
