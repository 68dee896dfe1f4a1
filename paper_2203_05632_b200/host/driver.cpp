// driver.cpp — run control around the device walker loop: RunConfig, blocking statistics,
// DeviceWorker (one C-ABI handle per reference worker), Engine with checkpoint/resume,
// convergence traces, merging and the report (reference proj/core/src/driver.cpp,
// estimator.cpp:77-131, sampler.cpp:95-120; cited per function).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <thread>

#include <cuda_runtime.h>

#include "mcmp2.hpp"

namespace mcmp2 {

// ------------------------------------------------------------------ estimator.cpp:77-131
BlockingAccumulator::BlockingAccumulator(long nb) : nb_(nb) {
  if (nb_ < 1) throw std::invalid_argument("BlockingAccumulator: block size must be >= 1");
}

void BlockingAccumulator::add(double value, double imag) {
  sum_ += value;
  imag_sum_ += imag;
  ++n_;
  partial_ += value;
  if (++in_block_ == nb_) {
    means_.push_back(partial_ / double(nb_));
    partial_ = 0.0;
    in_block_ = 0;
  }
}

double BlockingAccumulator::sigma() const {  // mean includes the unfinished block
  if (means_.empty()) return 0.0;
  const double m = mean();
  double s2 = 0.0;
  for (double b : means_) s2 += (b - m) * (b - m);
  return std::sqrt(s2 / double(means_.size()));
}

double BlockingAccumulator::sigma_bar() const {
  return means_.empty() ? 0.0 : sigma() / std::sqrt(double(means_.size()));
}

std::vector<BlockingAccumulator::TracePoint> BlockingAccumulator::trace() const {
  std::vector<TracePoint> out;
  double cum = 0.0;
  for (std::size_t k = 0; k < means_.size(); ++k) {
    cum += means_[k];
    const double mk = cum / double(k + 1);
    double s2 = 0.0;
    for (std::size_t j = 0; j <= k; ++j) s2 += (means_[j] - mk) * (means_[j] - mk);
    out.push_back({(long long)(k + 1) * nb_, mk, std::sqrt(s2 / double(k + 1)) / std::sqrt(double(k + 1))});
  }
  return out;
}

void BlockingAccumulator::restore(long long n, double sum, double imag_sum, long in_block, double partial,
                                  std::vector<double> means) {
  n_ = n;
  sum_ = sum;
  imag_sum_ = imag_sum;
  in_block_ = in_block;
  partial_ = partial;
  means_ = std::move(means);
}

// ------------------------------------------------------------------ config (driver.cpp:50-181)
namespace {
std::vector<std::string> split_line(const std::string& line) {
  std::string s = line.substr(0, line.find('#'));
  std::istringstream is(s);
  std::vector<std::string> out;
  for (std::string w; is >> w;) out.push_back(w);
  return out;
}

long long as_int(const std::string& tok, const std::string& key) {
  char* end = nullptr;
  errno = 0;
  const long long v = std::strtoll(tok.c_str(), &end, 10);
  if (tok.empty() || *end != '\0' || errno)
    throw std::runtime_error("config: key '" + key + "' expects an integer, got '" + tok + "'");
  return v;
}

double as_num(const std::string& tok, const std::string& key) {
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(tok.c_str(), &end);
  if (tok.empty() || *end != '\0' || errno == ERANGE)
    throw std::runtime_error("config: key '" + key + "' expects a number, got '" + tok + "'");
  return v;
}

void put_weights(std::ostream& os, const RunConfig& c) {
  for (const auto& [z, w] : c.weight_overrides)
    os << "weight " << element_symbol(z) << ' ' << format_double(w.c1) << ' ' << format_double(w.zeta1) << ' '
       << format_double(w.c2) << ' ' << format_double(w.zeta2) << "\n";
}
}  // namespace

void RunConfig::validate() const {
  if (spinor_path.empty()) throw std::runtime_error("config: no spinor file given");
  if (steps.has_value() == target_rel_err.has_value())
    throw std::runtime_error("config: exactly one stopping rule required (steps or target-rel-err)");
  if (steps && *steps < 1) throw std::runtime_error("config: steps must be positive");
  if (target_rel_err && !(*target_rel_err > 0)) throw std::runtime_error("config: target-rel-err must be positive");
  if (walkers < 2) throw std::runtime_error("config: walkers must be >= 2");
  if (workers < 1) throw std::runtime_error("config: workers must be >= 1");
  if (block_size < 1) throw std::runtime_error("config: blocksize must be >= 1");
  if (burn_in < 0) throw std::runtime_error("config: burnin must be >= 0");
  if (checkpoint_interval < 1) throw std::runtime_error("config: checkpoint-interval must be >= 1");
  if (step_size && !(*step_size > 0)) throw std::runtime_error("config: step-size must be positive");
}

RunConfig parse_config_text(const std::string& text) {
  RunConfig c;
  std::istringstream in(text);
  for (std::string line; std::getline(in, line);) {
    const auto t = split_line(line);
    if (t.empty()) continue;
    const std::string& k = t[0];
    auto arity = [&](std::size_t n) {
      if (t.size() != n + 1)
        throw std::runtime_error("config: key '" + k + "' expects " + std::to_string(n) + " value(s)");
    };
    if (k == "spinors") arity(1), c.spinor_path = t[1];
    else if (k == "steps") arity(1), c.steps = as_int(t[1], k);
    else if (k == "target-rel-err") arity(1), c.target_rel_err = as_num(t[1], k);
    else if (k == "walkers") arity(1), c.walkers = int(as_int(t[1], k));
    else if (k == "seed") arity(1), c.seed = std::uint64_t(as_int(t[1], k));
    else if (k == "workers") arity(1), c.workers = int(as_int(t[1], k));
    else if (k == "blocksize") arity(1), c.block_size = long(as_int(t[1], k));
    else if (k == "burnin") arity(1), c.burn_in = long(as_int(t[1], k));
    else if (k == "checkpoint") arity(1), c.checkpoint_path = t[1];
    else if (k == "checkpoint-interval") arity(1), c.checkpoint_interval = long(as_int(t[1], k));
    else if (k == "trace") arity(1), c.trace_path = t[1];
    else if (k == "step-size") arity(1), c.step_size = as_num(t[1], k);
    else if (k == "estimator") {
      arity(1);
      if (t[1] != "literal" && t[1] != "physical")
        throw std::runtime_error("config: key 'estimator' expects literal or physical, got '" + t[1] + "'");
      c.physical = t[1] == "physical";
    }
    else if (k == "weight") {
      arity(5);
      c.weight_overrides[atomic_number(t[1])] = {as_num(t[2], k), as_num(t[3], k), as_num(t[4], k), as_num(t[5], k)};
    } else
      throw std::runtime_error("config: unknown key '" + k + "'");
  }
  return c;
}

RunConfig parse_config_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open config file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return parse_config_text(ss.str());
}

std::uint64_t fnv1a64(const std::string& bytes) {
  std::uint64_t h = 14695981039346656037ull;
  for (unsigned char c : bytes) h = (h ^ c) * 1099511628211ull;
  return h;
}

std::string canonical_config_text(const RunConfig& c) {  // driver.cpp:140-159, keys sorted
  std::ostringstream os;
  os << "blocksize " << c.block_size << "\n" << "burnin " << c.burn_in << "\n";
  if (!c.checkpoint_path.empty()) os << "checkpoint " << c.checkpoint_path << "\n";
  os << "checkpoint-interval " << c.checkpoint_interval << "\n" << "seed " << c.seed << "\n";
  os << "spinors " << c.spinor_path << "\n";
  if (c.step_size) os << "step-size " << format_double(*c.step_size) << "\n";
  if (c.physical) os << "estimator physical\n";
  if (c.steps) os << "steps " << *c.steps << "\n";
  if (c.target_rel_err) os << "target-rel-err " << format_double(*c.target_rel_err) << "\n";
  if (!c.trace_path.empty()) os << "trace " << c.trace_path << "\n";
  os << "walkers " << c.walkers << "\n";
  put_weights(os, c);
  os << "workers " << c.workers << "\n";
  return os.str();
}

std::uint64_t config_hash(const RunConfig& c, std::uint64_t spinor_hash) {  // driver.cpp:161-172
  std::ostringstream os;
  os << "blocksize " << c.block_size << "\n" << "burnin " << c.burn_in << "\n";
  os << "spinorhash " << spinor_hash << "\n";
  if (c.step_size) os << "step-size " << format_double(*c.step_size) << "\n";
  if (c.physical) os << "estimator physical\n";
  os << "walkers " << c.walkers << "\n";
  put_weights(os, c);
  return fnv1a64(os.str());
}

std::uint64_t hash_file_contents(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open file for hashing: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return fnv1a64(ss.str());
}

MergedEstimate merge_estimates(const std::vector<WorkerSummary>& parts) {  // driver.cpp:183-196
  if (parts.empty()) throw std::invalid_argument("merge: no records");
  MergedEstimate out;
  for (const auto& p : parts) out.total_steps += p.steps;
  if (out.total_steps == 0) throw std::invalid_argument("merge: no accumulated steps");
  double var = 0.0;
  for (const auto& p : parts) {
    const double f = double(p.steps) / double(out.total_steps);
    out.value += f * p.mean;
    var += f * f * p.sigma_bar * p.sigma_bar;
  }
  out.sigma_bar = std::sqrt(var);
  return out;
}

long long worker_share(long long total, int workers, int index) {  // driver.cpp:307-309
  return total / workers + (index < total % workers ? 1 : 0);
}

// ------------------------------------------------------------------ device worker
void check_dev(int rc, const mcmp2dev_t* h) {
  if (rc == MCMP2DEV_OK) return;
  const std::string msg = mcmp2dev_last_error(h);
  if (rc == MCMP2DEV_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

DeviceWorker::DeviceWorker(const SpinorSet& s, const WeightSpec& w, const RunConfig& cfg, int index, int device)
    : acc(cfg.block_size), index_(index), walkers_(cfg.walkers), cfg_(&cfg) {
  DeviceSystem sys = make_device_system(s, w, cfg.physical ? MCMP2DEV_ESTIMATOR_PHYSICAL : MCMP2DEV_ESTIMATOR_LITERAL);
  check_dev(mcmp2dev_create(&sys.view, device, cfg.walkers, &h_), nullptr);
}

DeviceWorker::DeviceWorker(std::shared_ptr<DeviceBatch> batch, int ens, const RunConfig& cfg, int index)
    : acc(cfg.block_size), index_(index), walkers_(cfg.walkers), h_(batch->h), cfg_(&cfg), batch_(std::move(batch)),
      ens_(ens) {}

DeviceWorker::~DeviceWorker() {
  if (!batch_) mcmp2dev_destroy(h_);
}

DeviceBatch::~DeviceBatch() { mcmp2dev_destroy(h); }

void DeviceWorker::init_and_burn_in() {  // driver.cpp:354-358 (+ step-size extension)
  if (batch_) {  // the whole batch at its first worker: ensemble e = init_ensemble(m, seed, first + e)
    if (batch_->ready) return;
    check_dev(mcmp2dev_init_batch(h_, batch_->nens, walkers_, cfg_->seed, std::uint32_t(batch_->first)), h_);
    batch_->ready = true;
    batch_->states_valid = false;
  } else {
    check_dev(mcmp2dev_init_ensemble(h_, walkers_, cfg_->seed, std::uint32_t(index_)), h_);
  }
  if (cfg_->step_size) check_dev(mcmp2dev_set_sigma_step(h_, *cfg_->step_size), h_);
  check_dev(mcmp2dev_burn_in(h_, cfg_->burn_in, cfg_->step_size ? 0 : 1), h_);
  check_dev(mcmp2dev_prepare(h_), h_);
  if (batch_) batch_->states_valid = false;
}

void DeviceWorker::advance(long long nsteps) {  // driver.cpp:440-450
  if (nsteps <= 0) return;
  if (batch_) throw std::logic_error("DeviceWorker::advance: batched workers advance through advance_batch");
  values_.resize(nsteps);
  imags_.resize(nsteps);
  check_dev(mcmp2dev_advance(h_, long(nsteps), values_.data(), imags_.data()), h_);
  for (long long s = 0; s < nsteps; ++s) acc.add(values_[s], imags_[s]);
  done += nsteps;
}

void DeviceWorker::advance_batch(DeviceBatch& b, const std::vector<DeviceWorker*>& ws,
                                 const std::vector<long long>& nsteps) {
  // the step shares of a batch differ by at most one, the extra steps at the lowest indices
  // (worker_share, driver.cpp:307-309), so the active ensembles are always a prefix
  long long done = 0, most = 0;
  for (long long n : nsteps) most = std::max(most, n);
  while (done < most) {
    int na = 0;
    while (na < b.nens && nsteps[na] > done) ++na;
    for (int e = na; e < b.nens; ++e)
      if (nsteps[e] > done) throw std::logic_error("advance_batch: step shares are not a prefix");
    long long n = most - done;
    for (int e = 0; e < na; ++e) n = std::min(n, nsteps[e] - done);
    b.values.resize(std::size_t(n) * b.nens);
    b.imags.resize(std::size_t(n) * b.nens);
    b.states_valid = false;
    check_dev(mcmp2dev_advance_batch(b.h, long(n), na, b.values.data(), b.imags.data()), b.h);
    for (int e = 0; e < na; ++e) {
      DeviceWorker& w = *ws[e];
      for (long long s = 0; s < n; ++s) w.acc.add(b.values[std::size_t(s) * b.nens + e], b.imags[std::size_t(s) * b.nens + e]);
      w.done += n;
    }
    done += n;
  }
}

const mcmp2dev_ensemble& DeviceBatch::state(int ens) {
  if (!states_valid) {
    states.assign(std::size_t(nens), mcmp2dev_ensemble{});
    state_walkers.resize(std::size_t(nens) * m * 9);
    for (int k = 0; k < nens; ++k) states[k].walkers = state_walkers.data() + std::size_t(k) * m * 9;
    check_dev(mcmp2dev_get_ensembles(h, states.data()), h);
    states_valid = true;
  }
  return states[std::size_t(ens)];
}

void DeviceWorker::get_state(mcmp2dev_ensemble* e) const {
  if (batch_) {
    const mcmp2dev_ensemble& s = batch_->state(ens_);
    double* w = e->walkers;
    *e = s;
    e->walkers = w;
    std::copy(s.walkers, s.walkers + std::size_t(s.m) * 9, w);
  } else {
    check_dev(mcmp2dev_get_ensemble(h_, e), h_);
  }
}

double DeviceWorker::acceptance() const {
  std::vector<double> w(std::size_t(walkers_) * 9);
  mcmp2dev_ensemble e{};
  e.walkers = w.data();
  get_state(&e);
  return e.proposed ? double(e.accepted) / double(e.proposed) : 0.0;
}

WorkerSummary DeviceWorker::summary() const {  // driver.cpp:207-216
  const double re = acc.real_sum(), im = acc.imag_sum();
  return WorkerSummary{index_, acc.count(), acc.mean(), acc.sigma_bar(), acceptance(),
                       re != 0.0 ? std::abs(im) / std::abs(re) : std::abs(im)};
}

std::string DeviceWorker::save_ensemble() const {  // sampler.cpp:95-105 + rng.cpp:76-81
  std::vector<double> w(std::size_t(walkers_) * 9);
  mcmp2dev_ensemble e{};
  e.walkers = w.data();
  get_state(&e);
  std::ostringstream os;
  os << e.m << ' ' << format_double(e.sigma_step) << ' ' << e.proposed << ' ' << e.accepted << '\n';
  os << e.rng_key[0] << ' ' << e.rng_key[1];
  for (auto c : e.rng_counter) os << ' ' << c;
  os << ' ' << e.rng_idx << '\n';
  for (int p = 0; p < e.m; ++p) {
    for (int k = 0; k < 9; ++k) os << (k ? " " : "") << format_double(w[std::size_t(p) * 9 + k]);
    os << '\n';
  }
  return os.str();
}

void DeviceWorker::load_ensemble(const std::string& text) {  // sampler.cpp:107-120
  std::istringstream is(text);
  mcmp2dev_ensemble e{};
  is >> e.m >> e.sigma_step >> e.proposed >> e.accepted;
  is >> e.rng_key[0] >> e.rng_key[1];
  for (auto& c : e.rng_counter) is >> c;
  is >> e.rng_idx;
  if (!is || e.m < 2) throw std::runtime_error("checkpoint: malformed ensemble record");
  std::vector<double> w(std::size_t(e.m) * 9);
  for (auto& v : w)
    if (!(is >> v)) throw std::runtime_error("checkpoint: malformed walker record");
  e.walkers = w.data();
  if (batch_) {
    if (!batch_->ready) {  // the batch's layout (ensembles, seed, streams); states loaded below
      check_dev(mcmp2dev_init_batch(h_, batch_->nens, walkers_, cfg_->seed, std::uint32_t(batch_->first)), h_);
      batch_->ready = true;
    }
    batch_->states_valid = false;
    check_dev(mcmp2dev_set_ensemble_at(h_, ens_, &e), h_);
  } else {
    check_dev(mcmp2dev_set_ensemble(h_, &e), h_);
  }
  check_dev(mcmp2dev_prepare(h_), h_);
}

// ------------------------------------------------------------------ checkpoint (driver.cpp:218-305)
// one worker's checkpoint record (driver.cpp:232-247) and trace lines (driver.cpp:311-321) as
// text: the Engine writes them itself, a multi-process driver sends them to the writing rank
std::string worker_record_text(const DeviceWorker& w) {
  std::ostringstream out;
  out << "worker " << w.index() << "\n" << "steps " << w.acc.count() << "\n";
  out << "sums " << format_double(w.acc.real_sum()) << ' ' << format_double(w.acc.imag_sum()) << "\n";
  out << "partial " << w.acc.in_block() << ' ' << format_double(w.acc.partial()) << "\n";
  out << "blocks " << w.acc.block_means().size() << "\n";
  for (double b : w.acc.block_means()) out << format_double(b) << "\n";
  out << "ensemble\n" << w.save_ensemble() << "end-worker\n";
  return out.str();
}

std::string worker_trace_text(const DeviceWorker& w) {
  std::ostringstream out;
  for (const auto& t : w.acc.trace()) out << t.n << ' ' << format_double(t.mean) << ' ' << format_double(t.sigma_bar) << "\n";
  return out.str();
}

namespace {
struct SavedWorker {
  int index = 0;
  long long steps = 0;
  double sum = 0, imag = 0, partial = 0;
  long in_block = 0;
  std::vector<double> means;
  std::string ensemble;  // WalkerEnsemble::save text
};

struct Checkpoint {
  std::uint64_t hash = 0;
  RunConfig config;
  std::vector<SavedWorker> workers;
};

Checkpoint read_checkpoint(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open checkpoint: " + path);
  std::string word;
  int version = 0;
  in >> word;
  if (word != "mcmp2-checkpoint") throw std::runtime_error("checkpoint: bad header");
  in >> version;
  if (version != 1) throw std::runtime_error("checkpoint: unsupported version");
  Checkpoint ck;
  in >> word >> ck.hash;
  if (word != "confighash") throw std::runtime_error("checkpoint: missing confighash");
  std::string line;
  std::getline(in, line);
  std::getline(in, line);
  if (line != "config-begin") throw std::runtime_error("checkpoint: missing config section");
  std::ostringstream cfg;
  while (std::getline(in, line) && line != "config-end") cfg << line << "\n";
  ck.config = parse_config_text(cfg.str());
  std::size_t nw = 0;
  in >> word >> nw;
  if (word != "workers") throw std::runtime_error("checkpoint: missing workers record");
  auto want = [&](const char* w) {
    in >> word;
    if (word != w) throw std::runtime_error(std::string("checkpoint: missing ") + (std::strcmp(w, "worker") == 0 ? "worker record" : w));
  };
  for (std::size_t k = 0; k < nw; ++k) {
    SavedWorker w;
    want("worker");
    in >> w.index;
    want("steps");
    in >> w.steps;
    want("sums");
    in >> w.sum >> w.imag;
    want("partial");
    in >> w.in_block >> w.partial;
    std::size_t nb = 0;
    want("blocks");
    in >> nb;
    w.means.resize(nb);
    for (auto& b : w.means) in >> b;
    want("ensemble");
    std::getline(in, line);
    std::ostringstream ens;
    int m = 0;
    {
      std::getline(in, line);  // m sigma proposed accepted
      ens << line << "\n";
      std::istringstream hs(line);
      hs >> m;
      std::getline(in, line);  // rng state
      ens << line << "\n";
      for (int p = 0; p < m && std::getline(in, line); ++p) ens << line << "\n";
    }
    w.ensemble = ens.str();
    want("end-worker");
    if (!in) throw std::runtime_error("checkpoint: truncated file");
    ck.workers.push_back(std::move(w));
  }
  return ck;
}

std::string header_text(std::uint64_t hash, const RunConfig& cfg, std::size_t nworkers) {
  std::ostringstream out;
  out << "mcmp2-checkpoint 1\n" << "confighash " << hash << "\n";
  out << "config-begin\n" << canonical_config_text(cfg) << "config-end\n";
  out << "workers " << nworkers << "\n";
  return out.str();
}

void write_checkpoint(const std::string& path, std::uint64_t hash, const RunConfig& cfg,
                      const std::vector<std::unique_ptr<DeviceWorker>>& workers) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream out(tmp);
    if (!out) throw std::runtime_error("cannot write checkpoint: " + tmp);
    out << header_text(hash, cfg, workers.size());
    for (const auto& w : workers) out << worker_record_text(*w);
    if (!out) throw std::runtime_error("failed writing checkpoint: " + tmp);
  }
  std::filesystem::rename(tmp, path);
}

// one saved record back into a worker; cached weights re-verified against recomputation
// (driver.cpp:360-373)
void restore_worker(DeviceWorker& w, const SavedWorker& s, const WeightSpec& spec, const RunConfig& cfg) {
  w.acc = BlockingAccumulator(cfg.block_size);
  w.acc.restore(s.steps, s.sum, s.imag, s.in_block, s.partial, s.means);
  w.done = s.steps;
  std::istringstream is(s.ensemble);
  int m;
  is >> m;
  if (m != cfg.walkers) throw std::runtime_error("checkpoint: walker count disagrees with config");
  std::string line;
  std::getline(is, line);
  std::getline(is, line);
  for (int p = 0; p < m; ++p) {
    double v[9];
    for (double& x : v) is >> x;
    const double g1 = spec.g({v[0], v[1], v[2]}), g2 = spec.g({v[3], v[4], v[5]});
    if (std::abs(g1 - v[6]) > 1e-12 * std::abs(g1) || std::abs(g2 - v[7]) > 1e-12 * std::abs(g2))
      throw std::runtime_error("checkpoint: cached walker weights disagree with recomputation");
  }
  w.load_ensemble(s.ensemble);
}

WorkerSummary summarize_saved(const SavedWorker& w, long block_size) {
  BlockingAccumulator a(block_size);
  a.restore(w.steps, w.sum, w.imag, w.in_block, w.partial, w.means);
  std::istringstream is(w.ensemble);
  int m;
  double sigma;
  long long prop = 0, acc = 0;
  is >> m >> sigma >> prop >> acc;
  const double re = a.real_sum(), im = a.imag_sum();
  return WorkerSummary{w.index, a.count(), a.mean(), a.sigma_bar(), prop ? double(acc) / double(prop) : 0.0,
                       re != 0.0 ? std::abs(im) / std::abs(re) : std::abs(im)};
}

void write_trace(const std::string& trace_path, const DeviceWorker& w) {  // driver.cpp:311-321
  const std::string path = trace_path + ".w" + std::to_string(w.index());
  {
    std::ofstream out(path + ".tmp");
    if (!out) throw std::runtime_error("cannot write trace file: " + path + ".tmp");
    out << worker_trace_text(w);
  }
  std::filesystem::rename(path + ".tmp", path);
}

void join_traces(const std::string& trace_path, std::size_t n) {  // driver.cpp:323-334
  {
    std::ofstream out(trace_path);
    if (!out) throw std::runtime_error("cannot write trace file: " + trace_path);
    for (std::size_t k = 0; k < n; ++k) {
      std::ifstream in(trace_path + ".w" + std::to_string(k));
      if (in) out << in.rdbuf();
    }
  }
  for (std::size_t k = 0; k < n; ++k) std::filesystem::remove(trace_path + ".w" + std::to_string(k));
}

class Engine {  // driver.cpp:336-475
 public:
  Engine(RunConfig cfg, std::vector<SavedWorker> restored, const RunHooks& hooks)
      : cfg_(std::move(cfg)), spinors_(load_spinor_set(cfg_.spinor_path)),
        hash_(config_hash(cfg_, hash_file_contents(cfg_.spinor_path))) {
    cfg_.validate();
    if (!spinors_.nuclei) throw std::runtime_error("spinor file has no nuclei record; the sampling weight needs it");
    spec_ = std::make_unique<WeightSpec>(*spinors_.nuclei, cfg_.weight_overrides);
    lambda_from_gap(spinors_);
    int ndev = hooks.device_count;
    if (ndev <= 0 && cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
    if (ndev <= 0) throw std::runtime_error("mcmp2: no CUDA device visible (the walker loop runs on the GPU only)");
    const int nw = restored.empty() ? cfg_.workers : int(restored.size());
    // workers in contiguous ranges per device; a range of several workers with walker counts
    // that suit batching runs as one batched handle (one launch sequence per step for all)
    for (int d = 0; d < ndev; ++d) {
      const int k0 = int((long long)d * nw / ndev), k1 = int((long long)(d + 1) * nw / ndev);
      if (k1 <= k0) continue;
      std::shared_ptr<DeviceBatch> batch;
      bool contiguous = true;
      for (int k = k0; k < k1; ++k)
        if ((restored.empty() ? k : restored[k].index) != (restored.empty() ? k0 : restored[k0].index) + (k - k0))
          contiguous = false;
      if (k1 - k0 > 1 && contiguous && cfg_.walkers % 16 == 0 && cfg_.walkers <= 480) {  // mcmp2dev_init_batch limits
        DeviceSystem sys =
            make_device_system(spinors_, *spec_, cfg_.physical ? MCMP2DEV_ESTIMATOR_PHYSICAL : MCMP2DEV_ESTIMATOR_LITERAL);
        batch = std::make_shared<DeviceBatch>();
        check_dev(mcmp2dev_create(&sys.view, d, (k1 - k0) * cfg_.walkers, &batch->h), nullptr);
      }
      for (int k = k0; k < k1; ++k) {
        const int index = restored.empty() ? k : restored[k].index;
        if (batch) {
          batch->first = restored.empty() ? k0 : restored[k0].index;
          batch->nens = k1 - k0;
          batch->m = cfg_.walkers;
          workers_.push_back(std::make_unique<DeviceWorker>(batch, k - k0, cfg_, index));
        } else {
          workers_.push_back(std::make_unique<DeviceWorker>(spinors_, *spec_, cfg_, index, d));
        }
      }
    }
    if (restored.empty()) {
      for (auto& w : workers_) w->init_and_burn_in();
    } else {
      for (std::size_t k = 0; k < restored.size(); ++k) {
        const SavedWorker& s = restored[k];
        DeviceWorker& w = *workers_[k];
        restore_worker(w, s, *spec_, cfg_);
      }
    }
  }

  RunReport drive(const RunHooks& hooks) {  // driver.cpp:376-420
    long intervals = 0;
    bool on_target = false;
    for (;;) {
      std::vector<long long> chunk(workers_.size(), cfg_.checkpoint_interval);
      if (cfg_.steps)
        for (std::size_t w = 0; w < workers_.size(); ++w)
          chunk[w] = std::min<long long>(cfg_.checkpoint_interval,
                                         worker_share(*cfg_.steps, cfg_.workers, workers_[w]->index()) - workers_[w]->done);
      advance_parallel(chunk);
      ++intervals;
      if (!cfg_.checkpoint_path.empty()) write_checkpoint(cfg_.checkpoint_path, hash_, cfg_, workers_);
      if (!cfg_.trace_path.empty())
        for (const auto& w : workers_) write_trace(cfg_.trace_path, *w);
      if (cfg_.steps) {
        bool all = true;
        for (const auto& w : workers_)
          if (w->done < worker_share(*cfg_.steps, cfg_.workers, w->index())) all = false;
        if (all) break;
      } else {
        bool ready = true;
        for (const auto& w : workers_)
          if (w->acc.block_means().empty()) ready = false;
        if (ready) {
          const MergedEstimate m = merged();
          if (m.sigma_bar > 0 && m.value != 0 && m.sigma_bar / std::abs(m.value) <= *cfg_.target_rel_err) {
            on_target = true;
            break;
          }
        }
      }
      if (hooks.abort_after_intervals > 0 && intervals >= hooks.abort_after_intervals) return report(false);
    }
    if (!cfg_.trace_path.empty()) join_traces(cfg_.trace_path, workers_.size());
    return report(on_target);
  }

 private:
  void advance_parallel(const std::vector<long long>& chunk) {  // driver.cpp:423-438
    std::vector<std::thread> threads;
    std::vector<std::exception_ptr> errors(workers_.size());
    for (std::size_t w = 0; w < workers_.size(); ++w) {
      const DeviceBatch* b = workers_[w]->batch();
      if (b && w > 0 && workers_[w - 1]->batch() == b) continue;  // the batch's first worker drives it
      threads.emplace_back([&, w, b] {
        try {
          if (b) {
            std::vector<DeviceWorker*> ws;
            std::vector<long long> n;
            for (std::size_t k = w; k < workers_.size() && workers_[k]->batch() == b; ++k) {
              ws.push_back(workers_[k].get());
              n.push_back(std::max<long long>(chunk[k], 0));
            }
            DeviceWorker::advance_batch(*const_cast<DeviceBatch*>(b), ws, n);
          } else {
            workers_[w]->advance(chunk[w]);
          }
        } catch (...) {
          errors[w] = std::current_exception();
        }
      });
    }
    for (auto& t : threads) t.join();
    for (auto& e : errors)
      if (e) std::rethrow_exception(e);
  }

  MergedEstimate merged() const {
    std::vector<WorkerSummary> parts;
    for (const auto& w : workers_) parts.push_back(w->summary());
    return merge_estimates(parts);
  }

  RunReport report(bool on_target) const {
    RunReport r;
    for (const auto& w : workers_) r.workers.push_back(w->summary());
    r.merged = merge_estimates(r.workers);
    r.stopped_on_target = on_target;
    return r;
  }

  RunConfig cfg_;
  SpinorSet spinors_;
  std::uint64_t hash_;
  std::unique_ptr<WeightSpec> spec_;
  std::vector<std::unique_ptr<DeviceWorker>> workers_;
};
}  // namespace

RunReport run(const RunConfig& cfg, const RunHooks& hooks) {  // driver.cpp:477-480
  Engine e(cfg, {}, hooks);
  return e.drive(hooks);
}

RunReport resume(const std::string& path, const RunHooks& hooks) {  // driver.cpp:482-491
  Checkpoint ck = read_checkpoint(path);
  if (config_hash(ck.config, hash_file_contents(ck.config.spinor_path)) != ck.hash)
    throw std::runtime_error("checkpoint: config hash mismatch (spinor file or physics settings changed)");
  Engine e(ck.config, std::move(ck.workers), hooks);
  return e.drive(hooks);
}

std::string checkpoint_header_text(const RunConfig& cfg, std::size_t nworkers) {
  return header_text(config_hash(cfg, hash_file_contents(cfg.spinor_path)), cfg, nworkers);
}

RunConfig checkpoint_config(const std::string& path, std::vector<int>* indices) {
  Checkpoint ck = read_checkpoint(path);
  if (config_hash(ck.config, hash_file_contents(ck.config.spinor_path)) != ck.hash)
    throw std::runtime_error("checkpoint: config hash mismatch (spinor file or physics settings changed)");
  if (indices)
    for (const auto& w : ck.workers) indices->push_back(w.index);
  return ck.config;
}

void restore_workers(const std::string& path, const WeightSpec& spec, const RunConfig& cfg,
                     const std::vector<DeviceWorker*>& ws) {
  const Checkpoint ck = read_checkpoint(path);
  for (DeviceWorker* w : ws) {
    const SavedWorker* rec = nullptr;
    for (const auto& s : ck.workers)
      if (s.index == w->index()) rec = &s;
    if (!rec) throw std::runtime_error("checkpoint: missing worker record");
    restore_worker(*w, *rec, spec, cfg);
  }
}

MergedEstimate merge_checkpoint_files(const std::vector<std::string>& paths,
                                      std::vector<WorkerSummary>* parts_out) {  // driver.cpp:502-521
  if (paths.empty()) throw std::invalid_argument("merge: no checkpoint files");
  std::vector<WorkerSummary> parts;
  std::uint64_t hash = 0;
  for (std::size_t i = 0; i < paths.size(); ++i) {
    const Checkpoint ck = read_checkpoint(paths[i]);
    if (i == 0) hash = ck.hash;
    else if (ck.hash != hash)
      throw std::runtime_error("merge: config hash mismatch between " + paths.front() + " and " + paths[i]);
    for (const auto& w : ck.workers) parts.push_back(summarize_saved(w, ck.config.block_size));
  }
  if (parts_out) *parts_out = parts;
  return merge_estimates(parts);
}

std::string format_report(const RunReport& r) {  // driver.cpp:523-539
  std::ostringstream os;
  os << "E2        = " << format_double(r.merged.value) << " hartree\n";
  os << "sigma_bar = " << format_double(r.merged.sigma_bar) << " hartree\n";
  os << "steps     = " << r.merged.total_steps << "\n";
  if (r.stopped_on_target) os << "stopped on target relative uncertainty\n";
  for (const auto& w : r.workers) {
    char a[32], b[32];
    std::snprintf(a, sizeof a, "%.3f", w.acceptance);
    std::snprintf(b, sizeof b, "%.2e", w.imag_ratio);
    os << "worker " << w.index << ": steps " << w.steps << ", I " << format_double(w.mean) << ", sigma_bar "
       << format_double(w.sigma_bar) << ", acceptance " << a << ", imag ratio " << b << "\n";
  }
  return os.str();
}

}  // namespace mcmp2
