// mcmp2.hpp — host side of the B200 MC-MP2 walker loop (libmcmp2host.so, CLI `mcmp2`).
//
// Re-hosts the reference's input and driver interface (reference proj/core/include/mcmp2/
// model.hpp, weights.hpp, estimator.hpp, driver.hpp) around the device C ABI
// (include/mcmp2dev.h): SPINOR-TEXT loading and validation, the sampling weight, the run
// config, Engine (one device handle per worker), checkpoint/resume, traces, merge and the
// report. Only Engine::advance differs from the reference: its body is
// mcmp2dev_advance + BlockingAccumulator::add in order (driver.cpp:440-450).
#pragma once

#include <complex>
#include <cstdint>
#include <map>
#include <optional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/mcmp2dev.h"

namespace mcmp2 {

using Complex = std::complex<double>;

struct Vec3 {
  double x = 0, y = 0, z = 0;
};

// ---- gaussian.hpp:19-31 (setup-time integrals) ----
double primitive_norm(int l, double zeta);
double boys_f0(double t);
double primitive_overlap(int la, int ma, double a, const Vec3& A, int lb, int mb, double b, const Vec3& B);

// ---- model.hpp ----
struct Nucleus {
  double charge;
  Vec3 position;
};
struct Primitive {
  double zeta, coeff;
};

// contracted real-solid-harmonic Gaussian normalised to unit self-overlap (model.hpp:40-58)
struct BasisFunction {
  BasisFunction(const Vec3& center, int l, int m, std::vector<Primitive> prims);
  Vec3 center;
  int l, m;
  std::vector<Primitive> primitives;
  std::vector<double> evaluation_coeffs;
};
double contracted_overlap(const BasisFunction& a, const BasisFunction& b);

struct PairPrefactors {
  double direct, exchange;
};
PairPrefactors mp2_pair_prefactors(int ncomp);

// SpinorSet (model.hpp:74-117); coefficients row-major [row][spinor]
struct SpinorSet {
  SpinorSet(int ncomp, std::vector<std::vector<BasisFunction>> basis, std::vector<Complex> coeff,
            std::vector<double> energies, int n_occ, int n_vir,
            std::optional<std::vector<Nucleus>> nuclei);
  int ncomp, n_occ, n_vir;
  std::vector<std::vector<BasisFunction>> basis;
  std::vector<Complex> coeff;
  std::vector<double> energies;
  std::optional<std::vector<Nucleus>> nuclei;
  int rows() const;
  int n_spinor() const { return n_occ + n_vir; }
  double orthonormality_deviation() const;
};
SpinorSet load_spinor_set(const std::string& path);
void save_spinor_set(const SpinorSet& s, const std::string& path);
std::string format_double(double x);

// ---- weights.hpp ----
struct WeightParams {
  double c1, zeta1, c2, zeta2;
};
const std::map<int, WeightParams>& default_weight_params();
std::string element_symbol(int z);
int atomic_number(const std::string& sym);

struct WeightSpec {  // weights.hpp:28-51
  WeightSpec(const std::vector<Nucleus>& nuclei, const std::map<int, WeightParams>& overrides = {});
  double g(const Vec3& r) const;
  double ng = 0;
  std::vector<Vec3> pos;
  std::vector<double> prim;   // [site][2][2] (coeff incl. norm, zeta)
  std::vector<double> zeta1;
};
double lambda_from_gap(const SpinorSet& s);

// flattened copy of a system in the C-ABI layout (include/mcmp2dev.h)
struct DeviceSystem {
  std::vector<int> channel_count, fn_lm, fn_prim_offset;
  std::vector<double> fn_center, prim_zeta, prim_coeff, coeff, energies, site_pos, site_prim, site_zeta1;
  mcmp2dev_system view{};
};
DeviceSystem make_device_system(const SpinorSet& s, const WeightSpec& w, int estimator);

// ---- estimator.hpp:60-97 ----
class BlockingAccumulator {
 public:
  explicit BlockingAccumulator(long block_size = 100);
  void add(double value, double imag = 0.0);
  long long count() const { return n_; }
  double mean() const { return n_ ? sum_ / double(n_) : 0.0; }
  double sigma() const;
  double sigma_bar() const;
  double real_sum() const { return sum_; }
  double imag_sum() const { return imag_sum_; }
  const std::vector<double>& block_means() const { return means_; }
  long in_block() const { return in_block_; }
  double partial() const { return partial_; }
  long block_size() const { return nb_; }
  struct TracePoint {
    long long n;
    double mean, sigma_bar;
  };
  std::vector<TracePoint> trace() const;
  void restore(long long n, double sum, double imag_sum, long in_block, double partial,
               std::vector<double> means);

 private:
  long nb_;
  long long n_ = 0;
  double sum_ = 0, imag_sum_ = 0, partial_ = 0;
  long in_block_ = 0;
  std::vector<double> means_;
};

// ---- driver.hpp ----
struct RunConfig {
  std::string spinor_path;
  std::optional<long long> steps;
  std::optional<double> target_rel_err;
  int walkers = 8;
  std::uint64_t seed = 1;
  int workers = 1;
  long block_size = 100;
  long burn_in = 1000;
  std::string checkpoint_path;
  long checkpoint_interval = 5000;
  std::string trace_path;
  std::map<int, WeightParams> weight_overrides;
  std::optional<double> step_size;  // extension: fixed sigma_step, no adaptation
  bool physical = false;            // extension: `estimator physical`, default literal
  void validate() const;
};
RunConfig parse_config_text(const std::string& text);
RunConfig parse_config_file(const std::string& path);
std::uint64_t fnv1a64(const std::string& bytes);
std::string canonical_config_text(const RunConfig& c);
std::uint64_t config_hash(const RunConfig& c, std::uint64_t spinor_hash);
std::uint64_t hash_file_contents(const std::string& path);

struct WorkerSummary {
  int index;
  long long steps;
  double mean, sigma_bar, acceptance, imag_ratio;
};
struct MergedEstimate {
  double value = 0, sigma_bar = 0;
  long long total_steps = 0;
};
struct RunReport {
  MergedEstimate merged;
  std::vector<WorkerSummary> workers;
  bool stopped_on_target = false;
};
MergedEstimate merge_estimates(const std::vector<WorkerSummary>& parts);
long long worker_share(long long total, int workers, int index);

struct RunHooks {
  long abort_after_intervals = -1;
  int device_count = 0;  // 0: all visible devices; workers are placed in contiguous ranges per device
};
RunReport run(const RunConfig& cfg, const RunHooks& hooks = {});
RunReport resume(const std::string& checkpoint_path, const RunHooks& hooks = {});
MergedEstimate merge_checkpoint_files(const std::vector<std::string>& paths,
                                      std::vector<WorkerSummary>* parts = nullptr);
std::string format_report(const RunReport& r);

// ---- one device worker: the unit the distributed runner and the bench drive ----
// Several workers of one device in one batched handle (include/mcmp2dev.h, batched ensembles):
// worker first + e is ensemble e (Philox stream first + e, driver.cpp:354-356).
struct DeviceBatch {
  mcmp2dev_t* h = nullptr;
  int first = 0, nens = 0, m = 0;
  bool ready = false;  // init_batch done
  std::vector<double> values, imags;
  // every ensemble's state in one bulk copy (mcmp2dev_get_ensembles), reused until the batch
  // advances or an ensemble is loaded: reports, traces and checkpoints of k workers cost two
  // device copies instead of k x 10
  std::vector<mcmp2dev_ensemble> states;
  std::vector<double> state_walkers;
  bool states_valid = false;
  const mcmp2dev_ensemble& state(int ens);
  DeviceBatch() = default;
  DeviceBatch(const DeviceBatch&) = delete;
  DeviceBatch& operator=(const DeviceBatch&) = delete;
  ~DeviceBatch();
};

class DeviceWorker {
 public:
  DeviceWorker(const SpinorSet& s, const WeightSpec& w, const RunConfig& cfg, int index, int device);
  DeviceWorker(std::shared_ptr<DeviceBatch> batch, int ens, const RunConfig& cfg, int index);
  // advances a batch's workers (in ensemble order) by their own step counts (driver.cpp:440-450)
  static void advance_batch(DeviceBatch& b, const std::vector<DeviceWorker*>& ws,
                            const std::vector<long long>& nsteps);
  const DeviceBatch* batch() const { return batch_.get(); }
  ~DeviceWorker();
  DeviceWorker(const DeviceWorker&) = delete;
  DeviceWorker& operator=(const DeviceWorker&) = delete;
  void init_and_burn_in();                       // init_ensemble + burn_in (driver.cpp:354-358)
  void advance(long long nsteps);                // driver.cpp:440-450
  WorkerSummary summary() const;                 // driver.cpp:207-216
  mcmp2dev_t* handle() { return h_; }
  int index() const { return index_; }
  BlockingAccumulator acc;
  long long done = 0;
  // ensemble record in WalkerEnsemble::save format (sampler.cpp:95-105)
  std::string save_ensemble() const;
  void load_ensemble(const std::string& text);
  double acceptance() const;
  const std::vector<double>& last_values() const { return values_; }
  const std::vector<double>& last_imags() const { return imags_; }

 private:
  void get_state(mcmp2dev_ensemble* e) const;
  int index_;
  int walkers_;
  mcmp2dev_t* h_ = nullptr;
  const RunConfig* cfg_;
  std::vector<double> values_, imags_;
  std::shared_ptr<DeviceBatch> batch_;  // non-null: h_ is the batch's handle, ensemble ens_
  int ens_ = 0;
};

void check_dev(int rc, const mcmp2dev_t* h);

// The checkpoint file in pieces, for a driver whose workers live in several processes
// (distributed.py): header (driver.cpp:222-230; hashes the spinor file), then every worker's
// record in worker order (driver.cpp:232-247); a worker's trace lines (driver.cpp:311-321).
std::string checkpoint_header_text(const RunConfig& cfg, std::size_t nworkers);
std::string worker_record_text(const DeviceWorker& w);
std::string worker_trace_text(const DeviceWorker& w);
// the stored config after the hash check of resume (driver.cpp:482-491); the saved worker indices
RunConfig checkpoint_config(const std::string& path, std::vector<int>* indices = nullptr);
// restores each worker from the record carrying its index (weights re-verified, driver.cpp:360-373)
void restore_workers(const std::string& path, const WeightSpec& spec, const RunConfig& cfg,
                     const std::vector<DeviceWorker*>& ws);

// ---- BASELINE config generator (host/generate.cpp) ----
SpinorSet generate_spinor_set(const std::string& name);  // cfg1..cfg4, cfg5-N
std::string generate_run_config(const std::string& name, const std::string& spinor_path);
void write_generated(const std::string& name, const std::string& dir);  // rethrows the reference exception type

}  // namespace mcmp2
