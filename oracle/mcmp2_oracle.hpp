// mcmp2_oracle.hpp — CPU restatement of the reference MC-MP2 walker loop.
//
// TEST INFRASTRUCTURE ONLY. This is the parity oracle for the B200 path: a
// plain C++20 (no Eigen) restatement of the reference's hot path and the driver
// semantics around it. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load it. The product
// (paper_2203_05632_b200/) never links or calls it.
//
// Every function cites the reference file:line it follows (paths relative to
// /root/reference/proj/core/). The reference itself cannot be built here (it needs
// Eigen3, absent), except rng.cpp, which oracle/_ref builds from the reference
// sources to pin the Philox restatement (see oracle/build_ref.sh).
//
// Pinning: Philox KATs (tests/test_rng.cpp:10-31) and the reference rng.cpp itself
// (oracle/_ref), FNV-1a KATs (tests/test_driver.cpp:41-45), s value (2/pi)^{3/4}
// (tests/test_model.cpp:32-37), g(0) (tests/test_weights.cpp:22-27), N_g = 4 pi
// (tests/test_weights.cpp:62-67), tau inverse CDF (tests/test_weights.cpp:114-120),
// guarded_exp (tests/test_greens.cpp:198-202), blocking hand examples
// (tests/test_estimator.cpp:185-253), and the integrand identities of
// tests/test_estimator.cpp:27-147 restated in tests/test_oracle_*.py.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <iosfwd>
#include <map>
#include <optional>
#include <string>
#include <vector>

namespace oracle {

using Complex = std::complex<double>;

struct Vec3 {
  double x = 0, y = 0, z = 0;
};
inline Vec3 operator+(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline Vec3 operator-(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline Vec3 operator*(const Vec3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
// Eigen's squaredNorm on a Vector3d sums in storage order: (x^2 + y^2) + z^2
inline double sqnorm(const Vec3& a) { return a.x * a.x + a.y * a.y + a.z * a.z; }

// ---------------------------------------------------------------- rng.cpp
// Philox4x32-10 (rng.cpp:17-64), stream split by counter word 3 (rng.cpp:41-44)
class Philox {
 public:
  Philox() = default;
  Philox(std::uint64_t seed, std::uint32_t stream = 0);
  static std::array<std::uint32_t, 4> block(const std::array<std::uint32_t, 4>& ctr,
                                            const std::array<std::uint32_t, 2>& key);
  std::uint32_t next_u32();
  std::uint64_t next_u64();
  double uniform();
  std::array<double, 3> gaussian3();
  bool operator==(const Philox&) const = default;
  // text form "k0 k1 c0 c1 c2 c3 idx" (rng.cpp:76-94)
  std::string save() const;
  static Philox load(std::istream& is);

  std::array<std::uint32_t, 2> key{0, 0};
  std::array<std::uint32_t, 4> counter{0, 0, 0, 0};
  std::array<std::uint32_t, 4> out{0, 0, 0, 0};
  std::uint32_t idx = 4;

 private:
  void refill();
};

// ---------------------------------------------------------------- gaussian.cpp
struct SolidTerm {
  int ix, iy, iz;
  double coef;
};
// monomial table of S_lm (gaussian.cpp:21-39, :56-85)
const SolidTerm* solid_harmonic_terms(int l, int m, int* count);
double solid_harmonic(int l, int m, const Vec3& d);  // gaussian.cpp:87-92
double primitive_norm(int l, double zeta);           // gaussian.cpp:94-97
double boys_f0(double t);                            // gaussian.cpp:99-104
double primitive_overlap(int la, int ma, double a, const Vec3& A, int lb, int mb, double b,
                         const Vec3& B);  // gaussian.cpp:106-128

// ---------------------------------------------------------------- model.cpp
struct Nucleus {
  double charge;
  Vec3 position;
};

struct Primitive {
  double zeta;
  double coeff;
};

class BasisFunction {  // model.cpp:30-64
 public:
  BasisFunction(const Vec3& center, int l, int m, std::vector<Primitive> prims);
  double value(const Vec3& r) const;
  Vec3 center;
  int l, m;
  std::vector<Primitive> primitives;
  std::vector<double> eval_coeffs;
};

double contracted_overlap(const BasisFunction& a, const BasisFunction& b);  // model.cpp:66-76

struct PairPrefactors {
  double direct, exchange;
};
PairPrefactors mp2_pair_prefactors(int ncomp);  // model.cpp:86-88

// model.cpp:90-178. Coefficients stored row-major: coeff[row * cols + col].
class SpinorSet {
 public:
  SpinorSet(int ncomp, std::vector<std::vector<BasisFunction>> basis, std::vector<Complex> coeff,
            std::vector<double> energies, int n_occ, int n_vir,
            std::optional<std::vector<Nucleus>> nuclei = std::nullopt, bool validate = true);
  int ncomp, n_occ, n_vir, rows;
  std::vector<std::vector<BasisFunction>> basis;
  std::vector<Complex> coeff;
  std::vector<double> energies;
  std::vector<int> row_offset;
  std::optional<std::vector<Nucleus>> nuclei;
  int n_spinor() const { return n_occ + n_vir; }
  double homo() const { return energies[n_occ - 1]; }
  double lumo() const { return energies[n_occ]; }
  double orthonormality_deviation() const;  // model.cpp:153-158
  // occ: ncomp x n_occ, vir: ncomp x n_vir, row-major (model.cpp:166-178)
  void evaluate_into(const Vec3& point, Complex* occ, Complex* vir, double* chi_scratch) const;
  int max_channel_size() const;
};

SpinorSet load_spinor_set(const std::string& path, bool validate = true);  // model.cpp:275-351
void save_spinor_set(const SpinorSet& set, const std::string& path);      // model.cpp:353-388
std::string format_double(double x);                                       // model.cpp:180-184

// ---------------------------------------------------------------- weights.cpp
struct WeightParams {
  double c1, zeta1, c2, zeta2;
};
const std::map<int, WeightParams>& default_weight_params();  // weights.cpp:28-37
std::string element_symbol(int z);
int atomic_number(const std::string& symbol);

class WeightSpec {  // weights.cpp:52-99
 public:
  WeightSpec(const std::vector<Nucleus>& nuclei, const std::map<int, WeightParams>& overrides = {});
  double g(const Vec3& r) const;
  double ng() const { return ng_; }
  struct SitePrim {
    double coeff, zeta;
  };
  struct Site {
    Vec3 position;
    std::vector<SitePrim> prims;
    double zeta1;
  };
  std::vector<Site> sites;

 private:
  double ng_ = 0;
};

class TauSampler {  // weights.cpp:103-111
 public:
  explicit TauSampler(double lambda);
  double lambda() const { return lambda_; }
  double sample(double u) const;
  double pdf(double tau) const;

 private:
  double lambda_;
};
double lambda_from_gap(const SpinorSet& s);  // weights.cpp:113-120

// ---------------------------------------------------------------- sampler.cpp
struct WalkerPair {  // sampler.hpp:13-17
  Vec3 r1, r2;
  double g1 = 0, g2 = 0, weight = 0;
};

struct WalkerEnsemble {  // sampler.hpp:19-49
  std::vector<WalkerPair> pairs;
  double sigma_step = 1.0;
  Philox rng;
  long long proposed = 0, accepted = 0;
  int m() const { return int(pairs.size()); }
  double acceptance_fraction() const {
    return proposed ? double(accepted) / double(proposed) : 0.0;
  }
  void save(std::ostream& os) const;       // sampler.cpp:95-105
  static WalkerEnsemble load(std::istream& is);  // sampler.cpp:107-120
};

WalkerEnsemble init_ensemble(int m, const std::vector<Nucleus>& nuclei, const WeightSpec& spec,
                             std::uint64_t seed, std::uint32_t stream = 0);  // sampler.cpp:21-47
int metropolis_step(WalkerEnsemble& ens, const WeightSpec& spec);           // sampler.cpp:49-79
void burn_in(WalkerEnsemble& ens, const WeightSpec& spec, long n_burn, bool adapt = true);

// ---------------------------------------------------------------- greens.cpp
double guarded_exp(double exponent, int spinor_index);  // greens.cpp:9-16

// greens.cpp:42-79: per-step cache of spinor values (raw and tau-weighted)
class TraceWorkspace {
 public:
  TraceWorkspace(const SpinorSet& s, int max_points);
  void load_points(const Vec3* pts, int n);
  void set_tau(double tau);
  // out: ncomp x ncomp row-major
  void occupied(int d, int o, Complex* out) const;
  void virtuals(int d, int o, Complex* out) const;
  int npoints = 0;

 private:
  const SpinorSet* s_;
  int nc_, no_, nv_, max_points_;
  std::vector<Complex> occ_, vir_, occw_, virw_;  // [point][x][i]
  std::vector<double> wocc_, wvir_, chi_;
};

// ---------------------------------------------------------------- estimator.cpp
struct SampleTerm {  // estimator.hpp:13-18
  Complex direct, exchange;
  double total() const { return (direct + exchange).real(); }
  double imag() const { return (direct + exchange).imag(); }
};

struct StepEstimate {  // estimator.hpp:23-26, plus the direct/exchange split for replay dumps
  double value = 0, imag = 0;
  Complex direct_sum{0, 0}, exchange_sum{0, 0};  // sums over pairs, before /C(m,2)
};

class EstimatorWorkspace {  // estimator.cpp:8-13
 public:
  EstimatorWorkspace(const SpinorSet& s, int m);
  SampleTerm pair_term(int p, int q, double inv_weight, const PairPrefactors& w);  // :15-33
  TraceWorkspace traces;
  std::vector<Vec3> points;
  // pair estimator convention: literal element-wise (reference default) or the
  // physical trace form Tr(o1 va) Tr(o2 vb), Tr(o1 vd o2 vc)
  bool physical = false;

 private:
  int nc_;
  std::vector<Complex> o1_, o2_, va_, vb_, vc_, vd_;
};

StepEstimate mc_step_estimate(const SpinorSet& s, const WalkerEnsemble& ens, double tau,
                              const WeightSpec& spec, const TauSampler& ts,
                              EstimatorWorkspace& ws);  // estimator.cpp:35-63
// restricted to walker rows p in [p_begin, p_end): the bounded CPU-baseline sample
StepEstimate mc_step_estimate_rows(const SpinorSet& s, const WalkerEnsemble& ens, double tau,
                                   const WeightSpec& spec, const TauSampler& ts,
                                   EstimatorWorkspace& ws, int p_begin, int p_end,
                                   long long* npairs_out);
SampleTerm sample_term(const SpinorSet& s, const WalkerPair& p, const WalkerPair& q, double tau,
                       const WeightSpec& spec, const TauSampler& ts,
                       bool physical = false);  // estimator.cpp:65-75

class BlockingAccumulator {  // estimator.cpp:77-131
 public:
  explicit BlockingAccumulator(long block_size = 100);
  void add(double value, double imag = 0.0);
  long long count() const { return n_; }
  long block_size() const { return nb_; }
  double mean() const { return n_ ? sum_ / double(n_) : 0.0; }
  double sigma() const;
  double sigma_bar() const;
  double imag_sum() const { return imag_sum_; }
  double real_sum() const { return sum_; }
  const std::vector<double>& block_means() const { return block_means_; }
  struct TracePoint {
    long long n;
    double mean, sigma_bar;
  };
  std::vector<TracePoint> trace() const;
  void restore(long long n, double sum, double imag_sum, long in_block, double partial,
               std::vector<double> block_means);
  long in_block() const { return in_block_; }
  double partial() const { return partial_; }

 private:
  long nb_;
  long long n_ = 0;
  double sum_ = 0, imag_sum_ = 0, partial_ = 0;
  long in_block_ = 0;
  std::vector<double> block_means_;
};

// ---------------------------------------------------------------- driver.cpp
struct RunConfig {  // driver.hpp:17-32 (+ `step-size` extension)
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
  std::optional<double> step_size;  // extension: fixed sigma_step, burn-in without adaptation
  bool physical = false;            // extension: `estimator physical`
  void validate() const;            // driver.cpp:50-63
};

RunConfig parse_config_text(const std::string& text);  // driver.cpp:65-121
std::uint64_t fnv1a64(const std::string& bytes);       // driver.cpp:131-138
std::string canonical_config_text(const RunConfig& c);  // driver.cpp:140-159
std::uint64_t config_hash(const RunConfig& c, std::uint64_t spinor_hash);  // driver.cpp:161-172
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
MergedEstimate merge_estimates(const std::vector<WorkerSummary>& parts);  // driver.cpp:183-196
long long worker_share(long long total, int workers, int index);         // driver.cpp:307-309

struct StepRecord {  // replay dump row: positions used by the step's estimate
  double tau;
  std::vector<double> walkers;  // m x {r1x r1y r1z r2x r2y r2z g1 g2}
  StepEstimate est;
};
struct RunHooks {
  long abort_after_intervals = -1;                 // driver.hpp:70-72
  std::vector<std::vector<StepRecord>>* record = nullptr;  // per worker replay dump
};
RunReport run(const RunConfig& cfg, const RunHooks& hooks = {});          // driver.cpp:477-480
RunReport resume(const std::string& checkpoint, const RunHooks& hooks = {});  // :482-491
MergedEstimate merge_checkpoint_files(const std::vector<std::string>& paths,
                                      std::vector<WorkerSummary>* parts = nullptr);
std::string format_report(const RunReport& r);  // driver.cpp:523-539

}  // namespace oracle
