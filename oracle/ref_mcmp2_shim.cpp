// ref_mcmp2_shim.cpp — TEST INFRASTRUCTURE ONLY. C entry points over the reference's own
// hot-path code (rng, gaussian, model, weights, sampler, greens, estimator, driver .cpp, compiled
// unmodified from /root/reference by build_ref.sh against oracle/eigen_subset) so the tests can
// pin the oracle and the device path against the reference implementation itself:
//   ref2_system_load   load_spinor_set + WeightSpec(molecule, config weight lines) + TauSampler
//                      (as Engine's constructor, driver.cpp:338-346)
//   ref2_replay        mc_step_estimate at given walkers and tau (estimator.cpp:35-63), plus the
//                      direct / exchange sums from sample_term per pair (estimator.cpp:65-75)
//   ref2_evaluate      SpinorSet::evaluate_into (model.cpp:166-178)
//   ref2_g             WeightSpec::g (weights.cpp:92-99)
//   ref2_run_config    run(parse_config_text(text)) + format_report (driver.cpp:477-480, :523-539)
//   ref2_fixture       the deterministic oracle's fixtures (oracle.cpp: make_fixture, MP2 energy)
// Errors: return 1 (std::invalid_argument) or 2 (other exceptions), message in ref2_last_error.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "mcmp2/driver.hpp"
#include "mcmp2/estimator.hpp"
#include "mcmp2/model.hpp"
#include "mcmp2/oracle.hpp"
#include "mcmp2/sampler.hpp"
#include "mcmp2/weights.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
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

struct RefSystem {
  mcmp2::SpinorSet spinors;
  std::optional<mcmp2::WeightSpec> spec;
  std::optional<mcmp2::TauSampler> tau;
  explicit RefSystem(const std::string& path) : spinors(mcmp2::load_spinor_set(path)) {}
};

// the ensemble record of WalkerEnsemble::save (sampler.cpp:95-105) for walkers[m][8] =
// r1, r2, g1, g2; the estimator reads positions and g only
mcmp2::WalkerEnsemble make_ensemble(int m, const double* w) {
  std::ostringstream os;
  os << m << " 1 0 0\n" << mcmp2::PhiloxRng(1, 0) << '\n';
  for (int p = 0; p < m; ++p) {
    const double* x = w + 8 * p;
    for (int k = 0; k < 8; ++k) os << mcmp2::format_double(x[k]) << ' ';
    os << "1\n";
  }
  std::istringstream is(os.str());
  return mcmp2::WalkerEnsemble::load(is);
}
}  // namespace

// built with -fvisibility=hidden -Wl,-Bsymbolic: the reference's mcmp2:: symbols stay private
// to this library (the product host library and the oracle define mcmp2:: names of their own)
#define REF2_API __attribute__((visibility("default")))

extern "C" {

REF2_API const char* ref2_last_error(void) { return g_err.c_str(); }

REF2_API void* ref2_system_load(const char* spinor_path, const char* config_text) {
  RefSystem* s = nullptr;
  const int rc = guarded([&] {
    auto sys = std::make_unique<RefSystem>(spinor_path);
    // weight overrides as the driver parses them (driver.cpp:65-121); run-control keys are
    // supplied so the text validates
    std::string text = std::string("spinors ") + spinor_path + "\nsteps 1\n";
    std::istringstream in(config_text ? config_text : "");
    for (std::string line; std::getline(in, line);)
      if (line.rfind("weight", 0) == 0) text += line + "\n";
    const mcmp2::RunConfig cfg = mcmp2::parse_config_text(text);
    if (!sys->spinors.molecule()) throw std::runtime_error("spinor file has no nuclei record");
    sys->spec.emplace(*sys->spinors.molecule(), cfg.weight_overrides);
    sys->tau.emplace(mcmp2::lambda_from_gap(sys->spinors));
    s = sys.release();
  });
  return rc ? nullptr : s;
}

REF2_API void ref2_system_free(void* h) { delete static_cast<RefSystem*>(h); }

// ints: ncomp, n_occ, n_vir; dbls: ng, lambda
REF2_API int ref2_system_info(void* h, int* ints, double* dbls) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    ints[0] = s->spinors.ncomp();
    ints[1] = s->spinors.n_occ();
    ints[2] = s->spinors.n_vir();
    dbls[0] = s->spec->ng();
    dbls[1] = s->tau->lambda();
  });
}

// out[nsteps][6] = value, imag, direct re/im, exchange re/im (sums over p < q before / C(m,2))
REF2_API int ref2_replay(void* h, int m, long nsteps, const double* walkers, const double* tau, int pair_sums,
                double* out) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    mcmp2::EstimatorWorkspace ws(s->spinors, m);
    for (long st = 0; st < nsteps; ++st) {
      const mcmp2::WalkerEnsemble ens = make_ensemble(m, walkers + size_t(st) * m * 8);
      const mcmp2::StepEstimate e = mcmp2::mc_step_estimate(s->spinors, ens, tau[st], *s->spec, *s->tau, ws);
      double* o = out + 6 * st;
      o[0] = e.value;
      o[1] = e.imag;
      std::complex<double> d = 0, x = 0;
      if (pair_sums) {
        const auto& pairs = ens.pairs();
        for (int p = 0; p < m; ++p)
          for (int q = p + 1; q < m; ++q) {
            const mcmp2::SampleTerm t = mcmp2::sample_term(s->spinors, pairs[p], pairs[q], tau[st], *s->spec, *s->tau);
            d += t.direct;
            x += t.exchange;
          }
      }
      o[2] = d.real();
      o[3] = d.imag();
      o[4] = x.real();
      o[5] = x.imag();
    }
  });
}

// occ[n][ncomp][n_occ][2], vir[n][ncomp][n_vir][2]
REF2_API int ref2_evaluate(void* h, const double* pts, int n, double* occ, double* vir) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    const int nc = s->spinors.ncomp(), no = s->spinors.n_occ(), nv = s->spinors.n_vir();
    mcmp2::MatrixXcd o, v;
    for (int i = 0; i < n; ++i) {
      s->spinors.evaluate_into(mcmp2::Vec3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]), o, v);
      for (int x = 0; x < nc; ++x) {
        for (int k = 0; k < no; ++k) {
          occ[((size_t(i) * nc + x) * no + k) * 2] = o(x, k).real();
          occ[((size_t(i) * nc + x) * no + k) * 2 + 1] = o(x, k).imag();
        }
        for (int k = 0; k < nv; ++k) {
          vir[((size_t(i) * nc + x) * nv + k) * 2] = v(x, k).real();
          vir[((size_t(i) * nc + x) * nv + k) * 2 + 1] = v(x, k).imag();
        }
      }
    }
  });
}

REF2_API int ref2_g(void* h, const double* pts, int n, double* out) {
  return guarded([&] {
    auto* s = static_cast<RefSystem*>(h);
    for (int i = 0; i < n; ++i) out[i] = s->spec->g(mcmp2::Vec3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
  });
}

// the reference's deterministic oracle: the fixture's MP2 energy (oracle.cpp, make_fixture) and
// its SPINOR-TEXT (save_spinor_set), e.g. syn4c
REF2_API int ref2_fixture(const char* name, const char* spinor_out, double* e2) {
  return guarded([&] {
    const mcmp2::Fixture fx = mcmp2::make_fixture(name);
    *e2 = fx.e2;
    if (spinor_out && *spinor_out) mcmp2::save_spinor_set(fx.spinors, spinor_out);
  });
}

REF2_API int ref2_run_config(const char* text, char* report, int cap) {
  return guarded([&] {
    const mcmp2::RunReport r = mcmp2::run(mcmp2::parse_config_text(text));
    std::snprintf(report, size_t(cap), "%s", mcmp2::format_report(r).c_str());
  });
}

}  // extern "C"
