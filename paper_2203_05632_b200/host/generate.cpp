// generate.cpp — synthetic SPINOR-TEXT inputs and run configs for the BASELINE.json configs
// (SURVEY.md section 8(d) "Synthetic inputs"). Public datasets are not involved: the paper's
// Dirac-Hartree-Fock spinors are unavailable, so each config is a seeded synthetic set with
// the config's shapes.
//
// Construction (pattern of the reference's syn4c fixture, oracle.cpp:346-393, generalised):
//  * 4 channels (L alpha, L beta, S alpha, S beta); L lists identical, S lists identical.
//  * kinetic balance: every L shell (l, zeta) contributes S shells l-1 (if l > 0) and l+1 with
//    the same exponent and centre (the exact sigma.p gradient of an l >= 1 function has an
//    r^2 S_{l-1} part that SPINOR-TEXT cannot express; SURVEY finding 4).
//  * coefficients: seeded Philox complex vectors U(-1/2,1/2) + i U(-1/2,1/2), Gram-Schmidt
//    twice in the block-diagonal S metric, normalised, followed by the time-reversal partner
//    (La, Lb, Sa, Sb) -> (-Lb*, La*, -Sb*, Sa*) (oracle.cpp:346-355), so columns are Kramers
//    pairs and the literal estimator stays real (SURVEY finding 3).
//  * energies: one value per Kramers pair, sorted ascending per block.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <numbers>
#include <sstream>
#include <stdexcept>

#include "../csrc/philox.h"
#include "mcmp2.hpp"

namespace mcmp2 {

namespace {

struct Shell {
  Vec3 center;
  int l;
  double zeta;
  std::vector<Primitive> prims;  // contracted shell when non-empty (else one unit primitive)
};

struct Recipe {
  std::string name;
  std::vector<Nucleus> nuclei;
  std::vector<Shell> shells;  // L-channel shells
  int occ_pairs;
  double occ_lo, occ_hi;   // uniform
  double vir_lo, vir_hi;   // log-uniform
  bool occ_fixed = false;  // cfg1: all occupied pairs at occ_lo
  int walkers;
  long long steps;
  std::optional<double> step_size;
  std::vector<std::string> weights;  // weight lines
  std::uint64_t seed;
  int ncomp = 4;  // 1: real spatial orbitals (L only); 2: (alpha, beta) Kramers pairs; 4: Dirac
};

void even_tempered(std::vector<Shell>& out, const Vec3& c, int l, int n, double base, double ratio) {
  double z = base;
  for (int k = 0; k < n; ++k, z *= ratio) out.push_back({c, l, z, {}});
}

// sequential reference-order Philox uniforms (rng.cpp:46-64)
struct Uniforms {
  mcmp2dev::StreamReader r;
  explicit Uniforms(std::uint64_t seed) : r(std::uint32_t(seed), std::uint32_t(seed >> 32), 0x5eedu, 0) {}
  double next() { return r.uniform(); }
};

Recipe recipe(const std::string& name) {
  Recipe r;
  r.name = name;
  const Vec3 o{0, 0, 0};
  if (name == "cfg1") {  // 2e atom, 12 even-tempered s (0.05 2.5^k), 1 occ pair at -0.9
    r.nuclei = {{2.0, o}};
    even_tempered(r.shells, o, 0, 12, 0.05, 2.5);
    r.occ_pairs = 1;
    r.occ_lo = r.occ_hi = -0.9;
    r.occ_fixed = true;
    r.vir_lo = 0.1, r.vir_hi = 50.0;
    r.walkers = 16;
    r.steps = 2000;
    r.step_size = 0.3;
    r.weights = {"weight He 0.3 0.2 0.7 1.5"};
    r.seed = 0x22030001ull;
  } else if (name == "cfg2") {  // 10e atom, 14s (0.03 2.7^k) 9p (0.05 2.6^k)
    r.nuclei = {{10.0, o}};
    even_tempered(r.shells, o, 0, 14, 0.03, 2.7);
    even_tempered(r.shells, o, 1, 9, 0.05, 2.6);
    r.occ_pairs = 5;
    r.occ_lo = -30.0, r.occ_hi = -0.7;
    r.vir_lo = 0.2, r.vir_hi = 400.0;
    r.walkers = 128;
    r.steps = 10000;
    r.weights = {"weight Ne 0.5 0.3 1.5 2.5"};
    r.seed = 0x22030002ull;
  } else if (name == "cfg3") {  // 18e diatomic Cl-H, 17s12p4d + 6s2p, R = 2.41
    const Vec3 h{0, 0, 2.41};
    r.nuclei = {{17.0, o}, {1.0, h}};
    even_tempered(r.shells, o, 0, 17, 0.04, 2.5);
    even_tempered(r.shells, o, 1, 12, 0.06, 2.5);
    even_tempered(r.shells, o, 2, 4, 0.15, 2.5);
    even_tempered(r.shells, h, 0, 6, 0.05, 2.8);
    even_tempered(r.shells, h, 1, 2, 0.3, 3.0);
    r.occ_pairs = 9;
    r.occ_lo = -110.0, r.occ_hi = -0.5;
    r.vir_lo = 0.1, r.vir_hi = 2000.0;
    r.walkers = 512;
    r.steps = 10000;
    r.weights = {"weight Cl 0.8 0.3 2.0 0.6"};
    r.seed = 0x22030003ull;
  } else if (name == "cfg4") {  // 54e diatomic I-H, 24s20p14d + 6s2p, R = 3.04
    const Vec3 h{0, 0, 3.04};
    r.nuclei = {{53.0, o}, {1.0, h}};
    even_tempered(r.shells, o, 0, 24, 0.03, 2.3);
    even_tempered(r.shells, o, 1, 20, 0.045, 2.3);
    even_tempered(r.shells, o, 2, 14, 0.1, 2.3);
    even_tempered(r.shells, h, 0, 6, 0.05, 2.8);
    even_tempered(r.shells, h, 1, 2, 0.3, 3.0);
    r.occ_pairs = 27;
    r.occ_lo = -1200.0, r.occ_hi = -0.4;
    r.vir_lo = 0.1, r.vir_hi = 1.0e4;
    r.walkers = 2048;
    r.steps = 20000;
    r.weights = {"weight I 0.1 0.1 0.8 0.6"};
    r.seed = 0x22030004ull;
  } else if (name == "syn1c" || name == "syn2c") {  // small H2-like test sets (contracted s)
    const Vec3 h{0, 0, 1.4};
    r.nuclei = {{1.0, o}, {1.0, h}};
    for (const Vec3& c : {o, h}) {
      r.shells.push_back({c, 0, 0.0, {{3.4, 0.15}, {0.62, 0.53}, {0.17, 0.44}}});
      r.shells.push_back({c, 0, 0.12, {}});
      r.shells.push_back({c, 1, 0.8, {}});
    }
    r.ncomp = name == "syn1c" ? 1 : 2;
    r.occ_pairs = 1;
    r.occ_lo = r.occ_hi = -0.6;
    r.occ_fixed = true;
    r.vir_lo = 0.2, r.vir_hi = 5.0;
    r.walkers = 8;
    r.steps = 2000;
    r.seed = name == "syn1c" ? 0x22031001ull : 0x22032001ull;
  } else if (name.rfind("cfg5-", 0) == 0) {  // size sweep: single centre, Z = n_elec
    const int n = std::stoi(name.substr(5));
    static const std::map<int, std::string> el = {{2, "He"}, {10, "Ne"}, {18, "Ar"},
                                                  {36, "Kr"}, {54, "Xe"}, {86, "Rn"}};
    if (!el.count(n)) throw std::invalid_argument("generate: cfg5 n_elec must be one of 2,10,18,36,54,86");
    r.nuclei = {{double(n), o}};
    // basis grows with n_elec: s 6 + n/3, p n/4, d n/8 (even-tempered)
    even_tempered(r.shells, o, 0, 6 + n / 3, 0.03, 2.4);
    if (n / 4) even_tempered(r.shells, o, 1, n / 4, 0.045, 2.4);
    if (n / 8) even_tempered(r.shells, o, 2, n / 8, 0.1, 2.4);
    r.occ_pairs = n / 2;
    r.occ_lo = n <= 2 ? -0.9 : -0.5 * n * n / 4.0, r.occ_hi = n <= 2 ? -0.9 : -0.4;
    r.occ_fixed = n <= 2;
    r.vir_lo = 0.1, r.vir_hi = 50.0 * n;
    r.walkers = 8192;
    r.steps = 0;  // run to target-rel-err 0.01
    const std::map<std::string, std::string> w = {{"He", "0.3 0.2 0.7 1.5"},  {"Ne", "0.5 0.3 1.5 2.5"},
                                                  {"Ar", "0.8 0.3 2.0 0.6"},  {"Kr", "0.8 0.35 2.0 0.6"},
                                                  {"Xe", "0.1 0.1 0.8 0.6"},  {"Rn", "0.05 0.6 4.0 0.8"}};
    r.weights = {"weight " + el.at(n) + " " + w.at(el.at(n))};
    r.seed = 0x22030500ull + std::uint64_t(n);
  } else if (name == "wide") {  // stress set: n_vir 446 > 384 (the INT8 path's two-pass slicing)
    r.nuclei = {{54.0, o}};
    even_tempered(r.shells, o, 0, 30, 0.02, 2.0);
    even_tempered(r.shells, o, 1, 30, 0.03, 2.0);
    even_tempered(r.shells, o, 2, 26, 0.05, 2.0);
    r.occ_pairs = 27;
    r.occ_lo = -1200.0, r.occ_hi = -0.4;
    r.occ_fixed = false;
    r.vir_lo = 0.1, r.vir_hi = 1e4;
    r.walkers = 2048;
    r.steps = 2000;
    r.weights = {"weight Xe 0.1 0.1 0.8 0.6"};
    r.seed = 0x22039001ull;
  } else {
    throw std::invalid_argument("generate: unknown config '" + name + "' (cfg1..cfg4, cfg5-N, syn1c, syn2c, wide)");
  }
  return r;
}

// (l, m) functions of one shell in SPINOR-TEXT order m = -l..l
void shell_functions(const Shell& s, std::vector<BasisFunction>& out) {
  for (int m = -s.l; m <= s.l; ++m)
    out.emplace_back(s.center, s.l, m, s.prims.empty() ? std::vector<Primitive>{{s.zeta, 1.0}} : s.prims);
}

}  // namespace

SpinorSet generate_spinor_set(const std::string& name) {
  const Recipe r = recipe(name);
  std::vector<BasisFunction> L, S;
  for (const auto& sh : r.shells) shell_functions(sh, L);
  if (r.ncomp == 4)
    for (const auto& sh : r.shells) {  // kinetic-balance partners l -> l-1, l+1
      if (sh.prims.size() > 1) throw std::invalid_argument("generate: kinetic balance of contracted shells");
      if (sh.l > 0) shell_functions({sh.center, sh.l - 1, sh.zeta, {}}, S);
      shell_functions({sh.center, sh.l + 1, sh.zeta, {}}, S);
    }
  const int nc = r.ncomp;
  const int nL = int(L.size()), nS = int(S.size());
  const int R = nc == 4 ? 2 * nL + 2 * nS : nc * nL;
  const int npairs = nL;  // n_p = nc/2 * 2 n_L positive-energy spinors (1c: n_L orbitals)
  const int ncols = nc == 1 ? nL : 2 * npairs;

  // channel overlap matrices
  auto overlap = [](const std::vector<BasisFunction>& b) {
    const int n = int(b.size());
    std::vector<double> s(std::size_t(n) * n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) s[std::size_t(i) * n + j] = s[std::size_t(j) * n + i] = contracted_overlap(b[i], b[j]);
    return s;
  };
  const std::vector<double> SL = overlap(L), SS = overlap(S);
  const int off[4] = {0, nL, 2 * nL, 2 * nL + nS};
  const int len[4] = {nL, nL, nS, nS};
  auto apply_s = [&](const std::vector<Complex>& v) {
    std::vector<Complex> out(R, Complex(0, 0));
    for (int c = 0; c < nc; ++c) {
      const std::vector<double>& Sm = c < 2 ? SL : SS;
      const int n = len[c];
      for (int i = 0; i < n; ++i) {
        Complex acc(0, 0);
        for (int j = 0; j < n; ++j) acc += Sm[std::size_t(i) * n + j] * v[off[c] + j];
        out[off[c] + i] = acc;
      }
    }
    return out;
  };
  auto dot = [&](const std::vector<Complex>& a, const std::vector<Complex>& b) {  // a^H b
    Complex acc(0, 0);
    for (int i = 0; i < R; ++i) acc += std::conj(a[i]) * b[i];
    return acc;
  };
  auto kramers = [&](const std::vector<Complex>& v) {
    std::vector<Complex> w(R);
    for (int d = 0; d < nc / 2; ++d) {
      const int a = off[2 * d], b = off[2 * d + 1], n = len[2 * d];
      for (int i = 0; i < n; ++i) {
        w[a + i] = -std::conj(v[b + i]);
        w[b + i] = std::conj(v[a + i]);
      }
    }
    return w;
  };

  Uniforms u(r.seed);
  // energies (one per Kramers pair), drawn before the coefficients
  std::vector<double> occ(r.occ_pairs), vir(npairs - r.occ_pairs);
  if (r.occ_pairs > npairs) throw std::invalid_argument("generate: more occupied pairs than basis pairs");
  if (nc == 1) vir.resize(nL - r.occ_pairs);
  for (auto& e : occ) e = r.occ_fixed ? r.occ_lo : r.occ_lo + (r.occ_hi - r.occ_lo) * u.next();
  for (auto& e : vir) e = std::exp(std::log(r.vir_lo) + (std::log(r.vir_hi) - std::log(r.vir_lo)) * u.next());
  std::sort(occ.begin(), occ.end());
  std::sort(vir.begin(), vir.end());
  std::vector<double> eps;
  const int per = nc == 1 ? 1 : 2;  // spinors per energy
  for (double e : occ) eps.insert(eps.end(), std::size_t(per), e);
  for (double e : vir) eps.insert(eps.end(), std::size_t(per), e);

  std::vector<std::vector<Complex>> cols, scols;  // columns and S * columns
  for (int p = 0; p < (nc == 1 ? ncols : npairs); ++p) {
    std::vector<Complex> v(R);
    for (auto& c : v) {
      const double re = u.next() - 0.5;
      const double im = nc == 1 ? 0.0 : u.next() - 0.5;  // 1c: real orbitals
      c = Complex(re, im);
    }
    for (int rep = 0; rep < 2; ++rep)
      for (std::size_t j = 0; j < cols.size(); ++j) {
        const Complex proj = dot(scols[j], v);  // C_j^H S v
        for (int i = 0; i < R; ++i) v[i] -= cols[j][i] * proj;
      }
    std::vector<Complex> sv = apply_s(v);
    const double nrm = std::sqrt(dot(v, sv).real());
    for (auto& c : v) c /= nrm;
    for (auto& c : sv) c /= nrm;
    std::vector<Complex> k = kramers(v);
    std::vector<Complex> sk = apply_s(k);
    cols.push_back(std::move(v));
    scols.push_back(std::move(sv));
    if (nc == 1) continue;
    cols.push_back(std::move(k));
    scols.push_back(std::move(sk));
  }
  std::vector<Complex> coeff(std::size_t(R) * ncols);
  for (int j = 0; j < ncols; ++j)
    for (int i = 0; i < R; ++i) coeff[std::size_t(i) * ncols + j] = cols[j][i];
  std::vector<std::vector<BasisFunction>> channels;
  if (nc == 4) channels = {L, L, S, S};
  else if (nc == 2) channels = {L, L};
  else channels = {L};
  const int nocc = per * r.occ_pairs;
  return SpinorSet(nc, std::move(channels), std::move(coeff), std::move(eps), nocc, ncols - nocc, r.nuclei);
}

std::string generate_run_config(const std::string& name, const std::string& spinor_path) {
  const Recipe r = recipe(name);
  std::ostringstream os;
  os << "# " << name << " (BASELINE.json configs; synthetic seeded inputs, see host/generate.cpp)\n";
  os << "spinors " << spinor_path << "\n";
  if (r.steps > 0) os << "steps " << r.steps << "\n";
  else os << "target-rel-err 0.01\ncheckpoint-interval 100\n";
  os << "walkers " << r.walkers << "\n";
  if (r.step_size) os << "step-size " << format_double(*r.step_size) << "\n";
  for (const auto& w : r.weights) os << w << "\n";
  return os.str();
}

void write_generated(const std::string& name, const std::string& dir) {
  const std::string sp = dir + "/" + name + ".spinor";
  save_spinor_set(generate_spinor_set(name), sp);
  std::ofstream c(dir + "/" + name + ".conf");
  if (!c) throw std::runtime_error("cannot write " + dir + "/" + name + ".conf");
  c << generate_run_config(name, sp);
}

}  // namespace mcmp2
