// model.cpp — setup-time host code: Gaussian integrals for normalisation and validation,
// the SPINOR-TEXT reader/writer, SpinorSet validation, the sampling weight WeightSpec and
// the flattening of a system into the device C ABI. Follows reference
// proj/core/src/gaussian.cpp, model.cpp, weights.cpp (cited per function).
#include <algorithm>
#include <thread>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <numbers>
#include <sstream>
#include <stdexcept>

#include "mcmp2.hpp"

namespace mcmp2 {

namespace {
constexpr double kPi = std::numbers::pi;

struct Mono {
  int e[3];
  double c;
};

// real solid harmonics S_lm as monomials (gaussian.cpp:21-39); key = (l, m)
const std::vector<Mono>& monomials(int l, int m) {
  static const std::map<std::pair<int, int>, std::vector<Mono>> table = [] {
    const double s00 = 0.28209479177387814, s1 = 0.4886025119029199, s2a = 1.0925484305920792,
                 s2b = 0.31539156525252005, s2c = 0.5462742152960396, s3a = 0.5900435899266435,
                 s3b = 2.890611442640554, s3c = 0.4570457994644658, s3d = 0.3731763325901154;
    std::map<std::pair<int, int>, std::vector<Mono>> t;
    t[{0, 0}] = {{{0, 0, 0}, s00}};
    t[{1, -1}] = {{{0, 1, 0}, s1}};
    t[{1, 0}] = {{{0, 0, 1}, s1}};
    t[{1, 1}] = {{{1, 0, 0}, s1}};
    t[{2, -2}] = {{{1, 1, 0}, s2a}};
    t[{2, -1}] = {{{0, 1, 1}, s2a}};
    t[{2, 0}] = {{{0, 0, 2}, 2 * s2b}, {{2, 0, 0}, -s2b}, {{0, 2, 0}, -s2b}};
    t[{2, 1}] = {{{1, 0, 1}, s2a}};
    t[{2, 2}] = {{{2, 0, 0}, s2c}, {{0, 2, 0}, -s2c}};
    t[{3, -3}] = {{{2, 1, 0}, 3 * s3a}, {{0, 3, 0}, -s3a}};
    t[{3, -2}] = {{{1, 1, 1}, s3b}};
    t[{3, -1}] = {{{0, 1, 2}, 4 * s3c}, {{2, 1, 0}, -s3c}, {{0, 3, 0}, -s3c}};
    t[{3, 0}] = {{{0, 0, 3}, 2 * s3d}, {{2, 0, 1}, -3 * s3d}, {{0, 2, 1}, -3 * s3d}};
    t[{3, 1}] = {{{1, 0, 2}, 4 * s3c}, {{3, 0, 0}, -s3c}, {{1, 2, 0}, -s3c}};
    t[{3, 2}] = {{{2, 0, 1}, s2c}, {{0, 2, 1}, -s2c}};
    t[{3, 3}] = {{{3, 0, 0}, s3a}, {{1, 2, 0}, -3 * s3a}};
    return t;
  }();
  auto it = table.find({l, m});
  if (it == table.end()) throw std::invalid_argument("solid_harmonic_terms: l must be in [0,3], m in [-l,l]");
  return it->second;
}

// McMurchie-Davidson E^{ij}_0 by the standard recursion (gaussian.cpp:42-53)
double hermite_e(int i, int j, int t, double inv2p, double pa, double pb) {
  if (t < 0 || t > i + j) return 0.0;
  if (i == 0 && j == 0) return t == 0 ? 1.0 : 0.0;
  if (i > 0)
    return inv2p * hermite_e(i - 1, j, t - 1, inv2p, pa, pb) + pa * hermite_e(i - 1, j, t, inv2p, pa, pb) +
           (t + 1) * hermite_e(i - 1, j, t + 1, inv2p, pa, pb);
  return inv2p * hermite_e(i, j - 1, t - 1, inv2p, pa, pb) + pb * hermite_e(i, j - 1, t, inv2p, pa, pb) +
         (t + 1) * hermite_e(i, j - 1, t + 1, inv2p, pa, pb);
}

double sq(const Vec3& a) { return a.x * a.x + a.y * a.y + a.z * a.z; }
Vec3 sub(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
}  // namespace

double primitive_norm(int l, double zeta) {  // gaussian.cpp:94-97
  if (zeta <= 0.0) throw std::invalid_argument("primitive_norm: exponent must be positive");
  return std::sqrt(2.0 * std::pow(2.0 * zeta, l + 1.5) / std::tgamma(l + 1.5));
}

double boys_f0(double t) {  // gaussian.cpp:99-104
  if (t < 0.0) throw std::invalid_argument("boys_f0: negative argument");
  if (t < 1e-12) return 1.0 - t / 3.0;
  return 0.5 * std::sqrt(kPi / t) * std::erf(std::sqrt(t));
}

double primitive_overlap(int la, int ma, double a, const Vec3& A, int lb, int mb, double b,
                         const Vec3& B) {  // gaussian.cpp:106-128
  const double p = a + b, mu = a * b / p, inv2p = 0.5 / p;
  const Vec3 P{(a * A.x + b * B.x) / p, (a * A.y + b * B.y) / p, (a * A.z + b * B.z) / p};
  const Vec3 PA = sub(P, A), PB = sub(P, B);
  const double pref = std::pow(kPi / p, 1.5) * std::exp(-mu * sq(sub(A, B)));
  double sum = 0.0;
  for (const auto& ta : monomials(la, ma))
    for (const auto& tb : monomials(lb, mb))
      sum += ta.c * tb.c * hermite_e(ta.e[0], tb.e[0], 0, inv2p, PA.x, PB.x) *
             hermite_e(ta.e[1], tb.e[1], 0, inv2p, PA.y, PB.y) *
             hermite_e(ta.e[2], tb.e[2], 0, inv2p, PA.z, PB.z);
  return pref * sum;
}

BasisFunction::BasisFunction(const Vec3& c, int l_, int m_, std::vector<Primitive> prims)
    : center(c), l(l_), m(m_), primitives(std::move(prims)) {  // model.cpp:30-53
  if (l < 0 || l > 3) throw std::invalid_argument("BasisFunction: l must be in [0,3]");
  if (m < -l || m > l) throw std::invalid_argument("BasisFunction: m out of range");
  if (primitives.empty()) throw std::invalid_argument("BasisFunction: needs at least one primitive");
  for (const auto& p : primitives)
    if (!(p.zeta > 0.0)) throw std::invalid_argument("BasisFunction: exponents must be strictly positive");
  for (const auto& p : primitives) evaluation_coeffs.push_back(p.coeff * primitive_norm(l, p.zeta));
  double s = 0.0;
  for (std::size_t i = 0; i < primitives.size(); ++i)
    for (std::size_t j = 0; j < primitives.size(); ++j)
      s += evaluation_coeffs[i] * evaluation_coeffs[j] *
           primitive_overlap(l, m, primitives[i].zeta, center, l, m, primitives[j].zeta, center);
  if (!(s > 0.0)) throw std::invalid_argument("BasisFunction: vanishing contraction");
  const double rescale = 1.0 / std::sqrt(s);
  for (auto& v : evaluation_coeffs) v *= rescale;
}

double contracted_overlap(const BasisFunction& a, const BasisFunction& b) {  // model.cpp:66-76
  double s = 0.0;
  for (std::size_t i = 0; i < a.primitives.size(); ++i)
    for (std::size_t j = 0; j < b.primitives.size(); ++j)
      s += a.evaluation_coeffs[i] * b.evaluation_coeffs[j] *
           primitive_overlap(a.l, a.m, a.primitives[i].zeta, a.center, b.l, b.m, b.primitives[j].zeta, b.center);
  return s;
}

PairPrefactors mp2_pair_prefactors(int ncomp) {  // model.cpp:86-88
  return ncomp == 1 ? PairPrefactors{2.0, -1.0} : PairPrefactors{0.5, -0.5};
}

SpinorSet::SpinorSet(int nc, std::vector<std::vector<BasisFunction>> b, std::vector<Complex> c,
                     std::vector<double> e, int no, int nv, std::optional<std::vector<Nucleus>> nuc)
    : ncomp(nc), n_occ(no), n_vir(nv), basis(std::move(b)), coeff(std::move(c)), energies(std::move(e)),
      nuclei(std::move(nuc)) {  // model.cpp:90-138
  if (ncomp != 1 && ncomp != 2 && ncomp != 4)
    throw std::invalid_argument("SpinorSet: component count must be 1, 2 or 4");
  if (int(basis.size()) != ncomp) throw std::invalid_argument("SpinorSet: one basis list per component required");
  if (n_occ < 0 || n_vir < 0 || n_occ + n_vir == 0)
    throw std::invalid_argument("SpinorSet: invalid occupied/virtual counts");
  for (const auto& bl : basis)
    if (bl.empty()) throw std::invalid_argument("SpinorSet: empty basis list for a component");
  if (coeff.size() != std::size_t(rows()) * n_spinor())
    throw std::runtime_error("SpinorSet: coefficient rows do not match component basis sizes");
  if (int(energies.size()) != n_spinor()) throw std::runtime_error("SpinorSet: one energy per spinor required");
  for (int p = 1; p < n_occ; ++p)
    if (energies[p] < energies[p - 1]) throw std::runtime_error("SpinorSet: occupied energies not ascending");
  for (int p = n_occ + 1; p < n_spinor(); ++p)
    if (energies[p] < energies[p - 1]) throw std::runtime_error("SpinorSet: virtual energies not ascending");
  if (n_occ > 0 && n_vir > 0 && !(energies[n_occ - 1] < energies[n_occ]))
    throw std::runtime_error("SpinorSet: occupied and virtual energies overlap");
  const double dev = orthonormality_deviation();
  if (!(dev < 1e-8)) {
    std::ostringstream os;
    os << "SpinorSet: coefficients not orthonormal, max deviation of C^H S C from identity is " << dev;
    throw std::runtime_error(os.str());
  }
}

int SpinorSet::rows() const {
  int r = 0;
  for (const auto& b : basis) r += int(b.size());
  return r;
}

double SpinorSet::orthonormality_deviation() const {  // model.cpp:144-158, block-diagonal S
  // max |C^H S C - I| as sum over channels x of C_x^H (S_x C_x); the O(rows^2 n_p + rows n_p^2)
  // products run on all host threads (the serial part of every worker's setup, so of the
  // strong-scaling job)
  const int cols = n_spinor();
  const int nthreads = std::max(1, std::min(16, int(std::thread::hardware_concurrency())));
  auto parallel = [&](int n, auto&& body) {  // body(lo, hi) over [0, n)
    std::vector<std::thread> pool;
    const int chunk = (n + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads && t * chunk < n; ++t)
      pool.emplace_back([&, t] { body(t * chunk, std::min(n, (t + 1) * chunk)); });
    for (auto& th : pool) th.join();
  };
  std::vector<std::vector<Complex>> sc(basis.size());  // S_x C_x per channel
  std::vector<int> offs(basis.size());
  int off = 0;
  for (std::size_t x = 0; x < basis.size(); ++x) {
    const auto& bl = basis[x];
    const int n = int(bl.size());
    offs[x] = off;
    std::vector<double> sm(std::size_t(n) * n);
    parallel(n, [&](int lo, int hi) {
      for (int i = lo; i < hi; ++i)
        for (int j = 0; j < n; ++j) sm[std::size_t(i) * n + j] = contracted_overlap(bl[i], bl[j]);
    });
    sc[x].assign(std::size_t(n) * cols, Complex(0, 0));
    parallel(n, [&](int lo, int hi) {
      for (int i = lo; i < hi; ++i)
        for (int k = 0; k < n; ++k) {
          const double v = sm[std::size_t(i) * n + k];
          if (v == 0.0) continue;
          const Complex* row = &coeff[std::size_t(off + k) * cols];
          Complex* out = &sc[x][std::size_t(i) * cols];
          for (int c = 0; c < cols; ++c) out[c] += v * row[c];
        }
    });
    off += n;
  }
  std::vector<double> devs(std::size_t(cols), 0.0);
  parallel(cols, [&](int lo, int hi) {
    std::vector<Complex> g(static_cast<std::size_t>(cols));
    for (int a = lo; a < hi; ++a) {
      std::fill(g.begin(), g.end(), Complex(0, 0));
      for (std::size_t x = 0; x < basis.size(); ++x) {
        const int n = int(basis[x].size());
        for (int i = 0; i < n; ++i) {
          const Complex ca = std::conj(coeff[std::size_t(offs[x] + i) * cols + a]);
          const Complex* scr = &sc[x][std::size_t(i) * cols];
          for (int b = 0; b < cols; ++b) g[b] += ca * scr[b];
        }
      }
      double d = 0.0;
      for (int b = 0; b < cols; ++b) d = std::max(d, std::abs(g[b] - Complex(a == b ? 1.0 : 0.0, 0.0)));
      devs[std::size_t(a)] = d;
    }
  });
  return devs.empty() ? 0.0 : *std::max_element(devs.begin(), devs.end());
}

std::string format_double(double x) {  // model.cpp:180-184
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", x);
  return buf;
}

namespace {
// whitespace tokens, '#' comments to end of line (model.cpp:188-271)
class Tokens {
 public:
  explicit Tokens(const std::string& path) : in_(path) {
    if (!in_) throw std::runtime_error("cannot open spinor file: " + path);
  }
  bool more() {
    fill();
    return pos_ < line_.size();
  }
  std::string word() {
    fill();
    if (pos_ >= line_.size()) throw std::runtime_error("spinor file: unexpected end of file");
    const std::size_t end = line_.find_first_of(" \t\r\n\v\f", pos_);
    std::string w = line_.substr(pos_, end == std::string::npos ? std::string::npos : end - pos_);
    pos_ = end == std::string::npos ? line_.size() : end;
    return w;
  }
  long integer() {
    const std::string w = word();
    char* end = nullptr;
    errno = 0;
    const long v = std::strtol(w.c_str(), &end, 10);
    if (w.empty() || *end != '\0' || errno) throw std::runtime_error("spinor file: expected integer, got '" + w + "'");
    return v;
  }
  double number() {
    const std::string w = word();
    char* end = nullptr;
    errno = 0;
    const double v = std::strtod(w.c_str(), &end);
    if (w.empty() || *end != '\0' || errno == ERANGE)
      throw std::runtime_error("spinor file: expected number, got '" + w + "'");
    return v;
  }
  void expect(const char* w) {
    const std::string got = word();
    if (got != w) throw std::runtime_error(std::string("spinor file: expected '") + w + "', got '" + got + "'");
  }
  Vec3 vec3() {  // file order x, y, z (SURVEY finding 8)
    Vec3 v;
    v.x = number();
    v.y = number();
    v.z = number();
    return v;
  }

 private:
  void fill() {
    for (;;) {
      pos_ = line_.find_first_not_of(" \t\r\n\v\f", pos_);
      if (pos_ != std::string::npos) return;
      if (!std::getline(in_, line_)) {
        line_.clear();
        pos_ = 0;
        return;
      }
      if (auto h = line_.find('#'); h != std::string::npos) line_.erase(h);
      pos_ = 0;
    }
  }
  std::ifstream in_;
  std::string line_;
  std::size_t pos_ = 0;
};
}  // namespace

SpinorSet load_spinor_set(const std::string& path) {  // model.cpp:275-351
  Tokens t(path);
  t.expect("spinor-text");
  if (t.integer() != 1) throw std::runtime_error("spinor file: unsupported format version");
  std::optional<std::vector<Nucleus>> nuclei;
  int ncomp = 0, n_occ = -1, n_vir = -1;
  std::vector<std::vector<BasisFunction>> basis;
  std::vector<double> energies;
  std::vector<Complex> coeff;
  long ccols = -1;
  while (t.more()) {
    const std::string rec = t.word();
    if (rec == "nuclei") {
      const long n = t.integer();
      std::vector<Nucleus> v;
      for (long i = 0; i < n; ++i) {
        Nucleus nu;
        nu.charge = t.number();
        nu.position = t.vec3();
        v.push_back(nu);
      }
      if (v.empty()) throw std::invalid_argument("Molecule: at least one nucleus required");
      for (const auto& nu : v)
        if (!(nu.charge > 0.0)) throw std::invalid_argument("Molecule: nuclear charges must be strictly positive");
      nuclei = std::move(v);
    } else if (rec == "ncomp") {
      ncomp = int(t.integer());
      if (ncomp != 1 && ncomp != 2 && ncomp != 4) throw std::runtime_error("spinor file: ncomp must be 1, 2 or 4");
      basis.resize(ncomp);
    } else if (rec == "basis") {
      if (ncomp == 0) throw std::runtime_error("spinor file: basis before ncomp");
      const long comp = t.integer();
      if (comp < 0 || comp >= ncomp) throw std::runtime_error("spinor file: basis component index out of range");
      const long count = t.integer();
      for (long i = 0; i < count; ++i) {
        const Vec3 c = t.vec3();
        t.expect(";");
        const int l = int(t.integer());
        const int m = int(t.integer());
        t.expect(";");
        const long np = t.integer();
        t.expect(";");
        std::vector<Primitive> prims;
        for (long k = 0; k < np; ++k) {
          Primitive p;
          p.zeta = t.number();
          p.coeff = t.number();
          prims.push_back(p);
        }
        basis[comp].emplace_back(c, l, m, std::move(prims));
      }
    } else if (rec == "energies") {
      n_occ = int(t.integer());
      n_vir = int(t.integer());
      energies.assign(std::max(0, n_occ + n_vir), 0.0);
      for (auto& e : energies) e = t.number();
    } else if (rec == "coeff") {
      const long r = t.integer();
      ccols = t.integer();
      coeff.assign(std::size_t(r) * ccols, Complex(0, 0));
      for (auto& c : coeff) {
        const double re = t.number();
        const double im = t.number();
        c = Complex(re, im);
      }
    } else {
      throw std::runtime_error("spinor file: unknown record '" + rec + "'");
    }
  }
  if (ncomp == 0) throw std::runtime_error("spinor file: missing ncomp record");
  if (n_occ < 0) throw std::runtime_error("spinor file: missing energies record");
  if (ccols < 0) throw std::runtime_error("spinor file: missing coeff record");
  if (ccols != n_occ + n_vir) throw std::runtime_error("SpinorSet: n_occ + n_vir does not match coefficient columns");
  return SpinorSet(ncomp, std::move(basis), std::move(coeff), std::move(energies), n_occ, n_vir, std::move(nuclei));
}

void save_spinor_set(const SpinorSet& s, const std::string& path) {  // model.cpp:353-388
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write spinor file: " + path);
  out << "spinor-text 1\n";
  if (s.nuclei) {
    out << "nuclei " << s.nuclei->size() << "\n";
    for (const auto& n : *s.nuclei)
      out << format_double(n.charge) << ' ' << format_double(n.position.x) << ' ' << format_double(n.position.y)
          << ' ' << format_double(n.position.z) << "\n";
  }
  out << "ncomp " << s.ncomp << "\n";
  for (int x = 0; x < s.ncomp; ++x) {
    out << "basis " << x << ' ' << s.basis[x].size() << "\n";
    for (const auto& f : s.basis[x]) {
      out << format_double(f.center.x) << ' ' << format_double(f.center.y) << ' ' << format_double(f.center.z)
          << " ; " << f.l << ' ' << f.m << " ; " << f.primitives.size() << " ;";
      for (const auto& p : f.primitives) out << ' ' << format_double(p.zeta) << ' ' << format_double(p.coeff);
      out << "\n";
    }
  }
  out << "energies " << s.n_occ << ' ' << s.n_vir << "\n";
  for (double e : s.energies) out << format_double(e) << "\n";
  out << "coeff " << s.rows() << ' ' << s.n_spinor() << "\n";
  for (int i = 0; i < s.rows(); ++i) {
    for (int j = 0; j < s.n_spinor(); ++j) {
      if (j) out << ' ';
      const Complex c = s.coeff[std::size_t(i) * s.n_spinor() + j];
      out << format_double(c.real()) << ' ' << format_double(c.imag());
    }
    out << "\n";
  }
  if (!out) throw std::runtime_error("failed writing spinor file: " + path);
}

// ------------------------------------------------------------------ weights.cpp
namespace {
const char* const kElements[] = {
    "H",  "He", "Li", "Be", "B",  "C",  "N",  "O",  "F",  "Ne", "Na", "Mg", "Al", "Si", "P",  "S",  "Cl", "Ar",
    "K",  "Ca", "Sc", "Ti", "V",  "Cr", "Mn", "Fe", "Co", "Ni", "Cu", "Zn", "Ga", "Ge", "As", "Se", "Br", "Kr",
    "Rb", "Sr", "Y",  "Zr", "Nb", "Mo", "Tc", "Ru", "Rh", "Pd", "Ag", "Cd", "In", "Sn", "Sb", "Te", "I",  "Xe",
    "Cs", "Ba", "La", "Ce", "Pr", "Nd", "Pm", "Sm", "Eu", "Gd", "Tb", "Dy", "Ho", "Er", "Tm", "Yb", "Lu", "Hf",
    "Ta", "W",  "Re", "Os", "Ir", "Pt", "Au", "Hg", "Tl", "Pb", "Bi", "Po", "At", "Rn", "Fr", "Ra", "Ac", "Th",
    "Pa", "U",  "Np", "Pu", "Am", "Cm", "Bk", "Cf", "Es", "Fm", "Md", "No", "Lr"};
constexpr int kNumElements = int(sizeof(kElements) / sizeof(kElements[0]));
}  // namespace

const std::map<int, WeightParams>& default_weight_params() {  // weights.cpp:30-39 (Table I)
  static const std::map<int, WeightParams> t{{1, {0.25, 0.06, 0.15, 0.6}},
                                             {8, {0.8, 0.2, 1.0, 0.4}},
                                             {29, {0.8, 0.35, 2.0, 0.6}},
                                             {47, {0.1, 0.1, 0.8, 0.6}},
                                             {79, {0.05, 0.6, 4.0, 0.8}}};
  return t;
}

std::string element_symbol(int z) {
  if (z < 1 || z > kNumElements) throw std::invalid_argument("unknown atomic number");
  return kElements[z - 1];
}

int atomic_number(const std::string& sym) {
  for (int i = 0; i < kNumElements; ++i)
    if (sym == kElements[i]) return i + 1;
  throw std::invalid_argument("unknown element symbol '" + sym + "'");
}

WeightSpec::WeightSpec(const std::vector<Nucleus>& nuclei, const std::map<int, WeightParams>& overrides) {
  for (const auto& nu : nuclei) {  // weights.cpp:57-82
    const int z = int(std::lround(nu.charge));
    const WeightParams* p = nullptr;
    if (auto it = overrides.find(z); it != overrides.end()) p = &it->second;
    else if (auto jt = default_weight_params().find(z); jt != default_weight_params().end()) p = &jt->second;
    if (!p) {
      std::ostringstream os;
      os << "no weight parameters for element Z=" << z << "; supply them with a 'weight' configuration line";
      throw std::invalid_argument(os.str());
    }
    if (!(p->c1 > 0 && p->zeta1 > 0 && p->c2 > 0 && p->zeta2 > 0))
      throw std::invalid_argument("weight parameters must be positive");
    const double y00 = 0.28209479177387814;
    pos.push_back(nu.position);
    prim.insert(prim.end(), {p->c1 * (primitive_norm(0, p->zeta1) * y00), p->zeta1,
                             p->c2 * (primitive_norm(0, p->zeta2) * y00), p->zeta2});
    zeta1.push_back(p->zeta1);
  }
  // N_g = sum over primitive pairs of the two-centre Coulomb integral (weights.cpp:23-26, 84-89)
  ng = 0.0;
  const std::size_t n = pos.size();
  for (std::size_t i = 0; i < n; ++i)
    for (int a = 0; a < 2; ++a)
      for (std::size_t j = 0; j < n; ++j)
        for (int b = 0; b < 2; ++b) {
          const double za = prim[4 * i + 2 * a + 1], zb = prim[4 * j + 2 * b + 1];
          const double t = za * zb / (za + zb) * sq(sub(pos[i], pos[j]));
          const double j2 = 2.0 * std::pow(kPi, 2.5) / (za * zb * std::sqrt(za + zb)) * boys_f0(t);
          ng += prim[4 * i + 2 * a] * prim[4 * j + 2 * b] * j2;
        }
}

double WeightSpec::g(const Vec3& r) const {  // weights.cpp:92-99
  double v = 0.0;
  for (std::size_t i = 0; i < pos.size(); ++i) {
    const double d2 = sq(sub(r, pos[i]));
    v += prim[4 * i] * std::exp(-prim[4 * i + 1] * d2);
    v += prim[4 * i + 2] * std::exp(-prim[4 * i + 3] * d2);
  }
  return v;
}

double lambda_from_gap(const SpinorSet& s) {  // weights.cpp:113-120
  if (s.n_occ == 0 || s.n_vir == 0)
    throw std::runtime_error("lambda_from_gap: needs both occupied and virtual spinors");
  const double gap = s.energies[s.n_occ] - s.energies[s.n_occ - 1];
  if (!(gap > 0.0)) throw std::runtime_error("lambda_from_gap: non-positive HOMO-LUMO gap");
  return 2.0 * gap;
}

DeviceSystem make_device_system(const SpinorSet& s, const WeightSpec& w, int estimator) {
  DeviceSystem d;
  int nprim = 0;
  d.fn_prim_offset.push_back(0);
  for (const auto& bl : s.basis) {
    d.channel_count.push_back(int(bl.size()));
    for (const auto& f : bl) {
      d.fn_center.insert(d.fn_center.end(), {f.center.x, f.center.y, f.center.z});
      d.fn_lm.insert(d.fn_lm.end(), {f.l, f.m});
      for (std::size_t k = 0; k < f.primitives.size(); ++k) {
        d.prim_zeta.push_back(f.primitives[k].zeta);
        d.prim_coeff.push_back(f.evaluation_coeffs[k]);
      }
      nprim += int(f.primitives.size());
      d.fn_prim_offset.push_back(nprim);
    }
  }
  for (const Complex& c : s.coeff) d.coeff.insert(d.coeff.end(), {c.real(), c.imag()});
  d.energies = s.energies;
  for (const auto& p : w.pos) d.site_pos.insert(d.site_pos.end(), {p.x, p.y, p.z});
  d.site_prim = w.prim;
  d.site_zeta1 = w.zeta1;
  mcmp2dev_system& v = d.view;
  v.ncomp = s.ncomp;
  v.n_occ = s.n_occ;
  v.n_vir = s.n_vir;
  v.channel_count = d.channel_count.data();
  v.fn_center = d.fn_center.data();
  v.fn_lm = d.fn_lm.data();
  v.fn_prim_offset = d.fn_prim_offset.data();
  v.prim_zeta = d.prim_zeta.data();
  v.prim_coeff = d.prim_coeff.data();
  v.coeff = d.coeff.data();
  v.energies = d.energies.data();
  v.nsites = int(w.pos.size());
  v.site_pos = d.site_pos.data();
  v.site_prim = d.site_prim.data();
  v.site_zeta1 = d.site_zeta1.data();
  v.ng = w.ng;
  v.lambda = lambda_from_gap(s);
  const PairPrefactors pp = mp2_pair_prefactors(s.ncomp);
  v.w_direct = pp.direct;
  v.w_exchange = pp.exchange;
  v.estimator = estimator;
  return d;
}

}  // namespace mcmp2
