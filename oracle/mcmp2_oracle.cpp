// mcmp2_oracle.cpp — TEST INFRASTRUCTURE ONLY (see mcmp2_oracle.hpp header).
// CPU restatement of the reference hot path; citations are into
// /root/reference/proj/core/src/.
#include "mcmp2_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <filesystem>
#include <fstream>
#include <numbers>
#include <sstream>
#include <stdexcept>
#include <thread>

namespace oracle {

// =============================================================== rng.cpp:9-94
namespace {
constexpr std::uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
constexpr std::uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
}  // namespace

std::array<std::uint32_t, 4> Philox::block(const std::array<std::uint32_t, 4>& ctr,
                                           const std::array<std::uint32_t, 2>& key) {
  // rng.cpp:17-39: ten rounds, key bumped by the Weyl constants before rounds 1..9
  std::uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  std::uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += kW0;
      k1 += kW1;
    }
    const std::uint64_t p0 = std::uint64_t(kM0) * c0;
    const std::uint64_t p1 = std::uint64_t(kM1) * c2;
    const std::uint32_t n0 = std::uint32_t(p1 >> 32) ^ c1 ^ k0;
    const std::uint32_t n2 = std::uint32_t(p0 >> 32) ^ c3 ^ k1;
    c1 = std::uint32_t(p1);
    c3 = std::uint32_t(p0);
    c0 = n0;
    c2 = n2;
  }
  return {c0, c1, c2, c3};
}

Philox::Philox(std::uint64_t seed, std::uint32_t stream) {  // rng.cpp:41-44
  key = {std::uint32_t(seed), std::uint32_t(seed >> 32)};
  counter = {0, 0, 0, stream};
}

void Philox::refill() {  // rng.cpp:46-51, 96-bit counter, word 3 = stream
  out = block(counter, key);
  if (++counter[0] == 0 && ++counter[1] == 0) ++counter[2];
  idx = 0;
}

std::uint32_t Philox::next_u32() {
  if (idx >= 4) refill();
  return out[idx++];
}

std::uint64_t Philox::next_u64() {  // rng.cpp:58-62: first draw is the high word
  const std::uint64_t hi = next_u32();
  const std::uint64_t lo = next_u32();
  return (hi << 32) | lo;
}

double Philox::uniform() { return double(next_u64() >> 11) * 0x1.0p-53; }  // rng.cpp:64

std::array<double, 3> Philox::gaussian3() {  // rng.cpp:66-74
  const double u1 = uniform();
  const double u2 = uniform();
  const double u3 = uniform();
  const double u4 = uniform();
  const double r1 = std::sqrt(-2.0 * std::log1p(-u1));
  const double r2 = std::sqrt(-2.0 * std::log1p(-u2));
  const double a1 = 2.0 * std::numbers::pi * u3;
  const double a2 = 2.0 * std::numbers::pi * u4;
  return {r1 * std::cos(a1), r1 * std::sin(a1), r2 * std::cos(a2)};
}

std::string Philox::save() const {  // rng.cpp:76-81
  std::ostringstream os;
  os << key[0] << ' ' << key[1];
  for (auto c : counter) os << ' ' << c;
  os << ' ' << idx;
  return os.str();
}

Philox Philox::load(std::istream& is) {  // rng.cpp:83-94
  Philox r;
  is >> r.key[0] >> r.key[1];
  for (auto& c : r.counter) is >> c;
  is >> r.idx;
  if (r.idx < 4) {
    std::array<std::uint32_t, 4> prev = r.counter;
    if (prev[0]-- == 0 && prev[1]-- == 0) --prev[2];
    r.out = block(prev, r.key);
  }
  return r;
}

// =============================================================== gaussian.cpp
namespace {
constexpr double kS00 = 0.28209479177387814;
constexpr double kS1 = 0.4886025119029199;
constexpr double kS2a = 1.0925484305920792;
constexpr double kS2b = 0.31539156525252005;
constexpr double kS2c = 0.5462742152960396;
constexpr double kS3a = 0.5900435899266435;
constexpr double kS3b = 2.890611442640554;
constexpr double kS3c = 0.4570457994644658;
constexpr double kS3d = 0.3731763325901154;

// tables restated from gaussian.cpp:21-39 (index m + l)
struct Table {
  SolidTerm t[3];
  int n;
};
const Table kTab0[1] = {{{{0, 0, 0, kS00}}, 1}};
const Table kTab1[3] = {{{{0, 1, 0, kS1}}, 1}, {{{0, 0, 1, kS1}}, 1}, {{{1, 0, 0, kS1}}, 1}};
const Table kTab2[5] = {
    {{{1, 1, 0, kS2a}}, 1},
    {{{0, 1, 1, kS2a}}, 1},
    {{{0, 0, 2, 2 * kS2b}, {2, 0, 0, -kS2b}, {0, 2, 0, -kS2b}}, 3},
    {{{1, 0, 1, kS2a}}, 1},
    {{{2, 0, 0, kS2c}, {0, 2, 0, -kS2c}}, 2}};
const Table kTab3[7] = {
    {{{2, 1, 0, 3 * kS3a}, {0, 3, 0, -kS3a}}, 2},
    {{{1, 1, 1, kS3b}}, 1},
    {{{0, 1, 2, 4 * kS3c}, {2, 1, 0, -kS3c}, {0, 3, 0, -kS3c}}, 3},
    {{{0, 0, 3, 2 * kS3d}, {2, 0, 1, -3 * kS3d}, {0, 2, 1, -3 * kS3d}}, 3},
    {{{1, 0, 2, 4 * kS3c}, {3, 0, 0, -kS3c}, {1, 2, 0, -kS3c}}, 3},
    {{{2, 0, 1, kS2c}, {0, 2, 1, -kS2c}}, 2},
    {{{3, 0, 0, kS3a}, {1, 2, 0, -3 * kS3a}}, 2}};

// Hermite coefficient E_0^{ij} (gaussian.cpp:42-53)
double e_coeff(int i, int j, int t, double inv2p, double xpa, double xpb) {
  if (t < 0 || t > i + j) return 0.0;
  if (i == 0 && j == 0) return t == 0 ? 1.0 : 0.0;
  if (i > 0)
    return inv2p * e_coeff(i - 1, j, t - 1, inv2p, xpa, xpb) +
           xpa * e_coeff(i - 1, j, t, inv2p, xpa, xpb) +
           (t + 1) * e_coeff(i - 1, j, t + 1, inv2p, xpa, xpb);
  return inv2p * e_coeff(i, j - 1, t - 1, inv2p, xpa, xpb) +
         xpb * e_coeff(i, j - 1, t, inv2p, xpa, xpb) +
         (t + 1) * e_coeff(i, j - 1, t + 1, inv2p, xpa, xpb);
}
}  // namespace

const SolidTerm* solid_harmonic_terms(int l, int m, int* count) {  // gaussian.cpp:57-85
  if (l < 0 || l > 3 || m < -l || m > l)
    throw std::invalid_argument("solid_harmonic_terms: l must be in [0,3], m in [-l,l]");
  const Table* tab = l == 0 ? kTab0 : l == 1 ? kTab1 : l == 2 ? kTab2 : kTab3;
  *count = tab[m + l].n;
  return tab[m + l].t;
}

double solid_harmonic(int l, int m, const Vec3& d) {  // gaussian.cpp:87-92
  int n = 0;
  const SolidTerm* t = solid_harmonic_terms(l, m, &n);
  double s = 0.0;
  for (int k = 0; k < n; ++k)
    s += t[k].coef * std::pow(d.x, t[k].ix) * std::pow(d.y, t[k].iy) * std::pow(d.z, t[k].iz);
  return s;
}

double primitive_norm(int l, double zeta) {  // gaussian.cpp:94-97
  if (zeta <= 0.0) throw std::invalid_argument("primitive_norm: exponent must be positive");
  return std::sqrt(2.0 * std::pow(2.0 * zeta, l + 1.5) / std::tgamma(l + 1.5));
}

double boys_f0(double t) {  // gaussian.cpp:99-104
  if (t < 0.0) throw std::invalid_argument("boys_f0: negative argument");
  if (t < 1e-12) return 1.0 - t / 3.0;
  return 0.5 * std::sqrt(std::numbers::pi / t) * std::erf(std::sqrt(t));
}

double primitive_overlap(int la, int ma, double a, const Vec3& A, int lb, int mb, double b,
                         const Vec3& B) {  // gaussian.cpp:106-128
  const double p = a + b;
  const double mu = a * b / p;
  const Vec3 P{(a * A.x + b * B.x) / p, (a * A.y + b * B.y) / p, (a * A.z + b * B.z) / p};
  const Vec3 AB = A - B, PA = P - A, PB = P - B;
  const double inv2p = 0.5 / p;
  const double pref = std::pow(std::numbers::pi / p, 1.5) * std::exp(-mu * sqnorm(AB));
  int na = 0, nb = 0;
  const SolidTerm* ta = solid_harmonic_terms(la, ma, &na);
  const SolidTerm* tb = solid_harmonic_terms(lb, mb, &nb);
  double sum = 0.0;
  for (int i = 0; i < na; ++i)
    for (int j = 0; j < nb; ++j) {
      const double ex = e_coeff(ta[i].ix, tb[j].ix, 0, inv2p, PA.x, PB.x);
      const double ey = e_coeff(ta[i].iy, tb[j].iy, 0, inv2p, PA.y, PB.y);
      const double ez = e_coeff(ta[i].iz, tb[j].iz, 0, inv2p, PA.z, PB.z);
      sum += ta[i].coef * tb[j].coef * ex * ey * ez;
    }
  return pref * sum;
}

// =============================================================== model.cpp
BasisFunction::BasisFunction(const Vec3& c, int l_, int m_, std::vector<Primitive> prims)
    : center(c), l(l_), m(m_), primitives(std::move(prims)) {  // model.cpp:30-53
  if (l < 0 || l > 3) throw std::invalid_argument("BasisFunction: l must be in [0,3]");
  if (m < -l || m > l) throw std::invalid_argument("BasisFunction: m out of range");
  if (primitives.empty()) throw std::invalid_argument("BasisFunction: needs at least one primitive");
  for (const auto& p : primitives)
    if (!(p.zeta > 0.0))
      throw std::invalid_argument("BasisFunction: exponents must be strictly positive");
  eval_coeffs.resize(primitives.size());
  for (std::size_t k = 0; k < primitives.size(); ++k)
    eval_coeffs[k] = primitives[k].coeff * primitive_norm(l, primitives[k].zeta);
  double s = 0.0;
  for (std::size_t k = 0; k < primitives.size(); ++k)
    for (std::size_t n = 0; n < primitives.size(); ++n)
      s += eval_coeffs[k] * eval_coeffs[n] *
           primitive_overlap(l, m, primitives[k].zeta, center, l, m, primitives[n].zeta, center);
  if (!(s > 0.0)) throw std::invalid_argument("BasisFunction: vanishing contraction");
  const double rescale = 1.0 / std::sqrt(s);
  for (auto& c2 : eval_coeffs) c2 *= rescale;
}

double BasisFunction::value(const Vec3& r) const {  // model.cpp:55-64
  const Vec3 d = r - center;
  const double ang = solid_harmonic(l, m, d);
  if (ang == 0.0) return 0.0;
  const double r2 = sqnorm(d);
  double radial = 0.0;
  for (std::size_t k = 0; k < primitives.size(); ++k)
    radial += eval_coeffs[k] * std::exp(-primitives[k].zeta * r2);
  return ang * radial;
}

double contracted_overlap(const BasisFunction& a, const BasisFunction& b) {  // model.cpp:66-76
  double s = 0.0;
  for (std::size_t k = 0; k < a.eval_coeffs.size(); ++k)
    for (std::size_t n = 0; n < b.eval_coeffs.size(); ++n)
      s += a.eval_coeffs[k] * b.eval_coeffs[n] *
           primitive_overlap(a.l, a.m, a.primitives[k].zeta, a.center, b.l, b.m,
                             b.primitives[n].zeta, b.center);
  return s;
}

PairPrefactors mp2_pair_prefactors(int ncomp) {  // model.cpp:86-88
  return ncomp == 1 ? PairPrefactors{2.0, -1.0} : PairPrefactors{0.5, -0.5};
}

SpinorSet::SpinorSet(int nc, std::vector<std::vector<BasisFunction>> b, std::vector<Complex> c,
                     std::vector<double> e, int no, int nv,
                     std::optional<std::vector<Nucleus>> nuc, bool validate)
    : ncomp(nc), n_occ(no), n_vir(nv), rows(0), basis(std::move(b)), coeff(std::move(c)),
      energies(std::move(e)), nuclei(std::move(nuc)) {  // model.cpp:90-138
  if (ncomp != 1 && ncomp != 2 && ncomp != 4)
    throw std::invalid_argument("SpinorSet: component count must be 1, 2 or 4");
  if (int(basis.size()) != ncomp)
    throw std::invalid_argument("SpinorSet: one basis list per component required");
  if (n_occ < 0 || n_vir < 0 || n_occ + n_vir == 0)
    throw std::invalid_argument("SpinorSet: invalid occupied/virtual counts");
  row_offset.resize(ncomp);
  for (int x = 0; x < ncomp; ++x) {
    if (basis[x].empty()) throw std::invalid_argument("SpinorSet: empty basis list for a component");
    row_offset[x] = rows;
    rows += int(basis[x].size());
  }
  if (int(coeff.size()) != rows * (n_occ + n_vir))
    throw std::runtime_error("SpinorSet: coefficient rows do not match component basis sizes");
  if (int(energies.size()) != n_occ + n_vir)
    throw std::runtime_error("SpinorSet: one energy per spinor required");
  for (int p = 1; p < n_occ; ++p)
    if (energies[p] < energies[p - 1])
      throw std::runtime_error("SpinorSet: occupied energies not ascending");
  for (int p = n_occ + 1; p < n_occ + n_vir; ++p)
    if (energies[p] < energies[p - 1])
      throw std::runtime_error("SpinorSet: virtual energies not ascending");
  if (n_occ > 0 && n_vir > 0 && !(homo() < lumo()))
    throw std::runtime_error("SpinorSet: occupied and virtual energies overlap");
  if (validate) {
    const double dev = orthonormality_deviation();
    if (!(dev < 1e-8)) {
      std::ostringstream os;
      os << "SpinorSet: coefficients not orthonormal, max deviation of C^H S C from identity is "
         << dev;
      throw std::runtime_error(os.str());
    }
  }
}

int SpinorSet::max_channel_size() const {
  int mx = 0;
  for (const auto& b : basis) mx = std::max(mx, int(b.size()));
  return mx;
}

double SpinorSet::orthonormality_deviation() const {  // model.cpp:144-158 (block-diagonal S)
  const int cols = n_spinor();
  std::vector<Complex> g(std::size_t(cols) * cols, Complex(0, 0));
  for (int x = 0; x < ncomp; ++x) {
    const int n = int(basis[x].size()), off = row_offset[x];
    std::vector<double> s(std::size_t(n) * n);
    for (int i = 0; i < n; ++i)
      for (int j = i; j < n; ++j)
        s[i * n + j] = s[j * n + i] = contracted_overlap(basis[x][i], basis[x][j]);
    // t = S C_x  (n x cols)
    std::vector<Complex> t(std::size_t(n) * cols, Complex(0, 0));
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < n; ++k) {
        const double sik = s[i * n + k];
        const Complex* crow = &coeff[std::size_t(off + k) * cols];
        for (int c = 0; c < cols; ++c) t[std::size_t(i) * cols + c] += sik * crow[c];
      }
    for (int i = 0; i < n; ++i) {
      const Complex* crow = &coeff[std::size_t(off + i) * cols];
      for (int a = 0; a < cols; ++a) {
        const Complex ca = std::conj(crow[a]);
        for (int b = 0; b < cols; ++b) g[std::size_t(a) * cols + b] += ca * t[std::size_t(i) * cols + b];
      }
    }
  }
  double dev = 0.0;
  for (int a = 0; a < cols; ++a)
    for (int b = 0; b < cols; ++b)
      dev = std::max(dev, std::abs(g[std::size_t(a) * cols + b] - Complex(a == b ? 1.0 : 0.0, 0.0)));
  return dev;
}

void SpinorSet::evaluate_into(const Vec3& point, Complex* occ, Complex* vir,
                              double* chi) const {  // model.cpp:166-178
  const int cols = n_spinor();
  for (int x = 0; x < ncomp; ++x) {
    const auto& bas = basis[x];
    const int n = int(bas.size());
    for (int mu = 0; mu < n; ++mu) chi[mu] = bas[mu].value(point);
    Complex* o = occ + std::size_t(x) * n_occ;
    Complex* v = vir + std::size_t(x) * n_vir;
    for (int i = 0; i < n_occ; ++i) o[i] = Complex(0, 0);
    for (int a = 0; a < n_vir; ++a) v[a] = Complex(0, 0);
    for (int mu = 0; mu < n; ++mu) {
      const double c = chi[mu];
      const Complex* crow = &coeff[std::size_t(row_offset[x] + mu) * cols];
      for (int i = 0; i < n_occ; ++i) o[i] += c * crow[i];
      for (int a = 0; a < n_vir; ++a) v[a] += c * crow[n_occ + a];
    }
  }
}

std::string format_double(double x) {  // model.cpp:180-184
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", x);
  return buf;
}

namespace {
// whitespace token reader with '#' comments (model.cpp:188-271)
class TokenReader {
 public:
  explicit TokenReader(const std::string& path) : in_(path) {
    if (!in_) throw std::runtime_error("cannot open spinor file: " + path);
  }
  bool next_tok(std::string& tok) {
    if (!push_.empty()) {
      tok = std::move(push_);
      push_.clear();
      return true;
    }
    while (!(cur_ >> tok)) {
      std::string line;
      if (!std::getline(in_, line)) return false;
      if (auto pos = line.find('#'); pos != std::string::npos) line.erase(pos);
      cur_ = std::istringstream(line);
    }
    return true;
  }
  std::string next() {
    std::string t;
    if (!next_tok(t)) throw std::runtime_error("spinor file: unexpected end of file");
    return t;
  }
  long next_long() {
    const std::string tok = next();
    std::size_t used = 0;
    long v = 0;
    try {
      v = std::stol(tok, &used);
    } catch (const std::exception&) {
      throw std::runtime_error("spinor file: expected integer, got '" + tok + "'");
    }
    if (used != tok.size()) throw std::runtime_error("spinor file: expected integer, got '" + tok + "'");
    return v;
  }
  double next_double() {
    const std::string tok = next();
    std::size_t used = 0;
    double v = 0;
    try {
      v = std::stod(tok, &used);
    } catch (const std::exception&) {
      throw std::runtime_error("spinor file: expected number, got '" + tok + "'");
    }
    if (used != tok.size()) throw std::runtime_error("spinor file: expected number, got '" + tok + "'");
    return v;
  }
  void expect(const std::string& w) {
    const std::string tok = next();
    if (tok != w) throw std::runtime_error("spinor file: expected '" + w + "', got '" + tok + "'");
  }
  bool at_end() {
    std::string t;
    if (!next_tok(t)) return true;
    push_ = t;
    return false;
  }

 private:
  std::ifstream in_;
  std::istringstream cur_;
  std::string push_;
};

Vec3 read_vec3(TokenReader& r) {
  // file order x, y, z with separate statements (SURVEY finding 8)
  Vec3 v;
  v.x = r.next_double();
  v.y = r.next_double();
  v.z = r.next_double();
  return v;
}
}  // namespace

SpinorSet load_spinor_set(const std::string& path, bool validate) {  // model.cpp:275-351
  TokenReader r(path);
  r.expect("spinor-text");
  if (r.next_long() != 1) throw std::runtime_error("spinor file: unsupported format version");
  std::optional<std::vector<Nucleus>> nuclei;
  int ncomp = 0;
  std::vector<std::vector<BasisFunction>> basis;
  std::vector<double> energies;
  int n_occ = -1, n_vir = -1;
  std::vector<Complex> coeff;
  long crow = 0, ccol = 0;
  bool have_coeff = false;
  while (!r.at_end()) {
    const std::string rec = r.next();
    if (rec == "nuclei") {
      const long n = r.next_long();
      std::vector<Nucleus> nuc(n);
      for (auto& nu : nuc) {
        nu.charge = r.next_double();
        nu.position = read_vec3(r);
      }
      for (const auto& nu : nuc)  // Molecule ctor, model.cpp:10-19
        if (!(nu.charge > 0.0))
          throw std::invalid_argument("Molecule: nuclear charges must be strictly positive");
      if (nuc.empty()) throw std::invalid_argument("Molecule: at least one nucleus required");
      nuclei = std::move(nuc);
    } else if (rec == "ncomp") {
      ncomp = int(r.next_long());
      if (ncomp != 1 && ncomp != 2 && ncomp != 4)
        throw std::runtime_error("spinor file: ncomp must be 1, 2 or 4");
      basis.resize(ncomp);
    } else if (rec == "basis") {
      if (ncomp == 0) throw std::runtime_error("spinor file: basis before ncomp");
      const long comp = r.next_long();
      if (comp < 0 || comp >= ncomp)
        throw std::runtime_error("spinor file: basis component index out of range");
      const long count = r.next_long();
      for (long i = 0; i < count; ++i) {
        const Vec3 c = read_vec3(r);
        r.expect(";");
        const int l = int(r.next_long());
        const int m = int(r.next_long());
        r.expect(";");
        const long nprim = r.next_long();
        r.expect(";");
        std::vector<Primitive> prims(nprim);
        for (auto& p : prims) {
          p.zeta = r.next_double();
          p.coeff = r.next_double();
        }
        basis[comp].emplace_back(c, l, m, std::move(prims));
      }
    } else if (rec == "energies") {
      n_occ = int(r.next_long());
      n_vir = int(r.next_long());
      energies.resize(n_occ + n_vir);
      for (int p = 0; p < n_occ + n_vir; ++p) energies[p] = r.next_double();
    } else if (rec == "coeff") {
      crow = r.next_long();
      ccol = r.next_long();
      coeff.resize(std::size_t(crow) * ccol);
      for (long i = 0; i < crow; ++i)
        for (long j = 0; j < ccol; ++j) {
          const double re = r.next_double();
          const double im = r.next_double();
          coeff[std::size_t(i) * ccol + j] = Complex(re, im);
        }
      have_coeff = true;
    } else {
      throw std::runtime_error("spinor file: unknown record '" + rec + "'");
    }
  }
  if (ncomp == 0) throw std::runtime_error("spinor file: missing ncomp record");
  if (n_occ < 0) throw std::runtime_error("spinor file: missing energies record");
  if (!have_coeff) throw std::runtime_error("spinor file: missing coeff record");
  if (ccol != n_occ + n_vir)
    throw std::runtime_error("SpinorSet: n_occ + n_vir does not match coefficient columns");
  return SpinorSet(ncomp, std::move(basis), std::move(coeff), std::move(energies), n_occ, n_vir,
                   std::move(nuclei), validate);
}

void save_spinor_set(const SpinorSet& s, const std::string& path) {  // model.cpp:353-388
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write spinor file: " + path);
  out << "spinor-text 1\n";
  if (s.nuclei) {
    out << "nuclei " << s.nuclei->size() << "\n";
    for (const auto& n : *s.nuclei)
      out << format_double(n.charge) << ' ' << format_double(n.position.x) << ' '
          << format_double(n.position.y) << ' ' << format_double(n.position.z) << "\n";
  }
  out << "ncomp " << s.ncomp << "\n";
  for (int x = 0; x < s.ncomp; ++x) {
    out << "basis " << x << ' ' << s.basis[x].size() << "\n";
    for (const auto& f : s.basis[x]) {
      out << format_double(f.center.x) << ' ' << format_double(f.center.y) << ' '
          << format_double(f.center.z) << " ; " << f.l << ' ' << f.m << " ; "
          << f.primitives.size() << " ;";
      for (const auto& p : f.primitives)
        out << ' ' << format_double(p.zeta) << ' ' << format_double(p.coeff);
      out << "\n";
    }
  }
  out << "energies " << s.n_occ << ' ' << s.n_vir << "\n";
  for (int p = 0; p < s.n_spinor(); ++p) out << format_double(s.energies[p]) << "\n";
  out << "coeff " << s.rows << ' ' << s.n_spinor() << "\n";
  for (int i = 0; i < s.rows; ++i) {
    for (int j = 0; j < s.n_spinor(); ++j) {
      if (j) out << ' ';
      const Complex c = s.coeff[std::size_t(i) * s.n_spinor() + j];
      out << format_double(c.real()) << ' ' << format_double(c.imag());
    }
    out << "\n";
  }
  if (!out) throw std::runtime_error("failed writing spinor file: " + path);
}

// =============================================================== weights.cpp
namespace {
const char* const kSymbols[] = {
    "H",  "He", "Li", "Be", "B",  "C",  "N",  "O",  "F",  "Ne", "Na", "Mg", "Al", "Si", "P",
    "S",  "Cl", "Ar", "K",  "Ca", "Sc", "Ti", "V",  "Cr", "Mn", "Fe", "Co", "Ni", "Cu", "Zn",
    "Ga", "Ge", "As", "Se", "Br", "Kr", "Rb", "Sr", "Y",  "Zr", "Nb", "Mo", "Tc", "Ru", "Rh",
    "Pd", "Ag", "Cd", "In", "Sn", "Sb", "Te", "I",  "Xe", "Cs", "Ba", "La", "Ce", "Pr", "Nd",
    "Pm", "Sm", "Eu", "Gd", "Tb", "Dy", "Ho", "Er", "Tm", "Yb", "Lu", "Hf", "Ta", "W",  "Re",
    "Os", "Ir", "Pt", "Au", "Hg", "Tl", "Pb", "Bi", "Po", "At", "Rn", "Fr", "Ra", "Ac", "Th",
    "Pa", "U",  "Np", "Pu", "Am", "Cm", "Bk", "Cf", "Es", "Fm", "Md", "No", "Lr"};

double coulomb_2c(double a, const Vec3& A, double b, const Vec3& B) {  // weights.cpp:23-26
  const double t = a * b / (a + b) * sqnorm(A - B);
  return 2.0 * std::pow(std::numbers::pi, 2.5) / (a * b * std::sqrt(a + b)) * boys_f0(t);
}
}  // namespace

const std::map<int, WeightParams>& default_weight_params() {  // weights.cpp:30-39 (Table I)
  static const std::map<int, WeightParams> t = {
      {1, {0.25, 0.06, 0.15, 0.6}},
      {8, {0.8, 0.2, 1.0, 0.4}},
      {29, {0.8, 0.35, 2.0, 0.6}},
      {47, {0.1, 0.1, 0.8, 0.6}},
      {79, {0.05, 0.6, 4.0, 0.8}},
  };
  return t;
}

std::string element_symbol(int z) {
  if (z < 1 || z > int(std::size(kSymbols))) throw std::invalid_argument("unknown atomic number");
  return kSymbols[z - 1];
}

int atomic_number(const std::string& sym) {
  for (std::size_t i = 0; i < std::size(kSymbols); ++i)
    if (sym == kSymbols[i]) return int(i) + 1;
  throw std::invalid_argument("unknown element symbol '" + sym + "'");
}

WeightSpec::WeightSpec(const std::vector<Nucleus>& nuclei,
                       const std::map<int, WeightParams>& overrides) {  // weights.cpp:57-90
  for (const auto& nuc : nuclei) {
    const int z = int(std::lround(nuc.charge));
    const WeightParams* p = nullptr;
    if (auto it = overrides.find(z); it != overrides.end()) p = &it->second;
    else if (auto jt = default_weight_params().find(z); jt != default_weight_params().end())
      p = &jt->second;
    if (!p) {
      std::ostringstream os;
      os << "no weight parameters for element Z=" << z
         << "; supply them with a 'weight' configuration line";
      throw std::invalid_argument(os.str());
    }
    if (!(p->c1 > 0 && p->zeta1 > 0 && p->c2 > 0 && p->zeta2 > 0))
      throw std::invalid_argument("weight parameters must be positive");
    const double n1 = primitive_norm(0, p->zeta1) * 0.28209479177387814;
    const double n2 = primitive_norm(0, p->zeta2) * 0.28209479177387814;
    Site s;
    s.position = nuc.position;
    s.prims = {{p->c1 * n1, p->zeta1}, {p->c2 * n2, p->zeta2}};
    s.zeta1 = p->zeta1;
    sites.push_back(s);
  }
  ng_ = 0.0;
  for (const auto& si : sites)
    for (const auto& pi : si.prims)
      for (const auto& sj : sites)
        for (const auto& pj : sj.prims)
          ng_ += pi.coeff * pj.coeff * coulomb_2c(pi.zeta, si.position, pj.zeta, sj.position);
}

double WeightSpec::g(const Vec3& r) const {  // weights.cpp:92-99
  double v = 0.0;
  for (const auto& s : sites) {
    const double d2 = sqnorm(r - s.position);
    for (const auto& p : s.prims) v += p.coeff * std::exp(-p.zeta * d2);
  }
  return v;
}

TauSampler::TauSampler(double lambda) : lambda_(lambda) {  // weights.cpp:105-107
  if (!(lambda_ > 0.0)) throw std::invalid_argument("TauSampler: lambda must be positive");
}
double TauSampler::sample(double u) const { return -std::log1p(-u) / lambda_; }  // :109
double TauSampler::pdf(double tau) const { return lambda_ * std::exp(-lambda_ * tau); }  // :111

double lambda_from_gap(const SpinorSet& s) {  // weights.cpp:113-120
  if (s.n_occ == 0 || s.n_vir == 0)
    throw std::runtime_error("lambda_from_gap: needs both occupied and virtual spinors");
  const double gap = s.lumo() - s.homo();
  if (!(gap > 0.0)) throw std::runtime_error("lambda_from_gap: non-positive HOMO-LUMO gap");
  return 2.0 * gap;
}

// =============================================================== sampler.cpp
namespace {
Vec3 gaussian_displacement(Philox& rng, double scale) {  // sampler.cpp:14-17
  const auto g = rng.gaussian3();
  return Vec3{g[0], g[1], g[2]} * scale;
}
}  // namespace

WalkerEnsemble init_ensemble(int m, const std::vector<Nucleus>& nuclei, const WeightSpec& spec,
                             std::uint64_t seed, std::uint32_t stream) {  // sampler.cpp:21-47
  if (m < 2) throw std::invalid_argument("init_ensemble: at least two electron-pair walkers");
  if (spec.sites.size() != nuclei.size())
    throw std::invalid_argument("init_ensemble: weight spec does not match the molecule");
  WalkerEnsemble ens;
  ens.rng = Philox(seed, stream);
  ens.pairs.resize(m);
  const auto& sites = spec.sites;
  auto place = [&]() {
    const std::uint32_t idx = std::min<std::uint32_t>(
        std::uint32_t(ens.rng.uniform() * double(sites.size())), std::uint32_t(sites.size() - 1));
    const double spread = 1.0 / std::sqrt(2.0 * sites[idx].zeta1);
    return sites[idx].position + gaussian_displacement(ens.rng, spread);
  };
  for (auto& pr : ens.pairs) {
    pr.r1 = place();
    do {
      pr.r2 = place();
    } while (sqnorm(pr.r1 - pr.r2) == 0.0);
    pr.g1 = spec.g(pr.r1);
    pr.g2 = spec.g(pr.r2);
    pr.weight = pr.g1 * pr.g2 / (spec.ng() * std::sqrt(sqnorm(pr.r1 - pr.r2)));
  }
  return ens;
}

int metropolis_step(WalkerEnsemble& ens, const WeightSpec& spec) {  // sampler.cpp:49-79
  int naccept = 0;
  for (auto& pr : ens.pairs) {
    Vec3 n1, n2;
    double r12;
    do {
      n1 = pr.r1 + gaussian_displacement(ens.rng, ens.sigma_step);
      n2 = pr.r2 + gaussian_displacement(ens.rng, ens.sigma_step);
      r12 = std::sqrt(sqnorm(n1 - n2));
    } while (r12 == 0.0);
    const double g1 = spec.g(n1);
    const double g2 = spec.g(n2);
    const double wnew = g1 * g2 / (spec.ng() * r12);
    const double u = ens.rng.uniform();
    ++ens.proposed;
    if (u * pr.weight < wnew) {
      pr.r1 = n1;
      pr.r2 = n2;
      pr.g1 = g1;
      pr.g2 = g2;
      pr.weight = wnew;
      ++ens.accepted;
      ++naccept;
    }
  }
  return naccept;
}

void burn_in(WalkerEnsemble& ens, const WeightSpec& spec, long n_burn, bool adapt) {  // :81-93
  long long win_prop = 0, win_acc = 0;
  for (long s = 1; s <= n_burn; ++s) {
    win_acc += metropolis_step(ens, spec);
    win_prop += ens.m();
    if (adapt && s % 100 == 0) {
      const double rate = double(win_acc) / double(win_prop);
      ens.sigma_step = ens.sigma_step * (rate > 0.5 ? 1.1 : 1.0 / 1.1);
      win_prop = win_acc = 0;
    }
  }
  ens.proposed = ens.accepted = 0;
}

void WalkerEnsemble::save(std::ostream& os) const {  // sampler.cpp:95-105
  os << m() << ' ' << format_double(sigma_step) << ' ' << proposed << ' ' << accepted << '\n';
  os << rng.save() << '\n';
  for (const auto& p : pairs)
    os << format_double(p.r1.x) << ' ' << format_double(p.r1.y) << ' ' << format_double(p.r1.z)
       << ' ' << format_double(p.r2.x) << ' ' << format_double(p.r2.y) << ' '
       << format_double(p.r2.z) << ' ' << format_double(p.g1) << ' ' << format_double(p.g2) << ' '
       << format_double(p.weight) << '\n';
}

WalkerEnsemble WalkerEnsemble::load(std::istream& is) {  // sampler.cpp:107-120
  WalkerEnsemble e;
  int m = 0;
  is >> m >> e.sigma_step >> e.proposed >> e.accepted;
  e.rng = Philox::load(is);
  if (!is || m < 2) throw std::runtime_error("checkpoint: malformed ensemble record");
  e.pairs.resize(m);
  for (auto& p : e.pairs) {
    is >> p.r1.x >> p.r1.y >> p.r1.z >> p.r2.x >> p.r2.y >> p.r2.z >> p.g1 >> p.g2 >> p.weight;
    if (!is) throw std::runtime_error("checkpoint: malformed walker record");
  }
  return e;
}

// =============================================================== greens.cpp
double guarded_exp(double exponent, int spinor_index) {  // greens.cpp:9-16
  if (exponent > 700.0)
    throw std::runtime_error("greens: exponential overflow for spinor " +
                             std::to_string(spinor_index) +
                             " (positive occupied or negative virtual energy with large tau?)");
  if (exponent < -700.0) return 0.0;
  return std::exp(exponent);
}

TraceWorkspace::TraceWorkspace(const SpinorSet& s, int max_points)
    : s_(&s), nc_(s.ncomp), no_(s.n_occ), nv_(s.n_vir), max_points_(max_points) {  // greens.cpp:42-55
  occ_.resize(std::size_t(max_points) * nc_ * no_);
  occw_.resize(occ_.size());
  vir_.resize(std::size_t(max_points) * nc_ * nv_);
  virw_.resize(vir_.size());
  wocc_.resize(no_);
  wvir_.resize(nv_);
  chi_.resize(s.max_channel_size());
}

void TraceWorkspace::load_points(const Vec3* pts, int n) {  // greens.cpp:57-61
  if (n > max_points_) throw std::invalid_argument("TraceWorkspace: too many points");
  npoints = n;
  for (int i = 0; i < n; ++i)
    s_->evaluate_into(pts[i], &occ_[std::size_t(i) * nc_ * no_], &vir_[std::size_t(i) * nc_ * nv_],
                      chi_.data());
}

void TraceWorkspace::set_tau(double tau) {  // greens.cpp:63-71
  for (int i = 0; i < no_; ++i) wocc_[i] = guarded_exp(s_->energies[i] * tau, i);
  for (int a = 0; a < nv_; ++a) wvir_[a] = guarded_exp(-s_->energies[no_ + a] * tau, no_ + a);
  for (int p = 0; p < npoints; ++p) {
    for (int x = 0; x < nc_; ++x) {
      const std::size_t bo = (std::size_t(p) * nc_ + x) * no_, bv = (std::size_t(p) * nc_ + x) * nv_;
      for (int i = 0; i < no_; ++i) occw_[bo + i] = occ_[bo + i] * wocc_[i];
      for (int a = 0; a < nv_; ++a) virw_[bv + a] = vir_[bv + a] * wvir_[a];
    }
  }
}

namespace {
// out(x,y) = sum_k a[x][k] conj(b[y][k]) for nc x K row-major blocks (greens.cpp:73-79)
inline void outer_conj(const Complex* a, const Complex* b, int nc, int K, Complex* out) {
  const double* ad = reinterpret_cast<const double*>(a);
  const double* bd = reinterpret_cast<const double*>(b);
  for (int x = 0; x < nc; ++x)
    for (int y = 0; y < nc; ++y) {
      const double* ax = ad + 2 * std::size_t(x) * K;
      const double* by = bd + 2 * std::size_t(y) * K;
      double re = 0.0, im = 0.0;
      for (int k = 0; k < K; ++k) {
        const double ar = ax[2 * k], ai = ax[2 * k + 1], br = by[2 * k], bi = by[2 * k + 1];
        re += ar * br + ai * bi;
        im += ai * br - ar * bi;
      }
      out[x * nc + y] = Complex(re, im);
    }
}
}  // namespace

void TraceWorkspace::occupied(int d, int o, Complex* out) const {
  outer_conj(&occw_[std::size_t(d) * nc_ * no_], &occ_[std::size_t(o) * nc_ * no_], nc_, no_, out);
}

void TraceWorkspace::virtuals(int d, int o, Complex* out) const {
  outer_conj(&virw_[std::size_t(d) * nc_ * nv_], &vir_[std::size_t(o) * nc_ * nv_], nc_, nv_, out);
}

// =============================================================== estimator.cpp
EstimatorWorkspace::EstimatorWorkspace(const SpinorSet& s, int m)
    : traces(s, 2 * m), nc_(s.ncomp) {  // estimator.cpp:8-13
  points.resize(2 * m);
  for (auto* v : {&o1_, &o2_, &va_, &vb_, &vc_, &vd_}) v->assign(nc_ * nc_, Complex(0, 0));
}

SampleTerm EstimatorWorkspace::pair_term(int p, int q, double inv_weight,
                                         const PairPrefactors& w) {  // estimator.cpp:15-33
  const int a = 2 * p, b = 2 * p + 1;  // (r1, r2) <- walker p
  const int c = 2 * q, d = 2 * q + 1;  // (r3, r4) <- walker q
  traces.occupied(a, c, o1_.data());
  traces.occupied(b, d, o2_.data());
  traces.virtuals(c, a, va_.data());
  traces.virtuals(d, b, vb_.data());
  traces.virtuals(d, a, vc_.data());
  traces.virtuals(c, b, vd_.data());
  const int n = nc_;
  if (!physical) {
    // literal element-wise sums, no transpose (estimator.cpp:26-29): the parity default
    Complex f1d(0, 0), f2d(0, 0), f1x(0, 0), f2x(0, 0);
    for (int y = 0; y < n; ++y)
      for (int x = 0; x < n; ++x) {
        const int e = x * n + y;
        f1d += o1_[e] * va_[e];
        f2d += o2_[e] * vb_[e];
        f1x += o1_[e] * vc_[e];
        f2x += o2_[e] * vd_[e];
      }
    return SampleTerm{-w.direct * f1d * f2d * inv_weight, -w.exchange * f1x * f2x * inv_weight};
  }
  // opt-in physical form: Tr(o1 va) Tr(o2 vb) and Tr(o1 vd o2 vc)
  Complex t1(0, 0), t2(0, 0), tx(0, 0);
  for (int x = 0; x < n; ++x)
    for (int y = 0; y < n; ++y) {
      t1 += o1_[x * n + y] * va_[y * n + x];
      t2 += o2_[x * n + y] * vb_[y * n + x];
    }
  std::vector<Complex> m1(n * n, Complex(0, 0)), m2(n * n, Complex(0, 0));
  for (int x = 0; x < n; ++x)
    for (int y = 0; y < n; ++y)
      for (int k = 0; k < n; ++k) {
        m1[x * n + y] += o1_[x * n + k] * vd_[k * n + y];
        m2[x * n + y] += o2_[x * n + k] * vc_[k * n + y];
      }
  for (int x = 0; x < n; ++x)
    for (int y = 0; y < n; ++y) tx += m1[x * n + y] * m2[y * n + x];
  return SampleTerm{-w.direct * t1 * t2 * inv_weight, -w.exchange * tx * inv_weight};
}

StepEstimate mc_step_estimate_rows(const SpinorSet& s, const WalkerEnsemble& ens, double tau,
                                   const WeightSpec& spec, const TauSampler& ts,
                                   EstimatorWorkspace& ws, int p_begin, int p_end,
                                   long long* npairs_out) {  // estimator.cpp:35-63
  const int m = ens.m();
  for (int p = 0; p < m; ++p) {
    ws.points[2 * p] = ens.pairs[p].r1;
    ws.points[2 * p + 1] = ens.pairs[p].r2;
  }
  ws.traces.load_points(ws.points.data(), 2 * m);
  ws.traces.set_tau(tau);
  const PairPrefactors w = mp2_pair_prefactors(s.ncomp);
  const double ng2 = spec.ng() * spec.ng();
  const double wtau = ts.pdf(tau);
  StepEstimate est;
  double sum = 0.0, imag = 0.0;
  long long np = 0;
  for (int p = p_begin; p < p_end; ++p) {
    const auto& wp = ens.pairs[p];
    for (int q = p + 1; q < m; ++q) {
      const auto& wq = ens.pairs[q];
      const double inv_weight = ng2 / (wp.g1 * wp.g2 * wq.g1 * wq.g2 * wtau);
      const SampleTerm t = ws.pair_term(p, q, inv_weight, w);
      sum += t.total();
      imag += t.imag();
      est.direct_sum += t.direct;
      est.exchange_sum += t.exchange;
      ++np;
    }
  }
  const double npairs = 0.5 * m * (m - 1);
  est.value = sum / npairs;
  est.imag = imag / npairs;
  if (npairs_out) *npairs_out = np;
  return est;
}

StepEstimate mc_step_estimate(const SpinorSet& s, const WalkerEnsemble& ens, double tau,
                              const WeightSpec& spec, const TauSampler& ts, EstimatorWorkspace& ws) {
  return mc_step_estimate_rows(s, ens, tau, spec, ts, ws, 0, ens.m(), nullptr);
}

SampleTerm sample_term(const SpinorSet& s, const WalkerPair& p, const WalkerPair& q, double tau,
                       const WeightSpec& spec, const TauSampler& ts,
                       bool physical) {  // estimator.cpp:65-75
  if (tau < 0) throw std::invalid_argument("sample_term: tau must be non-negative");
  EstimatorWorkspace ws(s, 2);
  ws.physical = physical;
  ws.points = {p.r1, p.r2, q.r1, q.r2};
  ws.traces.load_points(ws.points.data(), 4);
  ws.traces.set_tau(tau);
  const double inv_weight = spec.ng() * spec.ng() / (p.g1 * p.g2 * q.g1 * q.g2 * ts.pdf(tau));
  return ws.pair_term(0, 1, inv_weight, mp2_pair_prefactors(s.ncomp));
}

BlockingAccumulator::BlockingAccumulator(long nb) : nb_(nb) {  // estimator.cpp:77-79
  if (nb_ < 1) throw std::invalid_argument("BlockingAccumulator: block size must be >= 1");
}

void BlockingAccumulator::add(double value, double imag) {  // estimator.cpp:81-91
  sum_ += value;
  imag_sum_ += imag;
  ++n_;
  partial_ += value;
  if (++in_block_ == nb_) {
    block_means_.push_back(partial_ / double(nb_));
    partial_ = 0.0;
    in_block_ = 0;
  }
}

double BlockingAccumulator::sigma() const {  // estimator.cpp:93-100 (mean includes partial block)
  const std::size_t k = block_means_.size();
  if (k == 0) return 0.0;
  const double m = mean();
  double s2 = 0.0;
  for (double b : block_means_) s2 += (b - m) * (b - m);
  return std::sqrt(s2 / double(k));
}

double BlockingAccumulator::sigma_bar() const {  // estimator.cpp:102-105
  const std::size_t k = block_means_.size();
  return k ? sigma() / std::sqrt(double(k)) : 0.0;
}

std::vector<BlockingAccumulator::TracePoint> BlockingAccumulator::trace() const {  // :107-121
  std::vector<TracePoint> out;
  double cum = 0.0;
  for (std::size_t k = 0; k < block_means_.size(); ++k) {
    cum += block_means_[k];
    const double mean_k = cum / double(k + 1);
    double s2 = 0.0;
    for (std::size_t j = 0; j <= k; ++j)
      s2 += (block_means_[j] - mean_k) * (block_means_[j] - mean_k);
    const double sigma_k = std::sqrt(s2 / double(k + 1));
    out.push_back({(long long)(k + 1) * nb_, mean_k, sigma_k / std::sqrt(double(k + 1))});
  }
  return out;
}

void BlockingAccumulator::restore(long long n, double sum, double imag_sum, long in_block,
                                  double partial, std::vector<double> means) {
  n_ = n;
  sum_ = sum;
  imag_sum_ = imag_sum;
  in_block_ = in_block;
  partial_ = partial;
  block_means_ = std::move(means);
}

// =============================================================== driver.cpp
namespace {
std::vector<std::string> tokenize(const std::string& line) {  // driver.cpp:18-26
  std::string clean = line;
  if (auto pos = clean.find('#'); pos != std::string::npos) clean.erase(pos);
  std::istringstream is(clean);
  std::vector<std::string> toks;
  std::string t;
  while (is >> t) toks.push_back(t);
  return toks;
}
long long to_ll(const std::string& tok, const std::string& key) {
  try {
    std::size_t used = 0;
    const long long v = std::stoll(tok, &used);
    if (used == tok.size()) return v;
  } catch (const std::exception&) {
  }
  throw std::runtime_error("config: key '" + key + "' expects an integer, got '" + tok + "'");
}
double to_d(const std::string& tok, const std::string& key) {
  try {
    std::size_t used = 0;
    const double v = std::stod(tok, &used);
    if (used == tok.size()) return v;
  } catch (const std::exception&) {
  }
  throw std::runtime_error("config: key '" + key + "' expects a number, got '" + tok + "'");
}
}  // namespace

void RunConfig::validate() const {  // driver.cpp:50-63
  if (spinor_path.empty()) throw std::runtime_error("config: no spinor file given");
  if (steps.has_value() == target_rel_err.has_value())
    throw std::runtime_error("config: exactly one stopping rule required (steps or target-rel-err)");
  if (steps && *steps < 1) throw std::runtime_error("config: steps must be positive");
  if (target_rel_err && !(*target_rel_err > 0))
    throw std::runtime_error("config: target-rel-err must be positive");
  if (walkers < 2) throw std::runtime_error("config: walkers must be >= 2");
  if (workers < 1) throw std::runtime_error("config: workers must be >= 1");
  if (block_size < 1) throw std::runtime_error("config: blocksize must be >= 1");
  if (burn_in < 0) throw std::runtime_error("config: burnin must be >= 0");
  if (checkpoint_interval < 1) throw std::runtime_error("config: checkpoint-interval must be >= 1");
  if (step_size && !(*step_size > 0)) throw std::runtime_error("config: step-size must be positive");
}

RunConfig parse_config_text(const std::string& text) {  // driver.cpp:65-121
  RunConfig cfg;
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    const auto toks = tokenize(line);
    if (toks.empty()) continue;
    const std::string& key = toks[0];
    auto want = [&](std::size_t n) {
      if (toks.size() != n + 1)
        throw std::runtime_error("config: key '" + key + "' expects " + std::to_string(n) +
                                 " value(s)");
    };
    if (key == "spinors") { want(1); cfg.spinor_path = toks[1]; }
    else if (key == "steps") { want(1); cfg.steps = to_ll(toks[1], key); }
    else if (key == "target-rel-err") { want(1); cfg.target_rel_err = to_d(toks[1], key); }
    else if (key == "walkers") { want(1); cfg.walkers = int(to_ll(toks[1], key)); }
    else if (key == "seed") { want(1); cfg.seed = std::uint64_t(to_ll(toks[1], key)); }
    else if (key == "workers") { want(1); cfg.workers = int(to_ll(toks[1], key)); }
    else if (key == "blocksize") { want(1); cfg.block_size = long(to_ll(toks[1], key)); }
    else if (key == "burnin") { want(1); cfg.burn_in = long(to_ll(toks[1], key)); }
    else if (key == "checkpoint") { want(1); cfg.checkpoint_path = toks[1]; }
    else if (key == "checkpoint-interval") { want(1); cfg.checkpoint_interval = long(to_ll(toks[1], key)); }
    else if (key == "trace") { want(1); cfg.trace_path = toks[1]; }
    else if (key == "step-size") { want(1); cfg.step_size = to_d(toks[1], key); }
    else if (key == "estimator") {
      want(1);
      if (toks[1] != "literal" && toks[1] != "physical")
        throw std::runtime_error("config: key 'estimator' expects literal or physical, got '" + toks[1] + "'");
      cfg.physical = toks[1] == "physical";
    }
    else if (key == "weight") {
      want(5);
      const int z = atomic_number(toks[1]);
      cfg.weight_overrides[z] = {to_d(toks[2], key), to_d(toks[3], key), to_d(toks[4], key),
                                 to_d(toks[5], key)};
    } else {
      throw std::runtime_error("config: unknown key '" + key + "'");
    }
  }
  return cfg;
}

std::uint64_t fnv1a64(const std::string& bytes) {  // driver.cpp:131-138
  std::uint64_t h = 14695981039346656037ull;
  for (unsigned char c : bytes) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

namespace {
void weight_lines(std::ostream& os, const RunConfig& c) {
  for (const auto& [z, w] : c.weight_overrides)
    os << "weight " << element_symbol(z) << ' ' << format_double(w.c1) << ' '
       << format_double(w.zeta1) << ' ' << format_double(w.c2) << ' ' << format_double(w.zeta2)
       << "\n";
}
}  // namespace

std::string canonical_config_text(const RunConfig& c) {  // driver.cpp:140-159
  std::ostringstream os;
  os << "blocksize " << c.block_size << "\n";
  os << "burnin " << c.burn_in << "\n";
  if (!c.checkpoint_path.empty()) os << "checkpoint " << c.checkpoint_path << "\n";
  os << "checkpoint-interval " << c.checkpoint_interval << "\n";
  os << "seed " << c.seed << "\n";
  os << "spinors " << c.spinor_path << "\n";
  if (c.step_size) os << "step-size " << format_double(*c.step_size) << "\n";
  if (c.physical) os << "estimator physical\n";
  if (c.steps) os << "steps " << *c.steps << "\n";
  if (c.target_rel_err) os << "target-rel-err " << format_double(*c.target_rel_err) << "\n";
  if (!c.trace_path.empty()) os << "trace " << c.trace_path << "\n";
  os << "walkers " << c.walkers << "\n";
  weight_lines(os, c);
  os << "workers " << c.workers << "\n";
  return os.str();
}

std::uint64_t config_hash(const RunConfig& c, std::uint64_t spinor_hash) {  // driver.cpp:161-172
  std::ostringstream os;
  os << "blocksize " << c.block_size << "\n";
  os << "burnin " << c.burn_in << "\n";
  os << "spinorhash " << spinor_hash << "\n";
  if (c.step_size) os << "step-size " << format_double(*c.step_size) << "\n";
  if (c.physical) os << "estimator physical\n";
  os << "walkers " << c.walkers << "\n";
  weight_lines(os, c);
  return fnv1a64(os.str());
}

std::uint64_t hash_file_contents(const std::string& path) {  // driver.cpp:174-181
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

namespace {
struct WorkerState {  // driver.cpp:200-205
  int index = 0;
  WalkerEnsemble ensemble;
  BlockingAccumulator acc{100};
  long long done = 0;
};

WorkerSummary summarize(const WorkerState& w) {  // driver.cpp:207-216
  const double re = w.acc.real_sum(), im = w.acc.imag_sum();
  return WorkerSummary{w.index,         w.acc.count(),
                       w.acc.mean(),    w.acc.sigma_bar(),
                       w.ensemble.acceptance_fraction(),
                       re != 0.0 ? std::abs(im) / std::abs(re) : std::abs(im)};
}

void write_checkpoint(const std::string& path, std::uint64_t hash, const RunConfig& cfg,
                      const std::vector<WorkerState>& workers) {  // driver.cpp:218-243
  const std::string tmp = path + ".tmp";
  {
    std::ofstream out(tmp);
    if (!out) throw std::runtime_error("cannot write checkpoint: " + tmp);
    out << "mcmp2-checkpoint 1\n";
    out << "confighash " << hash << "\n";
    out << "config-begin\n" << canonical_config_text(cfg) << "config-end\n";
    out << "workers " << workers.size() << "\n";
    for (const auto& w : workers) {
      out << "worker " << w.index << "\n";
      out << "steps " << w.acc.count() << "\n";
      out << "sums " << format_double(w.acc.real_sum()) << ' ' << format_double(w.acc.imag_sum())
          << "\n";
      out << "partial " << w.acc.in_block() << ' ' << format_double(w.acc.partial()) << "\n";
      out << "blocks " << w.acc.block_means().size() << "\n";
      for (double b : w.acc.block_means()) out << format_double(b) << "\n";
      out << "ensemble\n";
      w.ensemble.save(out);
      out << "end-worker\n";
    }
    if (!out) throw std::runtime_error("failed writing checkpoint: " + tmp);
  }
  std::filesystem::rename(tmp, path);
}

struct CheckpointData {
  std::uint64_t hash = 0;
  RunConfig config;
  std::vector<WorkerState> workers;
};

CheckpointData read_checkpoint(const std::string& path) {  // driver.cpp:251-305
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open checkpoint: " + path);
  std::string word;
  in >> word;
  if (word != "mcmp2-checkpoint") throw std::runtime_error("checkpoint: bad header");
  int version = 0;
  in >> version;
  if (version != 1) throw std::runtime_error("checkpoint: unsupported version");
  CheckpointData data;
  in >> word >> data.hash;
  if (word != "confighash") throw std::runtime_error("checkpoint: missing confighash");
  std::string line;
  std::getline(in, line);
  std::getline(in, line);
  if (line != "config-begin") throw std::runtime_error("checkpoint: missing config section");
  std::ostringstream cfg;
  while (std::getline(in, line) && line != "config-end") cfg << line << "\n";
  data.config = parse_config_text(cfg.str());
  std::size_t nw = 0;
  in >> word >> nw;
  if (word != "workers") throw std::runtime_error("checkpoint: missing workers record");
  for (std::size_t k = 0; k < nw; ++k) {
    WorkerState w;
    w.acc = BlockingAccumulator(data.config.block_size);
    in >> word >> w.index;
    if (word != "worker") throw std::runtime_error("checkpoint: missing worker record");
    long long steps = 0;
    double sum = 0, imag = 0, partial = 0;
    long in_block = 0;
    std::size_t nblocks = 0;
    in >> word >> steps;
    if (word != "steps") throw std::runtime_error("checkpoint: missing steps");
    in >> word >> sum >> imag;
    if (word != "sums") throw std::runtime_error("checkpoint: missing sums");
    in >> word >> in_block >> partial;
    if (word != "partial") throw std::runtime_error("checkpoint: missing partial");
    in >> word >> nblocks;
    if (word != "blocks") throw std::runtime_error("checkpoint: missing blocks");
    std::vector<double> means(nblocks);
    for (auto& b : means) in >> b;
    w.acc.restore(steps, sum, imag, in_block, partial, std::move(means));
    w.done = steps;
    in >> word;
    if (word != "ensemble") throw std::runtime_error("checkpoint: missing ensemble");
    w.ensemble = WalkerEnsemble::load(in);
    in >> word;
    if (word != "end-worker") throw std::runtime_error("checkpoint: missing end-worker");
    if (!in) throw std::runtime_error("checkpoint: truncated file");
    data.workers.push_back(std::move(w));
  }
  return data;
}

void write_worker_trace(const std::string& trace_path, const WorkerState& w) {  // :311-321
  const std::string path = trace_path + ".w" + std::to_string(w.index);
  const std::string tmp = path + ".tmp";
  {
    std::ofstream out(tmp);
    if (!out) throw std::runtime_error("cannot write trace file: " + tmp);
    for (const auto& t : w.acc.trace())
      out << t.n << ' ' << format_double(t.mean) << ' ' << format_double(t.sigma_bar) << "\n";
  }
  std::filesystem::rename(tmp, path);
}

void concatenate_traces(const std::string& trace_path, std::size_t nw) {  // :323-334
  std::ofstream out(trace_path);
  if (!out) throw std::runtime_error("cannot write trace file: " + trace_path);
  for (std::size_t k = 0; k < nw; ++k) {
    std::ifstream in(trace_path + ".w" + std::to_string(k));
    if (in) out << in.rdbuf();
  }
  out.close();
  for (std::size_t k = 0; k < nw; ++k) std::filesystem::remove(trace_path + ".w" + std::to_string(k));
}

class Engine {  // driver.cpp:336-475
 public:
  Engine(RunConfig cfg, std::vector<WorkerState> restored)
      : cfg_(std::move(cfg)), spinors_(load_spinor_set(cfg_.spinor_path)),
        hash_(config_hash(cfg_, hash_file_contents(cfg_.spinor_path))) {
    cfg_.validate();
    if (!spinors_.nuclei)
      throw std::runtime_error("spinor file has no nuclei record; the sampling weight needs it");
    spec_.emplace(*spinors_.nuclei, cfg_.weight_overrides);
    tau_.emplace(lambda_from_gap(spinors_));
    if (restored.empty()) {
      for (int w = 0; w < cfg_.workers; ++w) {
        WorkerState ws;
        ws.index = w;
        ws.acc = BlockingAccumulator(cfg_.block_size);
        ws.ensemble = init_ensemble(cfg_.walkers, *spinors_.nuclei, *spec_, cfg_.seed,
                                    std::uint32_t(w));
        if (cfg_.step_size) ws.ensemble.sigma_step = *cfg_.step_size;
        burn_in(ws.ensemble, *spec_, cfg_.burn_in, !cfg_.step_size.has_value());
        workers_.push_back(std::move(ws));
      }
    } else {
      workers_ = std::move(restored);
      for (auto& w : workers_) {
        if (w.ensemble.m() != cfg_.walkers)
          throw std::runtime_error("checkpoint: walker count disagrees with config");
        for (const auto& p : w.ensemble.pairs) {
          const double g1 = spec_->g(p.r1), g2 = spec_->g(p.r2);
          if (std::abs(g1 - p.g1) > 1e-12 * std::abs(g1) || std::abs(g2 - p.g2) > 1e-12 * std::abs(g2))
            throw std::runtime_error("checkpoint: cached walker weights disagree with recomputation");
        }
      }
    }
  }

  RunReport drive(const RunHooks& hooks) {  // driver.cpp:376-420
    if (hooks.record) hooks.record->assign(workers_.size(), {});
    long intervals = 0;
    bool on_target = false;
    for (;;) {
      std::vector<long long> chunks(workers_.size(), cfg_.checkpoint_interval);
      if (cfg_.steps)
        for (std::size_t w = 0; w < workers_.size(); ++w)
          chunks[w] = std::min<long long>(cfg_.checkpoint_interval,
                                          worker_share(*cfg_.steps, cfg_.workers, int(w)) - workers_[w].done);
      advance_parallel(chunks, hooks);
      ++intervals;
      if (!cfg_.checkpoint_path.empty()) write_checkpoint(cfg_.checkpoint_path, hash_, cfg_, workers_);
      if (!cfg_.trace_path.empty())
        for (const auto& w : workers_) write_worker_trace(cfg_.trace_path, w);
      if (cfg_.steps) {
        bool all_done = true;
        for (std::size_t w = 0; w < workers_.size(); ++w)
          if (workers_[w].done < worker_share(*cfg_.steps, cfg_.workers, int(w))) all_done = false;
        if (all_done) break;
      } else {
        bool ready = true;
        for (const auto& w : workers_)
          if (w.acc.block_means().empty()) ready = false;
        if (ready) {
          const MergedEstimate m = current_merged();
          if (m.sigma_bar > 0 && m.value != 0 && m.sigma_bar / std::abs(m.value) <= *cfg_.target_rel_err) {
            on_target = true;
            break;
          }
        }
      }
      if (hooks.abort_after_intervals > 0 && intervals >= hooks.abort_after_intervals)
        return make_report(false);
    }
    if (!cfg_.trace_path.empty()) concatenate_traces(cfg_.trace_path, workers_.size());
    return make_report(on_target);
  }

 private:
  void advance_parallel(const std::vector<long long>& chunks, const RunHooks& hooks) {  // :423-438
    std::vector<std::thread> threads;
    std::vector<std::exception_ptr> errors(workers_.size());
    for (std::size_t w = 0; w < workers_.size(); ++w)
      threads.emplace_back([this, w, &chunks, &errors, &hooks] {
        try {
          advance(workers_[w], chunks[w], hooks.record ? &(*hooks.record)[w] : nullptr);
        } catch (...) {
          errors[w] = std::current_exception();
        }
      });
    for (auto& t : threads) t.join();
    for (auto& e : errors)
      if (e) std::rethrow_exception(e);
  }

  void advance(WorkerState& w, long long nsteps, std::vector<StepRecord>* rec) {  // :440-450
    if (nsteps <= 0) return;
    EstimatorWorkspace ws(spinors_, cfg_.walkers);
    ws.physical = cfg_.physical;
    for (long long s = 0; s < nsteps; ++s) {
      metropolis_step(w.ensemble, *spec_);
      const double tau = tau_->sample(w.ensemble.rng.uniform());
      const StepEstimate est = mc_step_estimate(spinors_, w.ensemble, tau, *spec_, *tau_, ws);
      w.acc.add(est.value, est.imag);
      if (rec) {
        StepRecord r;
        r.tau = tau;
        r.est = est;
        for (const auto& p : w.ensemble.pairs)
          for (double v : {p.r1.x, p.r1.y, p.r1.z, p.r2.x, p.r2.y, p.r2.z, p.g1, p.g2})
            r.walkers.push_back(v);
        rec->push_back(std::move(r));
      }
    }
    w.done += nsteps;
  }

  MergedEstimate current_merged() const {
    std::vector<WorkerSummary> parts;
    for (const auto& w : workers_) parts.push_back(summarize(w));
    return merge_estimates(parts);
  }

  RunReport make_report(bool on_target) const {
    RunReport rep;
    for (const auto& w : workers_) rep.workers.push_back(summarize(w));
    rep.merged = merge_estimates(rep.workers);
    rep.stopped_on_target = on_target;
    return rep;
  }

  RunConfig cfg_;
  SpinorSet spinors_;
  std::uint64_t hash_;
  std::optional<WeightSpec> spec_;
  std::optional<TauSampler> tau_;
  std::vector<WorkerState> workers_;
};

CheckpointData read_and_check(const std::string& path) {
  CheckpointData data = read_checkpoint(path);
  const std::uint64_t expect = config_hash(data.config, hash_file_contents(data.config.spinor_path));
  if (expect != data.hash)
    throw std::runtime_error("checkpoint: config hash mismatch (spinor file or physics settings changed)");
  return data;
}
}  // namespace

RunReport run(const RunConfig& cfg, const RunHooks& hooks) {  // driver.cpp:477-480
  Engine e(cfg, {});
  return e.drive(hooks);
}

RunReport resume(const std::string& checkpoint, const RunHooks& hooks) {  // driver.cpp:482-491
  CheckpointData data = read_and_check(checkpoint);
  Engine e(data.config, std::move(data.workers));
  return e.drive(hooks);
}

MergedEstimate merge_checkpoint_files(const std::vector<std::string>& paths,
                                      std::vector<WorkerSummary>* parts_out) {  // :502-521
  if (paths.empty()) throw std::invalid_argument("merge: no checkpoint files");
  std::vector<WorkerSummary> parts;
  std::uint64_t hash = 0;
  bool first = true;
  for (const auto& p : paths) {
    CheckpointData d = read_checkpoint(p);
    if (first) {
      hash = d.hash;
      first = false;
    } else if (d.hash != hash) {
      throw std::runtime_error("merge: config hash mismatch between " + paths.front() + " and " + p);
    }
    for (const auto& w : d.workers) parts.push_back(summarize(w));
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
    os << "worker " << w.index << ": steps " << w.steps << ", I " << format_double(w.mean)
       << ", sigma_bar " << format_double(w.sigma_bar) << ", acceptance ";
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.3f", w.acceptance);
    os << buf << ", imag ratio ";
    std::snprintf(buf, sizeof buf, "%.2e", w.imag_ratio);
    os << buf << "\n";
  }
  return os.str();
}

}  // namespace oracle
