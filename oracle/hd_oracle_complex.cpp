// TEST INFRASTRUCTURE ONLY — complex-field restatement of the reference hot
// path: the reference templates every operator on Scalar,
// and with Scalar = std::complex<double> uses
//   * draws: normal_complex_vector(len) = (a_i + i a_{len+i}) / sqrt(2) from one
//     normal_vector(2 len)                                  (random.cpp:178-188)
//   * make_reflector, complex branch: r = |v1|/||v||, phase = v1/|v1| (1 if 0),
//     a = v/||v|| + phase e1, c = 1/(1+r), s = -conj(phase) (reflect.hpp:142-153)
//   * <w, x> conjugate-linear in w; the adjoint swaps s for conj(s)
//                                                           (reflect.hpp:70-83)
//   * Ginibre / Haar probes exactly as in the real case with those primitives
//     (ginibre.hpp:58-106, haar.hpp:40-67); left probes answer Q^H x.
// Pinned by the reference's complex tests (test_reflect.cpp:115-143,282-293,
// test_haar.cpp:113-131, test_ginibre.cpp:117-132) in tests/.
#include <algorithm>
#include <cmath>
#include <complex>
#include <limits>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hd_oracle.hpp"

namespace hdc {

using hdo::Index;
using Cx = std::complex<double>;
using CVec = std::vector<Cx>;

void require(bool c, const std::string& msg) {
  if (!c) throw std::invalid_argument(msg);
}

bool all_finite(const CVec& x) {
  for (const Cx& v : x)
    if (!std::isfinite(v.real()) || !std::isfinite(v.imag())) return false;
  return true;
}

double sq_norm(const Cx* x, Index n) {
  double s = 0.0;
  for (Index i = 0; i < n; ++i) s += std::norm(x[i]);
  return s;
}

Cx cdot(const Cx* w, const Cx* x, Index n) {  // sum conj(w_i) x_i
  Cx s = 0.0;
  for (Index i = 0; i < n; ++i) s += std::conj(w[i]) * x[i];
  return s;
}

CVec normals(hdo::RandomSource& src, Index len) {  // random.cpp:178-188
  const hdo::Vec v = src.normal_complex_vector(len);
  CVec out(static_cast<size_t>(len));
  for (Index i = 0; i < len; ++i) out[(size_t)i] = Cx(v[(size_t)(2 * i)], v[(size_t)(2 * i + 1)]);
  return out;
}

struct Reflector {
  Index dim = 0, offset = 0;
  CVec w;
  double c = 0.0;
  Cx s = 1.0;
  bool identity = true;
  void apply_in_place(CVec& x, bool adjoint) const {  // reflect.hpp:70-83
    require((Index)x.size() == dim, "Reflector::apply: dimension mismatch");
    if (identity) return;
    Cx* tail = x.data() + offset;
    const Index L = dim - offset;
    const Cx proj = cdot(w.data(), tail, L);
    const Cx f = c * proj;
    for (Index i = 0; i < L; ++i) tail[i] -= f * w[(size_t)i];
    const Cx lead = adjoint ? std::conj(s) : s;
    for (Index i = 0; i < L; ++i) tail[i] *= lead;
  }
};

Reflector make_reflector(const CVec& p, Index offset) {  // reflect.hpp:120-153
  const Index n = (Index)p.size();
  require(n >= 1, "make_reflector: empty vector");
  require(offset >= 0 && offset < n, "make_reflector: offset out of range");
  require(all_finite(p), "make_reflector: non-finite entries");
  Reflector r;
  r.dim = n;
  r.offset = offset;
  const Index L = n - offset;
  const double nrm2 = sq_norm(p.data() + offset, L);
  double nrm = std::sqrt(nrm2);
  if (!(nrm2 >= std::numeric_limits<double>::min() && nrm2 <= std::numeric_limits<double>::max())) {
    double scale = 0.0;  // stableNorm fallback
    for (Index i = 0; i < L; ++i) scale = std::max(scale, std::abs(p[(size_t)(offset + i)]));
    if (scale > 0.0) {
      double s = 0.0;
      for (Index i = 0; i < L; ++i) s += std::norm(p[(size_t)(offset + i)] / scale);
      nrm = scale * std::sqrt(s);
    } else {
      nrm = 0.0;
    }
  }
  if (nrm == 0.0) return r;  // identity
  const Cx v1 = p[(size_t)offset];
  const double rr = std::abs(v1) / nrm;
  const Cx phase = (std::abs(v1) == 0.0) ? Cx(1.0) : v1 / std::abs(v1);
  r.w.resize((size_t)L);
  for (Index i = 0; i < L; ++i) r.w[(size_t)i] = p[(size_t)(offset + i)] / nrm;
  r.w[0] += phase;
  r.c = 1.0 / (1.0 + rr);
  r.s = -std::conj(phase);
  r.identity = false;
  return r;
}

struct Chain {  // reflect.hpp:193-231
  Index dim;
  std::vector<Reflector> m;
  void apply_in_place(CVec& x, bool reverse, bool adjoint) const {
    if (!reverse)
      for (const auto& h : m) h.apply_in_place(x, adjoint);
    else
      for (auto it = m.rbegin(); it != m.rend(); ++it) it->apply_in_place(x, adjoint);
  }
  CVec apply(const CVec& x, bool reverse, bool adjoint) const {
    CVec y = x;
    apply_in_place(y, reverse, adjoint);
    return y;
  }
};

struct Operator {
  virtual ~Operator() = default;
  virtual Index rows() const = 0;
  virtual Index cols() const = 0;
  virtual Index remaining() const = 0;
  virtual CVec probe(const CVec& x, int side) = 0;  // 0 right, 1 left
  void check(const CVec& x, int side) const {      // operators.hpp:44-48
    require((Index)x.size() == (side == 0 ? cols() : rows()), "probe: input dimension mismatch");
    require(all_finite(x), "probe: non-finite input");
  }
};

struct Ginibre final : Operator {  // ginibre.hpp:26-118 with Scalar = complex
  Index m, n;
  double sigma;
  hdo::RandomSource src;
  Chain L, R;
  std::vector<CVec> us, vs;
  Index r = 0, l = 0;
  bool skip;
  Ginibre(Index m_, Index n_, double s_, hdo::RandomSource src_, bool skip_)
      : m(m_), n(n_), sigma(s_), src(std::move(src_)), L{m_, {}}, R{n_, {}}, skip(skip_) {
    require(m >= 1 && n >= 1, "GinibreOperator: dims must be positive");
    require(sigma > 0.0, "GinibreOperator: sigma must be positive");
  }
  Index rows() const override { return m; }
  Index cols() const override { return n; }
  Index remaining() const override { return std::min(m, n) - (r + l); }
  CVec probe(const CVec& x, int side) override {
    check(x, side);
    if (remaining() == 0) throw hdo::BudgetExhausted("GinibreOperator: probe budget min(m, n) spent");
    const bool first = (r + l == 0);
    CVec y;
    if (side == 0) {
      ++r;
      CVec g = normals(src, m);
      CVec p = R.apply(x, false, false);
      Reflector h = make_reflector(p, r - 1);
      if (!(skip && first)) R.m.push_back(std::move(h));
      for (Index i = 0; i < l; ++i) g[(size_t)i] = 0.0;
      L.apply_in_place(g, true, true);
      CVec v((size_t)n, Cx(0.0));
      v[(size_t)(r - 1)] = 1.0;
      R.apply_in_place(v, true, true);
      us.push_back(std::move(g));
      vs.push_back(std::move(v));
      y.assign((size_t)m, Cx(0.0));
      for (size_t i = 0; i < us.size(); ++i) {
        const Cx cf = cdot(vs[i].data(), x.data(), n);
        for (Index k = 0; k < m; ++k) y[(size_t)k] += cf * us[i][(size_t)k];
      }
    } else {
      ++l;
      CVec g = normals(src, n);
      CVec q = L.apply(x, false, false);
      Reflector h = make_reflector(q, l - 1);
      if (!(skip && first)) L.m.push_back(std::move(h));
      for (Index i = 0; i < r; ++i) g[(size_t)i] = 0.0;
      R.apply_in_place(g, true, true);
      CVec u((size_t)m, Cx(0.0));
      u[(size_t)(l - 1)] = 1.0;
      L.apply_in_place(u, true, true);
      us.push_back(std::move(u));
      vs.push_back(std::move(g));
      y.assign((size_t)n, Cx(0.0));
      for (size_t i = 0; i < us.size(); ++i) {
        const Cx cf = cdot(us[i].data(), x.data(), m);
        for (Index k = 0; k < n; ++k) y[(size_t)k] += cf * vs[i][(size_t)k];
      }
    }
    for (Cx& v : y) v *= sigma;
    return y;
  }
};

struct Haar final : Operator {  // haar.hpp:21-91 with Scalar = complex
  Index n;
  hdo::RandomSource src;
  Chain Rc, Lc;
  Index t = 0;
  bool skip;
  Haar(Index n_, hdo::RandomSource src_, bool skip_) : n(n_), src(std::move(src_)), Rc{n_, {}}, Lc{n_, {}}, skip(skip_) {
    require(n >= 1, "HaarOperator: n must be positive");
  }
  Index rows() const override { return n; }
  Index cols() const override { return n; }
  Index remaining() const override { return n - t; }
  CVec probe(const CVec& x, int side) override {
    check(x, side);
    if (t == n) throw hdo::BudgetExhausted("HaarOperator: probe budget n spent");
    const bool first = (t == 0);
    ++t;
    const Index off = t - 1;
    CVec g = normals(src, n);
    Chain& fold = (side == 0) ? Rc : Lc;
    Chain& other = (side == 0) ? Lc : Rc;
    CVec p = fold.apply(x, false, false);
    Reflector hf = make_reflector(p, off);
    Reflector hm = make_reflector(g, off);
    CVec z = p;
    hf.apply_in_place(z, false);
    if (!(skip && first)) fold.m.push_back(std::move(hf));
    other.m.push_back(std::move(hm));
    other.apply_in_place(z, true, true);
    return z;
  }
};

CVec from_interleaved(const double* p, Index n) {
  CVec v((size_t)n);
  for (Index i = 0; i < n; ++i) v[(size_t)i] = Cx(p[2 * i], p[2 * i + 1]);
  return v;
}

void to_interleaved(const CVec& v, double* out) {
  for (size_t i = 0; i < v.size(); ++i) {
    out[2 * i] = v[i].real();
    out[2 * i + 1] = v[i].imag();
  }
}

thread_local std::string g_err;

int fail() {
  try {
    throw;
  } catch (const hdo::BudgetExhausted& e) {
    g_err = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

}  // namespace hdc

extern "C" {

const char* or_c_last_error() { return hdc::g_err.c_str(); }

int or_c_make_reflector(const double* p, std::int64_t n, std::int64_t off, double* w, double* c, double* s, int* ident) {
  try {
    const hdc::Reflector r = hdc::make_reflector(hdc::from_interleaved(p, n), off);
    *ident = r.identity ? 1 : 0;
    *c = r.c;
    s[0] = r.s.real();
    s[1] = r.s.imag();
    if (!r.identity) hdc::to_interleaved(r.w, w);
    return 0;
  } catch (...) {
    return hdc::fail();
  }
}

int or_c_reflector_apply(const double* p, std::int64_t n, std::int64_t off, const double* x, int adjoint, double* y) {
  try {
    const hdc::Reflector r = hdc::make_reflector(hdc::from_interleaved(p, n), off);
    hdc::CVec v = hdc::from_interleaved(x, n);
    r.apply_in_place(v, adjoint != 0);
    hdc::to_interleaved(v, y);
    return 0;
  } catch (...) {
    return hdc::fail();
  }
}

// chain of reflectors built from vectors p_k (interleaved, k x n) at offsets k
int or_c_chain_apply(const double* ps, std::int64_t k, std::int64_t n, const double* x, int reverse, int adjoint,
                     double* y) {
  try {
    hdc::Chain ch{n, {}};
    for (std::int64_t j = 0; j < k; ++j) ch.m.push_back(hdc::make_reflector(hdc::from_interleaved(ps + 2 * j * n, n), j));
    hdc::to_interleaved(ch.apply(hdc::from_interleaved(x, n), reverse != 0, adjoint != 0), y);
    return 0;
  } catch (...) {
    return hdc::fail();
  }
}

int or_c_op_new(int ensemble, std::int64_t m, std::int64_t n, double sigma, std::uint64_t seed, std::uint64_t stream,
                int skip, void** out) {
  try {
    hdo::RandomSource src(seed, stream);
    if (ensemble == 0)
      *out = new hdc::Ginibre(m, n, sigma, std::move(src), skip != 0);
    else if (ensemble == 1)
      *out = new hdc::Haar(n, std::move(src), skip != 0);
    else
      throw std::invalid_argument("or_c_op_new: complex operators are Ginibre (0) or Haar (1)");
    return 0;
  } catch (...) {
    return hdc::fail();
  }
}

void or_c_op_free(void* op) { delete static_cast<hdc::Operator*>(op); }

std::int64_t or_c_op_remaining(void* op) { return static_cast<hdc::Operator*>(op)->remaining(); }

int or_c_op_probe(void* op, const double* x, std::int64_t xlen, int side, double* y, std::int64_t ylen) {
  try {
    auto* o = static_cast<hdc::Operator*>(op);
    const hdc::CVec out = o->probe(hdc::from_interleaved(x, xlen), side);
    if ((std::int64_t)out.size() != ylen) throw std::invalid_argument("probe: output dimension mismatch");
    hdc::to_interleaved(out, y);
    return 0;
  } catch (...) {
    return hdc::fail();
  }
}

}  // extern "C"
