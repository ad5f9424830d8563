// TEST INFRASTRUCTURE ONLY — see hd_oracle.hpp. Restates the reference hot
// path (/root/reference/proj) in plain C++; every function cites the
// reference file:line it follows. Exposed to Python through the extern "C"
// block at the bottom (ctypes), used only by tests/, smoke() and bench.py's
// cpu_baseline / --impl reference legs.
#include "hd_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <limits>
#include <mutex>
#include <thread>

#if defined(__AVX2__)
#include <immintrin.h>
#endif

namespace hdo {

// ======================================================================= RNG
namespace {

// random.cpp:11-16 — splitmix64 state expansion.
std::uint64_t splitmix64(std::uint64_t& x) {
  std::uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// random.cpp:18-69 — 256-strip ziggurat for exp(-x^2/2). Tail boundary R is
// the 256-strip constant; strip s >= 1 spans [0, x_s]; strip 0 is the base
// strip whose overhang beyond R holds the Gaussian tail mass.
constexpr double kR = 3.6541528853610088;

struct Zig {
  std::array<double, 256> w{};
  std::array<double, 256> f{};
  std::array<std::uint64_t, 256> k{};
};

Zig build_zig() {
  const double fR = std::exp(-0.5 * kR * kR);
  const double tail = std::sqrt(1.5707963267948966) * std::erfc(kR / std::sqrt(2.0));
  const double area = kR * fR + tail;
  std::array<double, 256> x{};
  x[255] = kR;
  for (int s = 254; s >= 1; --s) {
    const double up = std::exp(-0.5 * x[s + 1] * x[s + 1]);
    x[s] = std::sqrt(-2.0 * std::log(area / x[s + 1] + up));
  }
  x[0] = 0.0;
  require(std::abs(area / x[1] + std::exp(-0.5 * x[1] * x[1]) - 1.0) < 1e-6,
          "ziggurat table generation drifted");
  Zig z;
  z.w[0] = area / fR;
  z.k[0] = static_cast<std::uint64_t>(kR * fR / area * 0x1.0p52);
  z.f[0] = 1.0;
  for (int s = 1; s < 256; ++s) {
    z.w[s] = x[s];
    z.k[s] = static_cast<std::uint64_t>(x[s - 1] / x[s] * 0x1.0p52);
    z.f[s] = std::exp(-0.5 * x[s] * x[s]);
  }
  return z;
}

const Zig& zig() {
  static const Zig z = build_zig();
  return z;
}

}  // namespace

std::uint64_t derive_seed(std::uint64_t base, std::uint64_t index) {  // random.cpp:73-76
  std::uint64_t s = base + index * 0x9e3779b97f4a7c15ULL;
  return splitmix64(s);
}

Xoshiro256pp::Xoshiro256pp(std::uint64_t seed) {  // random.cpp:78-81
  std::uint64_t s = seed;
  for (auto& w : s_) w = splitmix64(s);
}

void Xoshiro256pp::jump() {  // random.cpp:83-99 (2^128 steps)
  static constexpr std::uint64_t J[4] = {0x180ec6d33cfd0abaULL, 0xd5a61266f0c9392cULL,
                                         0xa9582618e03fc9aaULL, 0x39abdc4529b1661cULL};
  std::array<std::uint64_t, 4> acc{0, 0, 0, 0};
  for (std::uint64_t word : J) {
    for (int b = 0; b < 64; ++b) {
      if ((word >> b) & 1ULL) {
        for (int i = 0; i < 4; ++i) acc[i] ^= s_[i];
      }
      next();
    }
  }
  s_ = acc;
}

RandomSource::RandomSource(std::uint64_t seed, std::uint64_t stream) : eng_(seed) {  // random.cpp:101-104
  for (std::uint64_t i = 0; i < stream; ++i) eng_.jump();
}

double RandomSource::normal() {  // random.cpp:106-121 (Marsaglia polar)
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  double u, v, q;
  do {
    u = 2.0 * uniform() - 1.0;
    v = 2.0 * uniform() - 1.0;
    q = u * u + v * v;
  } while (q >= 1.0 || q == 0.0);
  const double f = std::sqrt(-2.0 * std::log(q) / q);
  spare_ = v * f;
  has_spare_ = true;
  return u * f;
}

Vec RandomSource::normal_vector(Index len) {  // random.cpp:130-176
  require(len >= 1, "normal_vector: len must be >= 1");
  if (queue_) {  // test hook: the queued draws (set_queue)
    require(qpos_ + static_cast<size_t>(len) <= queue_->size(), "normal_vector: draw queue exhausted");
    Vec out(queue_->begin() + static_cast<std::ptrdiff_t>(qpos_),
            queue_->begin() + static_cast<std::ptrdiff_t>(qpos_ + static_cast<size_t>(len)));
    qpos_ += static_cast<size_t>(len);
    return out;
  }
  const Zig& z = zig();
  Xoshiro256pp e = eng_;
  auto u53 = [&e] { return static_cast<double>(e.next() >> 11) * 0x1.0p-53; };
  Vec out(static_cast<size_t>(len));
  for (Index i = 0; i < len; ++i) {
    for (;;) {
      const std::uint64_t bits = e.next();
      const unsigned s = static_cast<unsigned>(bits & 0xFF);
      const std::uint64_t mant = bits >> 12;
      const double mag = (std::bit_cast<double>(0x3FF0000000000000ULL | mant) - 1.0) * z.w[s];
      const std::uint64_t sgn = (bits & 0x100) << 55;
      if (mant < z.k[s]) {
        out[static_cast<size_t>(i)] = std::bit_cast<double>(std::bit_cast<std::uint64_t>(mag) ^ sgn);
        break;
      }
      if (s == 0) {
        double e1, e2;
        do {
          e1 = -std::log1p(-u53()) * (1.0 / kR);
          e2 = -std::log1p(-u53());
        } while (e2 + e2 <= e1 * e1);
        out[static_cast<size_t>(i)] = std::bit_cast<double>(std::bit_cast<std::uint64_t>(kR + e1) ^ sgn);
        break;
      }
      const double wedge = z.f[s] + u53() * (z.f[s - 1] - z.f[s]);
      if (wedge < std::exp(-0.5 * mag * mag)) {
        out[static_cast<size_t>(i)] = std::bit_cast<double>(std::bit_cast<std::uint64_t>(mag) ^ sgn);
        break;
      }
    }
  }
  eng_ = e;
  return out;
}

Vec RandomSource::normal_complex_vector(Index len) {  // random.cpp:178-188
  require(len >= 1, "normal_complex_vector: len must be >= 1");
  constexpr double h = 0.7071067811865475244;
  const Vec parts = normal_vector(2 * len);
  Vec out(static_cast<size_t>(2 * len));
  for (Index i = 0; i < len; ++i) {
    out[static_cast<size_t>(2 * i)] = parts[static_cast<size_t>(i)] * h;
    out[static_cast<size_t>(2 * i + 1)] = parts[static_cast<size_t>(len + i)] * h;
  }
  return out;
}

// ============================================================ vector kernels
// Multi-accumulator dot product: Eigen's packet reduction (reflect.hpp:74
// `w_.dot(tail)`) keeps several partial sums; a single scalar chain would
// make the CPU baseline artificially slow. Summation order is therefore not
// sequential — Eigen's order is itself unpinned (see header).
static double dot(const double* a, const double* b, Index n) {
#if defined(__AVX2__) && defined(__FMA__)
  __m256d s0 = _mm256_setzero_pd(), s1 = _mm256_setzero_pd();
  __m256d s2 = _mm256_setzero_pd(), s3 = _mm256_setzero_pd();
  Index i = 0;
  for (; i + 16 <= n; i += 16) {
    s0 = _mm256_fmadd_pd(_mm256_loadu_pd(a + i), _mm256_loadu_pd(b + i), s0);
    s1 = _mm256_fmadd_pd(_mm256_loadu_pd(a + i + 4), _mm256_loadu_pd(b + i + 4), s1);
    s2 = _mm256_fmadd_pd(_mm256_loadu_pd(a + i + 8), _mm256_loadu_pd(b + i + 8), s2);
    s3 = _mm256_fmadd_pd(_mm256_loadu_pd(a + i + 12), _mm256_loadu_pd(b + i + 12), s3);
  }
  __m256d s = _mm256_add_pd(_mm256_add_pd(s0, s1), _mm256_add_pd(s2, s3));
  alignas(32) double t[4];
  _mm256_store_pd(t, s);
  double acc = (t[0] + t[1]) + (t[2] + t[3]);
  for (; i < n; ++i) acc += a[i] * b[i];
  return acc;
#else
  double p[4] = {0, 0, 0, 0};
  Index i = 0;
  for (; i + 4 <= n; i += 4)
    for (int j = 0; j < 4; ++j) p[j] += a[i + j] * b[i + j];
  double acc = (p[0] + p[1]) + (p[2] + p[3]);
  for (; i < n; ++i) acc += a[i] * b[i];
  return acc;
#endif
}

static bool all_finite(const Vec& x) {
  for (double v : x)
    if (!std::isfinite(v)) return false;
  return true;
}

static double sq_norm(const double* a, Index n) { return dot(a, a, n); }

// Eigen stableNorm stand-in: scaled sum of squares (no overflow/underflow).
static double stable_norm(const double* a, Index n) {
  double scale = 0.0;
  for (Index i = 0; i < n; ++i) scale = std::max(scale, std::abs(a[i]));
  if (scale == 0.0 || !std::isfinite(scale)) return scale;
  double s = 0.0;
  for (Index i = 0; i < n; ++i) {
    const double v = a[i] / scale;
    s += v * v;
  }
  return scale * std::sqrt(s);
}

static double norm(const Vec& x) { return std::sqrt(sq_norm(x.data(), static_cast<Index>(x.size()))); }

// ================================================================ reflectors
void Reflector::apply_in_place(Vec& x) const {  // reflect.hpp:70-83
  require(static_cast<Index>(x.size()) == dim, "Reflector::apply: dimension mismatch");
  if (identity) return;
  double* t = x.data() + offset;
  const Index len = dim - offset;
  const double cp = c * dot(w.data(), t, len);
  const double* wp = w.data();
  for (Index i = 0; i < len; ++i) t[i] = (t[i] - cp * wp[i]) * s;
}

Reflector make_reflector(const Vec& p, Index offset, double zero_tol, SignRule rule) {  // reflect.hpp:120-176
  const Index n = static_cast<Index>(p.size());
  require(n >= 1, "make_reflector: empty vector");
  require(offset >= 0 && offset < n, "make_reflector: offset out of range");
  require(all_finite(p), "make_reflector: non-finite entries");
  const double* tail = p.data() + offset;
  const Index len = n - offset;
  const double nrm2 = sq_norm(tail, len);
  const double nrm = (nrm2 >= std::numeric_limits<double>::min() &&
                      nrm2 <= std::numeric_limits<double>::max())
                         ? std::sqrt(nrm2)
                         : stable_norm(tail, len);
  Reflector r;
  r.dim = n;
  r.offset = offset;
  if (nrm == 0.0 || (zero_tol > 0.0 && nrm <= zero_tol * stable_norm(p.data(), n))) {
    return r;  // identity: c = 0, s = 1
  }
  const double v1 = tail[0];
  double sign = 1.0;
  switch (rule) {
    case SignRule::stable: sign = (v1 >= 0.0) ? 1.0 : -1.0; break;
    case SignRule::negative_at_zero: sign = (v1 > 0.0) ? 1.0 : -1.0; break;
    case SignRule::zero_when_negative: sign = (v1 >= 0.0) ? 1.0 : 0.0; break;
  }
  r.w.resize(static_cast<size_t>(len));
  for (Index i = 0; i < len; ++i) r.w[static_cast<size_t>(i)] = tail[i] / nrm;
  r.w[0] += sign;
  r.c = 2.0 / sq_norm(r.w.data(), len);
  r.s = -sign;
  r.identity = false;
  return r;
}

void ReflectorChain::apply_forward(Vec& x) const {  // reflect.hpp:211-215
  require(static_cast<Index>(x.size()) == dim_, "ReflectorChain::apply: dimension mismatch");
  for (const auto& r : m_) r.apply_in_place(x);
}

void ReflectorChain::apply_reverse(Vec& x) const {  // reflect.hpp:216-219
  require(static_cast<Index>(x.size()) == dim_, "ReflectorChain::apply: dimension mismatch");
  for (auto it = m_.rbegin(); it != m_.rend(); ++it) it->apply_in_place(x);
}

// ================================================================= operators
void ProbeOperator::check_probe_input(const Vec& x, Side side) const {  // operators.hpp:44-48
  const Index want = (side == Side::right) ? cols() : rows();
  require(static_cast<Index>(x.size()) == want, "probe: input dimension mismatch");
  require(all_finite(x), "probe: non-finite input");
}

GinibreOperator::GinibreOperator(Index m, Index n, double sigma, RandomSource src, FaultFlags f)
    : m_(m), n_(n), sigma_(sigma), src_(std::move(src)), L_(m >= 1 ? m : 1), R_(n >= 1 ? n : 1), f_(f) {
  require(m >= 1 && n >= 1, "GinibreOperator: dims must be positive");  // ginibre.hpp:40-41
  require(sigma > 0.0, "GinibreOperator: sigma must be positive");
}

Vec GinibreOperator::probe(const Vec& x, Side side) {  // ginibre.hpp:58-106
  check_probe_input(x, side);
  if (remaining_probes() == 0) throw BudgetExhausted("GinibreOperator: probe budget min(m, n) spent");
  const bool first = (r_ + l_ == 0);
  Vec y;
  if (side == Side::right) {
    ++r_;
    Vec g = src_.normal_vector(m_);
    Vec p = x;
    R_.apply_forward(p);
    Reflector h = make_reflector(p, r_ - 1, 0.0, f_.sign_rule);
    if (!(f_.skip_reflector && first)) R_.append(std::move(h));
    std::fill(g.begin(), g.begin() + l_, 0.0);
    L_.apply_reverse(g);
    Vec v(static_cast<size_t>(n_), 0.0);
    v[static_cast<size_t>(r_ - 1)] = 1.0;
    R_.apply_reverse(v);
    us_.push_back(std::move(g));
    vs_.push_back(std::move(v));
    y.assign(static_cast<size_t>(m_), 0.0);
    for (size_t i = 0; i < us_.size(); ++i) {
      const double a = dot(vs_[i].data(), x.data(), n_);
      const double* u = us_[i].data();
      for (Index j = 0; j < m_; ++j) y[static_cast<size_t>(j)] += a * u[j];
    }
  } else {
    ++l_;
    Vec g = src_.normal_vector(n_);
    Vec q = x;
    L_.apply_forward(q);
    Reflector h = make_reflector(q, l_ - 1, 0.0, f_.sign_rule);
    if (!(f_.skip_reflector && first)) L_.append(std::move(h));
    std::fill(g.begin(), g.begin() + r_, 0.0);
    R_.apply_reverse(g);
    Vec u(static_cast<size_t>(m_), 0.0);
    u[static_cast<size_t>(l_ - 1)] = 1.0;
    L_.apply_reverse(u);
    us_.push_back(std::move(u));
    vs_.push_back(std::move(g));
    y.assign(static_cast<size_t>(n_), 0.0);
    for (size_t i = 0; i < us_.size(); ++i) {
      const double a = dot(us_[i].data(), x.data(), m_);
      const double* v = vs_[i].data();
      for (Index j = 0; j < n_; ++j) y[static_cast<size_t>(j)] += a * v[j];
    }
  }
  for (double& v : y) v *= sigma_;  // ginibre.hpp:104 — sigma applied last
  return y;
}

HaarOperator::HaarOperator(Index n, RandomSource src, FaultFlags f)
    : n_(n), src_(std::move(src)), L_(n >= 1 ? n : 1), R_(n >= 1 ? n : 1), f_(f) {
  require(n >= 1, "HaarOperator: n must be positive");  // haar.hpp:30
}

Vec HaarOperator::probe(const Vec& x, Side side) {  // haar.hpp:40-67
  check_probe_input(x, side);
  if (t_ == n_) throw BudgetExhausted("HaarOperator: probe budget n spent");
  const bool first = (t_ == 0);
  ++t_;
  const Index off = t_ - 1;
  Vec g = src_.normal_vector(n_);
  ReflectorChain& fold_chain = (side == Side::right) ? R_ : L_;
  ReflectorChain& other = (side == Side::right) ? L_ : R_;
  Vec p = x;
  fold_chain.apply_forward(p);
  Reflector fold = make_reflector(p, off, 0.0, f_.sign_rule);
  Reflector mix = make_reflector(g, off, 0.0, f_.sign_rule);
  Vec z = p;
  fold.apply_in_place(z);
  if (!(f_.skip_reflector && first)) fold_chain.append(std::move(fold));
  other.append(std::move(mix));
  other.apply_reverse(z);
  return z;
}

GOEOperator::GOEOperator(Index n, double inner_sigma, RandomSource src, FaultFlags f)
    : inner_(n, n, inner_sigma, std::move(src), f) {}

Vec GOEOperator::probe(const Vec& x, Side) {  // ensembles.hpp:117-127
  check_probe_input(x, Side::right);
  if (remaining_probes() == 0) throw BudgetExhausted("GOEOperator: budget floor(n/2) spent");
  constexpr double h = 0.7071067811865475244;
  Vec y = inner_.probe(x, Side::right);
  const Vec yl = inner_.probe(x, Side::left);
  for (size_t i = 0; i < y.size(); ++i) y[i] = (y[i] + yl[i]) * h;
  return y;
}

// ================================================================== dynamics
std::vector<Vec> run_dynamics(ProbeOperator& op, const DynamicsSpec& spec) {  // dynamics.hpp:42-76
  require(spec.iterations >= 0, "run_dynamics: negative iteration count");
  require(spec.history_depth >= 0, "run_dynamics: negative history depth");
  require(static_cast<Index>(spec.initial.size()) == spec.history_depth + 1,
          "run_dynamics: initial history must hold d + 1 vectors");
  require(static_cast<bool>(spec.side_of), "run_dynamics: no side schedule");
  require(static_cast<bool>(spec.update), "run_dynamics: no update map");
  require(spec.iterations <= op.remaining_probes(),
          "run_dynamics: iteration count exceeds the operator's probe budget");
  std::vector<Vec> history = spec.initial;
  std::vector<Vec> traj;
  if (spec.keep_trajectory) traj.push_back(history.front());
  for (Index t = 1; t <= spec.iterations; ++t) {
    const Side side = spec.side_of(t);
    const Vec y = op.probe(history.front(), side);
    Vec next = spec.update(t, y, history);
    if (!all_finite(next))
      throw std::runtime_error("run_dynamics: non-finite iterate at step " + std::to_string(t));
    history.insert(history.begin(), next);
    history.pop_back();
    if (spec.keep_trajectory) traj.push_back(std::move(next));
  }
  if (!spec.keep_trajectory) traj.push_back(history.front());
  return traj;
}

static DynamicsSpec builtin_spec(UpdateKind kind, SideRule rule, Index T, const Vec& x1, const Vec* x0,
                                 bool keep) {
  DynamicsSpec spec;
  spec.iterations = T;
  spec.keep_trajectory = keep;
  switch (rule) {
    case SideRule::alternate: spec.side_of = [](Index t) { return (t % 2 == 1) ? Side::right : Side::left; }; break;
    case SideRule::all_right: spec.side_of = [](Index) { return Side::right; }; break;
    case SideRule::all_left: spec.side_of = [](Index) { return Side::left; }; break;
  }
  switch (kind) {
    case UpdateKind::identity:
      spec.history_depth = 0;
      spec.initial = {x1};
      spec.update = [](Index, const Vec& y, const std::vector<Vec>&) { return y; };
      break;
    case UpdateKind::normalize:  // bench.cpp:25-28
      spec.history_depth = 0;
      spec.initial = {x1};
      spec.update = [](Index, const Vec& y, const std::vector<Vec>&) {
        const double nrm = norm(y);
        const double inv = nrm > 0 ? 1.0 / nrm : 1.0;
        Vec out(y.size());
        for (size_t i = 0; i < y.size(); ++i) out[i] = inv * y[i];
        return out;
      };
      break;
    case UpdateKind::tanh_mix:  // BASELINE config 2
      spec.history_depth = 1;
      spec.initial = {x1, x0 ? *x0 : Vec(x1.size(), 0.0)};
      spec.update = [](Index, const Vec& y, const std::vector<Vec>& h) {
        Vec out(y.size());
        const Vec& prev = h[1];
        for (size_t i = 0; i < y.size(); ++i) out[i] = std::tanh(2.0 * y[i]) + 0.1 * prev[i];
        return out;
      };
      break;
  }
  return spec;
}

}  // namespace hdo

// =============================================================== C interface
using namespace hdo;

namespace {
thread_local std::string g_err;

int fail_from_current() {
  try {
    throw;
  } catch (const BudgetExhausted& e) {
    g_err = e.what();
    return 2;
  } catch (const ResourceCapExceeded& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  } catch (...) {
    g_err = "unknown error";
    return 4;
  }
}

struct OpBox {
  int ensemble = 0;  // 0 ginibre, 1 haar, 2 goe
  std::unique_ptr<ProbeOperator> op;
};
}  // namespace

#define OR_TRY try {
#define OR_CATCH \
  }              \
  catch (...) { return fail_from_current(); }

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

std::uint64_t or_derive_seed(std::uint64_t base, std::uint64_t index) { return derive_seed(base, index); }

void* or_rs_new(std::uint64_t seed, std::uint64_t stream) { return new RandomSource(seed, stream); }
void or_rs_free(void* p) { delete static_cast<RandomSource*>(p); }
std::uint64_t or_rs_next_u64(void* p) { return static_cast<RandomSource*>(p)->next_u64(); }
double or_rs_uniform(void* p) { return static_cast<RandomSource*>(p)->uniform(); }
double or_rs_normal(void* p) { return static_cast<RandomSource*>(p)->normal(); }
int or_rs_normal_vector(void* p, std::int64_t len, double* out) {
  OR_TRY
  const Vec v = static_cast<RandomSource*>(p)->normal_vector(len);
  std::memcpy(out, v.data(), v.size() * sizeof(double));
  return 0;
  OR_CATCH
}
int or_rs_normal_complex_vector(void* p, std::int64_t len, double* out) {
  OR_TRY
  const Vec v = static_cast<RandomSource*>(p)->normal_complex_vector(len);
  std::memcpy(out, v.data(), v.size() * sizeof(double));
  return 0;
  OR_CATCH
}

// Reflector construction + application in one call (Python make_reflector /
// Reflector.apply stand-ins, module.cpp:48-66).
int or_make_reflector(const double* p, std::int64_t n, std::int64_t offset, double zero_tol, int rule,
                      double* w_out, double* c, double* s, int* identity) {
  OR_TRY
  const Reflector r = make_reflector(Vec(p, p + n), offset, zero_tol, static_cast<SignRule>(rule));
  *c = r.c;
  *s = r.s;
  *identity = r.identity ? 1 : 0;
  if (!r.identity) std::memcpy(w_out, r.w.data(), r.w.size() * sizeof(double));
  return 0;
  OR_CATCH
}
int or_reflector_apply(const double* p, std::int64_t n, std::int64_t offset, int rule, const double* x,
                       double* y) {
  OR_TRY
  const Reflector r = make_reflector(Vec(p, p + n), offset, 0.0, static_cast<SignRule>(rule));
  Vec v(x, x + n);
  r.apply_in_place(v);
  std::memcpy(y, v.data(), v.size() * sizeof(double));
  return 0;
  OR_CATCH
}

int or_op_new(int ensemble, std::int64_t m, std::int64_t n, double sigma, std::uint64_t seed,
              std::uint64_t stream, int skip_reflector, int sign_rule, void** out) {
  OR_TRY
  FaultFlags f;
  f.skip_reflector = skip_reflector != 0;
  f.sign_rule = static_cast<SignRule>(sign_rule);
  auto box = std::make_unique<OpBox>();
  box->ensemble = ensemble;
  if (ensemble == 0)
    box->op = std::make_unique<GinibreOperator>(m, n, sigma, RandomSource(seed, stream), f);
  else if (ensemble == 1)
    box->op = std::make_unique<HaarOperator>(n, RandomSource(seed, stream), f);
  else if (ensemble == 2)
    box->op = std::make_unique<GOEOperator>(n, sigma, RandomSource(seed, stream), f);
  else
    throw std::invalid_argument("unknown ensemble");
  *out = box.release();
  return 0;
  OR_CATCH
}
// An operator whose matrix stream is the given draw sequence (one vector per
// probe, in probe order) instead of RandomSource(seed, stream): the checker
// for device runs in Philox mode (draws exported by hd_philox_normals).
int or_op_new_queued(int ensemble, std::int64_t m, std::int64_t n, double sigma, const double* draws,
                     std::int64_t len, void** out) {
  OR_TRY
  auto q = std::make_shared<std::vector<double>>(draws, draws + len);
  RandomSource src(1, 0);
  src.set_queue(q);
  auto box = std::make_unique<OpBox>();
  box->ensemble = ensemble;
  if (ensemble == 0)
    box->op = std::make_unique<GinibreOperator>(m, n, sigma, src);
  else if (ensemble == 1)
    box->op = std::make_unique<HaarOperator>(n, src);
  else if (ensemble == 2)
    box->op = std::make_unique<GOEOperator>(n, sigma, src);
  else
    throw std::invalid_argument("unknown ensemble");
  *out = box.release();
  return 0;
  OR_CATCH
}
void or_op_free(void* p) { delete static_cast<OpBox*>(p); }
std::int64_t or_op_remaining(void* p) { return static_cast<OpBox*>(p)->op->remaining_probes(); }
std::int64_t or_op_rows(void* p) { return static_cast<OpBox*>(p)->op->rows(); }
std::int64_t or_op_cols(void* p) { return static_cast<OpBox*>(p)->op->cols(); }
void or_op_counts(void* p, std::int64_t* r, std::int64_t* l) {
  *r = static_cast<OpBox*>(p)->op->right_count();
  *l = static_cast<OpBox*>(p)->op->left_count();
}
int or_op_chain_sizes(void* p, std::int64_t* right, std::int64_t* left) {
  auto* b = static_cast<OpBox*>(p);
  if (auto* g = dynamic_cast<GinibreOperator*>(b->op.get())) {
    *right = g->right_chain_size();
    *left = g->left_chain_size();
  } else if (auto* h = dynamic_cast<HaarOperator*>(b->op.get())) {
    *right = h->right_chain_size();
    *left = h->left_chain_size();
  } else {
    *right = *left = -1;
  }
  return 0;
}
int or_op_probe(void* p, const double* x, std::int64_t len, int side, double* y, std::int64_t ylen) {
  OR_TRY
  auto* b = static_cast<OpBox*>(p);
  const Vec out = b->op->probe(Vec(x, x + len), static_cast<Side>(side));
  require(static_cast<std::int64_t>(out.size()) == ylen, "or_op_probe: output length mismatch");
  std::memcpy(y, out.data(), out.size() * sizeof(double));
  return 0;
  OR_CATCH
}

// Built-in dynamics (kinds match the device path). traj: (T+1) x dim when
// keep != 0 else just x_{T+1} (dim). x0 may be null (zeros).
int or_run_builtin(void* p, int kind, int side_rule, std::int64_t T, const double* x1, const double* x0,
                   std::int64_t dim, int keep, double* out) {
  OR_TRY
  auto* b = static_cast<OpBox*>(p);
  Vec v1(x1, x1 + dim);
  Vec v0;
  if (x0) v0.assign(x0, x0 + dim);
  const DynamicsSpec spec = builtin_spec(static_cast<UpdateKind>(kind), static_cast<SideRule>(side_rule), T, v1,
                                         x0 ? &v0 : nullptr, keep != 0);
  const std::vector<Vec> traj = run_dynamics(*b->op, spec);
  for (size_t i = 0; i < traj.size(); ++i)
    std::memcpy(out + i * static_cast<size_t>(dim), traj[i].data(), static_cast<size_t>(dim) * sizeof(double));
  return 0;
  OR_CATCH
}

// CPU timing harness (the reference's trial-parallel layout,
// parallel.hpp:17-52 + bench.cpp:35-54): `trials` independent runs of one
// builtin workload spread over `threads` std::threads; each trial owns its
// operator (seed = derive_seed(seed, trial)). Wall time in seconds, operator
// construction inside the clock like bench.cpp:42-45.
int or_bench_workload(int ensemble, std::int64_t m, std::int64_t n, double sigma, int kind, int side_rule,
                      std::int64_t T, std::uint64_t seed, int trials, int threads, double* seconds,
                      double* checksum) {
  OR_TRY
  require(trials >= 1 && threads >= 1, "or_bench_workload: trials/threads must be positive");
  std::atomic<int> next{0};
  std::vector<double> sums(static_cast<size_t>(trials), 0.0);
  std::mutex emu;
  std::exception_ptr first;
  const auto t0 = std::chrono::steady_clock::now();
  auto worker = [&] {
    for (;;) {
      const int i = next.fetch_add(1);
      if (i >= trials) return;
      try {
        const std::uint64_t s = derive_seed(seed, static_cast<std::uint64_t>(i));
        std::unique_ptr<ProbeOperator> op;
        if (ensemble == 0)
          op = std::make_unique<GinibreOperator>(m, n, sigma, RandomSource(s, 0));
        else if (ensemble == 1)
          op = std::make_unique<HaarOperator>(n, RandomSource(s, 0));
        else
          op = std::make_unique<GOEOperator>(n, sigma, RandomSource(s, 0));
        RandomSource data(s, 1);
        Vec x1 = data.normal_vector(op->cols());
        const double inv = 1.0 / norm(x1);
        for (double& v : x1) v *= inv;
        const DynamicsSpec spec = builtin_spec(static_cast<UpdateKind>(kind), static_cast<SideRule>(side_rule), T,
                                               x1, nullptr, false);
        const std::vector<Vec> tr = run_dynamics(*op, spec);
        double acc = 0.0;
        for (double v : tr.back()) acc += v;
        sums[static_cast<size_t>(i)] = acc;
      } catch (...) {
        std::lock_guard<std::mutex> g(emu);
        if (!first) first = std::current_exception();
      }
    }
  };
  std::vector<std::thread> pool;
  const int nt = std::min(threads, trials);
  for (int i = 1; i < nt; ++i) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  const auto t1 = std::chrono::steady_clock::now();
  if (first) std::rethrow_exception(first);
  *seconds = std::chrono::duration<double>(t1 - t0).count();
  double acc = 0.0;
  for (double v : sums) acc += v;
  *checksum = acc;
  return 0;
  OR_CATCH
}

// ---------------------------------------------------------------------------
// BASELINE configs 4 and 5 dynamics (not in the reference, SPEC.md:439 lists
// AMP as a non-goal; defined here and in paper_2101_07464_b200/lazymat):
//
// AMP for sparse regression on A = Ginibre m x n (entries N(0, sigma^2)),
// delta = m / n, y = A beta + w (one right probe, experiments.cpp:80-82):
//   x^0 = 0, z^0 = y; for t = 0 .. T-1:
//     r   = x^t + A^T z^t                       (left probe)
//     th  = alpha * ||z^t|| / sqrt(m)           (tau_t = ||z^t|| / sqrt(m))
//     x^{t+1} = soft(r, th)                     (experiments.cpp:31-39)
//     b   = (#{i : x^{t+1}_i != 0} / n) / delta (Onsager coefficient)
//     z^{t+1} = y - A x^{t+1} + b z^t           (right probe)
//   mse_t = ||x^{t+1} - beta||^2 / n.
static void amp_run(ProbeOperator& A, const double* beta, const double* w, std::int64_t T, double alpha,
                    double* x_out, double* mse_out);
static void spiked_run(ProbeOperator& G, const double* u, const double* x1, std::int64_t T, double theta,
                       double* x_out, double* overlap_out);

int or_amp(void* p, const double* beta, const double* w, std::int64_t T, double alpha, double* x_out,
           double* mse_out) {
  OR_TRY
  amp_run(*static_cast<OpBox*>(p)->op, beta, w, T, alpha, x_out, mse_out);
  return 0;
  OR_CATCH
}

int or_spiked_power(void* p, const double* u, const double* x1, std::int64_t T, double theta, double* x_out,
                    double* overlap_out) {
  OR_TRY
  spiked_run(*static_cast<OpBox*>(p)->op, u, x1, T, theta, x_out, overlap_out);
  return 0;
  OR_CATCH
}

// CPU timing of the config-4 / config-5 workloads (bench.py's reference arm
// and cpu_baseline): `trials` independent trials on `threads` threads (one
// trial per thread at a time, like parallel_for, parallel.hpp:17-52), each
// timed from operator construction (bench.cpp:42-53). Trial i uses
// derive_seed(seed, i): matrix stream 0, data stream 1 (experiments.cpp:122-125).
//   kind 0: AMP, Ginibre m = 2n, sigma = 1/sqrt(m), beta ~ Bernoulli(0.1) N(0,1)
//           (sample_bernoulli_gaussian with rho = 0.9, experiments.cpp:19-29),
//           w = 0.1 N(0, I_m), alpha = 1.5, T iterations (2T + 1 probes)
//   kind 1: spiked GOE, sigma = 1/sqrt(n), u and x_1 unit vectors from the
//           data stream, theta = 2, T steps (2T inner probes)
int or_bench_app(int kind, std::int64_t n, std::int64_t T, std::uint64_t seed, int trials, int threads,
                 double* seconds, double* checksum) {
  OR_TRY
  require(trials >= 1 && threads >= 1, "or_bench_app: trials/threads must be positive");
  std::atomic<int> next{0};
  std::vector<double> sums(static_cast<size_t>(trials), 0.0);
  std::mutex emu;
  std::exception_ptr first;
  const auto t0 = std::chrono::steady_clock::now();
  auto worker = [&] {
    for (;;) {
      const int i = next.fetch_add(1);
      if (i >= trials) return;
      try {
        const std::uint64_t s = derive_seed(seed, static_cast<std::uint64_t>(i));
        RandomSource data(s, 1);
        Vec out(static_cast<size_t>(n));
        if (kind == 0) {
          const Index m = 2 * n;
          GinibreOperator A(m, n, 1.0 / std::sqrt(double(m)), RandomSource(s, 0));
          Vec beta(static_cast<size_t>(n));
          for (auto& v : beta) v = (data.uniform() < 0.9) ? 0.0 : data.normal();
          Vec w = data.normal_vector(m);
          for (auto& v : w) v *= 0.1;
          amp_run(A, beta.data(), w.data(), T, 1.5, out.data(), nullptr);
        } else {
          GOEOperator G(n, 1.0 / std::sqrt(double(n)), RandomSource(s, 0));
          Vec u = data.normal_vector(n), x1 = data.normal_vector(n);
          const double iu = 1.0 / norm(u), ix = 1.0 / norm(x1);
          for (auto& v : u) v *= iu;
          for (auto& v : x1) v *= ix;
          spiked_run(G, u.data(), x1.data(), T, 2.0, out.data(), nullptr);
        }
        double acc = 0.0;
        for (double v : out) acc += v;
        sums[static_cast<size_t>(i)] = acc;
      } catch (...) {
        std::lock_guard<std::mutex> g(emu);
        if (!first) first = std::current_exception();
      }
    }
  };
  std::vector<std::thread> pool;
  const int nt = std::min(threads, trials);
  for (int i = 1; i < nt; ++i) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  const auto t1 = std::chrono::steady_clock::now();
  if (first) std::rethrow_exception(first);
  *seconds = std::chrono::duration<double>(t1 - t0).count();
  double acc = 0.0;
  for (double v : sums) acc += v;
  *checksum = acc;
  return 0;
  OR_CATCH
}

}  // extern "C"

static void amp_run(ProbeOperator& A, const double* beta, const double* w, std::int64_t T, double alpha,
                    double* x_out, double* mse_out) {
  const Index m = A.rows(), n = A.cols();
  const double delta = double(m) / double(n);
  Vec bv(beta, beta + n);
  Vec y = A.probe(bv, Side::right);
  for (Index i = 0; i < m; ++i) y[static_cast<size_t>(i)] += w[i];
  Vec x(static_cast<size_t>(n), 0.0), z = y;
  for (Index t = 0; t < T; ++t) {
    const Vec atz = A.probe(z, Side::left);
    const double th = alpha * norm(z) / std::sqrt(double(m));
    Index nnz = 0;
    for (Index i = 0; i < n; ++i) {
      const double r = x[static_cast<size_t>(i)] + atz[static_cast<size_t>(i)];
      const double mag = std::abs(r) - th;
      x[static_cast<size_t>(i)] = (mag > 0.0) ? (r > 0.0 ? mag : -mag) : 0.0;
      nnz += (mag > 0.0) ? 1 : 0;
    }
    const double onsager = (double(nnz) / double(n)) / delta;
    const Vec ax = A.probe(x, Side::right);
    for (Index i = 0; i < m; ++i)
      z[static_cast<size_t>(i)] = y[static_cast<size_t>(i)] - ax[static_cast<size_t>(i)] + onsager * z[static_cast<size_t>(i)];
    double e = 0.0;
    for (Index i = 0; i < n; ++i) {
      const double d = x[static_cast<size_t>(i)] - beta[i];
      e += d * d;
    }
    if (mse_out) mse_out[t] = e / double(n);
  }
  std::memcpy(x_out, x.data(), x.size() * sizeof(double));
}

// Spiked-GOE power method (BASELINE config 5): G = GOE probe operator,
// x_{t+1} = (G x_t + theta <u, x_t> u) / ||.||, u a unit vector.
static void spiked_run(ProbeOperator& G, const double* u, const double* x1, std::int64_t T, double theta,
                       double* x_out, double* overlap_out) {
  const Index n = G.cols();
  Vec x(x1, x1 + n);
  for (Index t = 0; t < T; ++t) {
    Vec gx = G.probe(x, Side::right);
    const double ux = dot(u, x.data(), n);
    for (Index i = 0; i < n; ++i) gx[static_cast<size_t>(i)] += theta * ux * u[i];
    const double nr = norm(gx);
    const double inv = nr > 0 ? 1.0 / nr : 1.0;
    for (Index i = 0; i < n; ++i) x[static_cast<size_t>(i)] = inv * gx[static_cast<size_t>(i)];
    if (overlap_out) overlap_out[t] = dot(u, x.data(), n);
  }
  std::memcpy(x_out, x.data(), x.size() * sizeof(double));
}
