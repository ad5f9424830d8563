// TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT.
//
// CPU oracle: a plain C++20 restatement (no Eigen) of the reference's hot path
// in /root/reference/proj, used as the parity checker by tests/, by
// __graft_entry__.smoke() and as the CPU baseline leg of bench.py. The
// product library (paper_2101_07464_b200/) never links or calls this code.
//
// Why a restatement: the reference needs Eigen >= 3.3 (proj/CMakeLists.txt:12,
// include/lazymat/types.hpp:7), which is absent from the image, so it cannot
// be compiled here (oracle/_ref is "unbuildable").
//
// Pinning: the RNG is pinned bit-exactly by the reference's golden words
// (proj/tests/test_random.cpp:21-47, proj/tests/python/test_smoke.py:10-12);
// reflectors by the hand cases (proj/tests/test_reflect.cpp:25-64); the
// operators by the first-probe closed forms (proj/tests/test_ginibre.cpp:56-77,
// proj/tests/test_haar.cpp:35-45,98-111) and the property suites. Eigen's
// reduction order (third-party, version unpinned) is NOT reproduced, so
// floating-point parity with the reference is tolerance-level, not bitwise.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <memory>
#include <vector>

namespace hdo {

using Index = std::int64_t;
using Vec = std::vector<double>;

enum class Side { right = 0, left = 1 };
enum class SignRule { stable = 0, negative_at_zero = 1, zero_when_negative = 2 };

// types.hpp:32-43
struct BudgetExhausted : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ResourceCapExceeded : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// types.hpp:67-69
inline void require(bool cond, const std::string& msg) {
  if (!cond) throw std::invalid_argument(msg);
}

// ---------------------------------------------------------------- RNG
// random.cpp:73-76
std::uint64_t derive_seed(std::uint64_t base, std::uint64_t index);

// random.hpp:21-46, random.cpp:78-99
class Xoshiro256pp {
 public:
  explicit Xoshiro256pp(std::uint64_t seed);
  std::uint64_t next() {
    const std::uint64_t out = rotl(s_[0] + s_[3], 23) + s_[0];
    const std::uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return out;
  }
  void jump();

 private:
  static std::uint64_t rotl(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  std::array<std::uint64_t, 4> s_;
};

// random.hpp:55-112, random.cpp:101-188
class RandomSource {
 public:
  explicit RandomSource(std::uint64_t seed, std::uint64_t stream = 0);
  double uniform() { return static_cast<double>(eng_.next() >> 11) * 0x1.0p-53; }
  double normal();                        // polar method, random.cpp:106-121
  Vec normal_vector(Index len);           // ziggurat, random.cpp:130-176
  Vec normal_complex_vector(Index len);   // interleaved (re, im), random.cpp:178-188
  std::uint64_t next_u64() { return eng_.next(); }
  // Test-infrastructure hook (not in the reference): serve normal_vector from
  // a fixed queue of draws instead of the ziggurat, so the checker can consume
  // exactly the Gaussian stream the device generated (device Philox mode).
  void set_queue(std::shared_ptr<const std::vector<double>> q) {
    queue_ = std::move(q);
    qpos_ = 0;
  }

 private:
  std::shared_ptr<const std::vector<double>> queue_;
  size_t qpos_ = 0;
  Xoshiro256pp eng_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// ---------------------------------------------------------- reflectors
// reflect.hpp:47-104: (H x)[off:] = s * (x[off:] - c <w, x[off:]> w)
struct Reflector {
  Index dim = 0, offset = 0;
  Vec w;          // length dim - offset (empty for identity)
  double c = 0.0;
  double s = 1.0;
  bool identity = true;
  void apply_in_place(Vec& x) const;  // real: adjoint == plain
};

// reflect.hpp:120-176
Reflector make_reflector(const Vec& p, Index offset, double zero_tol = 0.0,
                         SignRule rule = SignRule::stable);

// reflect.hpp:193-231; order forward = append order, reverse = newest first
class ReflectorChain {
 public:
  explicit ReflectorChain(Index dim) : dim_(dim) { require(dim >= 1, "ReflectorChain: dim must be >= 1"); }
  Index size() const { return static_cast<Index>(m_.size()); }
  const Reflector& operator[](Index i) const { return m_[static_cast<size_t>(i)]; }
  void append(Reflector r) {
    require(r.dim == dim_, "ReflectorChain::append: dimension mismatch");
    m_.push_back(std::move(r));
  }
  void apply_forward(Vec& x) const;
  void apply_reverse(Vec& x) const;

 private:
  Index dim_;
  std::vector<Reflector> m_;
};

// --------------------------------------------------------- operators
struct FaultFlags {  // operators.hpp:16-22
  bool skip_reflector = false;
  SignRule sign_rule = SignRule::stable;
};

class ProbeOperator {  // operators.hpp:29-49
 public:
  virtual ~ProbeOperator() = default;
  virtual Index rows() const = 0;
  virtual Index cols() const = 0;
  virtual Index remaining_probes() const = 0;
  virtual Vec probe(const Vec& x, Side side) = 0;
  virtual Index right_count() const { return 0; }
  virtual Index left_count() const { return 0; }

 protected:
  void check_probe_input(const Vec& x, Side side) const;
};

// ginibre.hpp:26-118 (Algorithm 1)
class GinibreOperator final : public ProbeOperator {
 public:
  GinibreOperator(Index m, Index n, double sigma, RandomSource src, FaultFlags f = {});
  Index rows() const override { return m_; }
  Index cols() const override { return n_; }
  Index remaining_probes() const override { return std::min(m_, n_) - (r_ + l_); }
  Vec probe(const Vec& x, Side side) override;
  Index right_count() const override { return r_; }
  Index left_count() const override { return l_; }
  Index right_chain_size() const { return R_.size(); }
  Index left_chain_size() const { return L_.size(); }

 private:
  Index m_, n_;
  double sigma_;
  RandomSource src_;
  ReflectorChain L_, R_;
  std::vector<Vec> us_, vs_;
  Index r_ = 0, l_ = 0;
  FaultFlags f_;
};

// haar.hpp:21-76 (Algorithm 2)
class HaarOperator final : public ProbeOperator {
 public:
  HaarOperator(Index n, RandomSource src, FaultFlags f = {});
  Index rows() const override { return n_; }
  Index cols() const override { return n_; }
  Index remaining_probes() const override { return n_ - t_; }
  Vec probe(const Vec& x, Side side) override;
  Index right_count() const override { return t_; }
  Index right_chain_size() const { return R_.size(); }
  Index left_chain_size() const { return L_.size(); }

 private:
  Index n_;
  RandomSource src_;
  ReflectorChain L_, R_;
  Index t_ = 0;
  FaultFlags f_;
};

// ensembles.hpp:93-131: each matvec = (right + left probe of a square
// Ginibre)/sqrt(2); budget floor(inner / 2).
class GOEOperator final : public ProbeOperator {
 public:
  GOEOperator(Index n, double inner_sigma, RandomSource src, FaultFlags f = {});
  Index rows() const override { return inner_.rows(); }
  Index cols() const override { return inner_.cols(); }
  Index remaining_probes() const override { return inner_.remaining_probes() / 2; }
  Vec probe(const Vec& x, Side side) override;
  Index right_count() const override { return inner_.right_count(); }
  Index left_count() const override { return inner_.left_count(); }

 private:
  GinibreOperator inner_;
};

// ------------------------------------------------------------ dynamics
// dynamics.hpp:21-76
struct DynamicsSpec {
  Index iterations = 0;
  Index history_depth = 0;
  std::vector<Vec> initial;  // newest first
  std::function<Side(Index)> side_of;
  std::function<Vec(Index, const Vec&, const std::vector<Vec>&)> update;
  bool keep_trajectory = true;
};

std::vector<Vec> run_dynamics(ProbeOperator& op, const DynamicsSpec& spec);

// Built-in update maps shared with the device path (the BASELINE configs).
enum class UpdateKind {
  identity = 0,   // x_{t+1} = y_t
  normalize = 1,  // x_{t+1} = y / ||y|| (bench.cpp:25-28)
  tanh_mix = 2,   // x_{t+1} = tanh(2 y_t) + 0.1 x_{t-1} (BASELINE config 2)
};
enum class SideRule { alternate = 0, all_right = 1, all_left = 2 };

}  // namespace hdo
