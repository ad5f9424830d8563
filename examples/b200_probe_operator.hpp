// A ProbeOperator-shaped C++ adapter over the C-ABI (include/hd.h): what a
// reference maintainer adds to route lazymat's operators (operators.hpp:29-49,
// ginibre.hpp:31-42, haar.hpp:24-31) to the B200 library. Plain std::vector
// in place of Eigen vectors; the reference's exception types map 1:1 onto the
// status codes.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "hd.h"

namespace b200 {

enum class Side { right, left };

struct BudgetExhausted : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ResourceCapExceeded : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == HD_OK) return;
  const std::string msg = hd_last_error();
  if (rc == HD_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == HD_ERR_BUDGET_EXHAUSTED) throw BudgetExhausted(msg);
  if (rc == HD_ERR_RESOURCE_CAP) throw ResourceCapExceeded(msg);
  throw std::runtime_error(msg);
}

class ProbeOperator {
 public:
  // ensemble: HD_GINIBRE / HD_HAAR / HD_GOE; draws: HD_DRAWS_REFERENCE gives
  // the reference's RandomSource(seed) stream, HD_DRAWS_PHILOX the device one
  ProbeOperator(int ensemble, int64_t m, int64_t n, double sigma, uint64_t seed, int draws = HD_DRAWS_PHILOX) {
    hd_config c{};
    c.ensemble = ensemble;
    c.dtype = HD_F64;
    c.m = m;
    c.n = n;
    c.sigma = sigma;
    c.seed = seed;
    c.draw_mode = draws;
    check(hd_create(&c, &op_));
  }
  ~ProbeOperator() { hd_destroy(op_); }
  ProbeOperator(const ProbeOperator&) = delete;
  ProbeOperator& operator=(const ProbeOperator&) = delete;

  int64_t rows() const {
    int64_t r, c;
    check(hd_shape(op_, &r, &c));
    return r;
  }
  int64_t cols() const {
    int64_t r, c;
    check(hd_shape(op_, &r, &c));
    return c;
  }
  int64_t remaining_probes() const {
    int64_t v;
    check(hd_remaining(op_, &v));
    return v;
  }
  // Q x (right) or Q^T x (left), host vectors in and out (operators.hpp:41)
  std::vector<double> probe(const std::vector<double>& x, Side side) {
    std::vector<double> y(side == Side::right ? rows() : cols());
    check(hd_probe(op_, x.data(), (int64_t)x.size(), y.data(), (int64_t)y.size(),
                   side == Side::right ? HD_RIGHT : HD_LEFT, 0, nullptr));
    return y;
  }
  hd_op* handle() { return op_; }

 private:
  hd_op* op_ = nullptr;
};

}  // namespace b200
