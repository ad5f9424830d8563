// Host half of the reference RandomSource restatement (see hd_refrng.hpp).
// Compiled by g++ with the reference's flags (-O3 -mavx2 -mfma): the polar
// method's u*u + v*v and the ziggurat wedge test contract into the same FMAs
// as in the reference build, so the Gaussian stream matches bit for bit.
#include "hd_refrng.hpp"

namespace hd {
namespace refrng {
namespace {

// 256-strip ziggurat for exp(-x^2/2) (random.cpp:18-69). Strip s >= 1 covers
// [0, edge_s]; strip 0 is the base strip whose overhang beyond R is the tail.
struct ZigTables {
  static constexpr double R = 3.6541528853610088;  // random.cpp:27
  double scale[256];                                // mantissa -> magnitude
  double height[256];                               // f(edge_s)
  uint64_t accept[256];                             // 52-bit fast-accept bound
  ZigTables() {
    const double fR = std::exp(-0.5 * R * R);
    const double tail = std::sqrt(1.5707963267948966) * std::erfc(R / std::sqrt(2.0));
    const double area = R * fR + tail;  // common area of every strip
    double edge[256];
    edge[255] = R;
    for (int s = 254; s >= 1; --s) {
      const double f_up = std::exp(-0.5 * edge[s + 1] * edge[s + 1]);
      edge[s] = std::sqrt(-2.0 * std::log(area / edge[s + 1] + f_up));
    }
    edge[0] = 0.0;
    scale[0] = area / fR;
    accept[0] = static_cast<uint64_t>(R * fR / area * 0x1.0p52);
    height[0] = 1.0;
    for (int s = 1; s < 256; ++s) {
      scale[s] = edge[s];
      accept[s] = static_cast<uint64_t>(edge[s - 1] / edge[s] * 0x1.0p52);
      height[s] = std::exp(-0.5 * edge[s] * edge[s]);
    }
  }
};

const ZigTables& zig_tables() {
  static const ZigTables t;
  return t;
}

}  // namespace

double Source::normal() {  // random.cpp:106-121 (polar; caches the second value)
  if (spare_ok_) {
    spare_ok_ = false;
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
  spare_ok_ = true;
  return u * f;
}

// random.cpp:130-176: strip = low 8 bits, sign = bit 8, 52-bit mantissa from
// bits 12..63; fast accept, exact tail (strip 0), wedge test otherwise.
void Source::normal_fill(double* out, int64_t len) {
  const ZigTables& z = zig_tables();
  for (int64_t i = 0; i < len; ++i) {
    for (;;) {
      const uint64_t w = next();
      const unsigned s = static_cast<unsigned>(w & 0xFF);
      const uint64_t mant = w >> 12;
      const uint64_t sign = (w & 0x100) << 55;
      const double mag = (bits_to_double(0x3FF0000000000000ULL | mant) - 1.0) * z.scale[s];
      if (mant < z.accept[s]) {
        out[i] = bits_to_double(double_to_bits(mag) ^ sign);
        break;
      }
      if (s == 0) {
        double a, b;
        do {
          a = -std::log1p(-uniform()) * (1.0 / ZigTables::R);
          b = -std::log1p(-uniform());
        } while (b + b <= a * a);
        out[i] = bits_to_double(double_to_bits(ZigTables::R + a) ^ sign);
        break;
      }
      if (z.height[s] + uniform() * (z.height[s - 1] - z.height[s]) < std::exp(-0.5 * mag * mag)) {
        out[i] = bits_to_double(double_to_bits(mag) ^ sign);
        break;
      }
    }
  }
}

void Source::bernoulli_gaussian(double* out, int64_t n, double rho, double sigma_s) {
  for (int64_t i = 0; i < n; ++i) out[i] = (uniform() < rho) ? 0.0 : sigma_s * normal();
}

}  // namespace refrng
}  // namespace hd
